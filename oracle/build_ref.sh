#!/usr/bin/env bash
# Build the reference checker into oracle/_ref (TEST INFRASTRUCTURE ONLY).
#
# The reference (arrayneat 0.1.0, /root/reference/pkg) is pure Python + NumPy,
# so "building" it means installing its wheel, unmodified, into oracle/_ref.
# The install is git-ignored but NOT gpurun-ignored: it travels to the GPU box
# where bench.py's cpu_baseline / --impl reference leg times it on the host
# cores.  /root/reference is read-only, so the build runs from a /tmp copy.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src="${1:-/root/reference/pkg}"
if [ ! -f "$src/pyproject.toml" ]; then
    echo "build_ref: reference not found at $src (nothing to do)" >&2
    exit 0
fi
tmp="$(mktemp -d /tmp/arrayneat_ref.XXXXXX)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"
rm -rf "$here/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$here/_ref" "$tmp/pkg"
echo "build_ref: installed $(ls "$here/_ref" | grep -c arrayneat) arrayneat entries into $here/_ref"
