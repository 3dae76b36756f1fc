"""Build a tuning variant of libtneat.so with extra nvcc -D knobs into
tools/_var/libtneat_<name>.so (git-ignored), for A/B timing with
`tools/time_step.py --lib`.
    python tools/build_variant.py NAME [-DKNOB=V ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01817_b200 import build as b  # noqa: E402

name, flags = sys.argv[1], sys.argv[2:]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(root, "tools", "_var"), exist_ok=True)
b.OUT = os.path.join(root, "tools", "_var", f"libtneat_{name}.so")
b.BUILD = os.path.join(root, "build", f"var_{name}")
os.environ["TNEAT_NVCC_EXTRA"] = " ".join(flags)
print(b.build(force=True))
