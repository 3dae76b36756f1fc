"""The reference's population-parallel scaling criterion (SPEC.md acceptance,
pkg/tests/test_acceptance.py:216-226) with the GPU path beside it:
run_bench over pop sizes {50, 200, 1000, 5000} x 20 generations, the
reference's tensorized (all host threads) and sequential paths timed on this
host, growth factors between the smallest and largest population and the
speedups at pop 5000.  One JSON line; bench.csv under the given directory.

    python tools/spec_scaling.py [out_dir] [generations]
"""

from __future__ import annotations

import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main() -> None:
    out_dir = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "gpurun_out", "spec_scaling")
    gens = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    ref_dir = os.path.join(REPO, "oracle", "_ref")
    sys.path.insert(0, ref_dir)
    import arrayneat  # the unmodified reference (oracle/build_ref.sh), timing only

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200.runner import run_bench
    pops = [50, 200, 1000, 5000]
    threads = os.cpu_count() or 1
    cfg = tn.NeatConfig(seed=0, problem="xor")
    path = run_bench(cfg, pops, gens, out_dir, threads=threads, reference=arrayneat)
    totals = {}
    with open(path) as fh:
        for row in csv.DictReader(fh):
            t = totals.setdefault(int(row["pop_size"]), [0.0, 0.0, 0.0])
            for k, col in enumerate(("tensorized_seconds", "sequential_seconds", "gpu_seconds")):
                t[k] += float(row[col])
    lo, hi = pops[0], pops[-1]
    growth = [totals[hi][k] / totals[lo][k] for k in range(3)]
    line = {
        "criterion": "SPEC acceptance: population-parallel scaling (pkg/tests/test_acceptance.py:216-226)",
        "generations": gens, "host_threads": threads, "pop_sizes": pops,
        "total_seconds": {str(p): {"reference_tensorized": v[0], "reference_sequential": v[1], "gpu": v[2]}
                          for p, v in totals.items()},
        "growth_reference_tensorized": growth[0], "growth_reference_sequential": growth[1],
        "growth_gpu": growth[2],
        "ratio_reference_tensorized": growth[0] / growth[1], "ratio_gpu": growth[2] / growth[1],
        "speedup_at_5000_reference_tensorized": totals[hi][1] / totals[hi][0],
        "speedup_at_5000_gpu_vs_sequential": totals[hi][1] / totals[hi][2],
        "speedup_at_5000_gpu_vs_tensorized": totals[hi][0] / totals[hi][2],
        "pass_gpu": growth[2] / growth[1] <= 0.25 and totals[hi][1] / totals[hi][2] >= 4.0,
        "bench_csv": os.path.relpath(path, REPO),
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
