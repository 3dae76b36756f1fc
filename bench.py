"""Benchmark: population forward sweep (BASELINE.json configs[1]).

Workload per rank: pop 10k synthetic feed-forward genomes, max_nodes 128 /
max_conns 512, I=32, O=8, 4096 synthetic inputs per genome (5.2 GB fp32,
larger than the 126 MB L2, so no flush is needed between steps).  One step =
transform (K1, Kahn + CSR program) + forward (K2) of the whole population.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 is launched by torchrun (one rank per GPU, NCCL); the population is
partitioned with no data-path collective (weak scaling: 10k genomes per rank);
time is the max over ranks.  ``--impl reference`` times the reference CPU
implementation (oracle/_ref = the unmodified reference arrayneat, else the
oracle port) on the host cores.  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "genome-input evaluations/sec at pop 10k (population forward sweep)"
UNIT = "genome-input evals/s"
POP, MAXN, MAXC, NIN, NOUT, BATCH = 10_000, 128, 512, 32, 8, 4096
CONFIG = {
    "workload": "population forward sweep (BASELINE configs[1]): transform + forward",
    "pop_per_rank": POP, "max_nodes": MAXN, "max_conns": MAXC, "inputs": NIN, "outputs": NOUT,
    "inputs_per_genome": BATCH, "genomes": "synthetic SURVEY §8d generator, tanh/sum",
    "l2": "inputs 5.2 GB/rank > 126 MB L2 (no flush needed)",
    "step": "transform + forward per step; step k+1's transform overlaps step k's forward (two streams)",
}


def _parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--pop", type=int, default=POP)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clock and throttle reasons sampled every 20 ms during the timed
    region, in-process through NVML (no nvidia-smi child competing for the
    driver); falls back to `nvidia-smi -lms` when NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, list[str]]] = []
        self.proc = None
        self.thread = None
        self.stop_evt = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:  # noqa: BLE001 -- fall back to the CLI
            h = None
        if h is not None:
            self.thread = threading.Thread(target=self._nvml, args=(h,), daemon=True)
            self.thread.start()
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _nvml(self, h):
        import pynvml
        bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not self.stop_evt.is_set():
            try:
                sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:  # noqa: BLE001
                break
            self.samples.append((time.perf_counter(), [str(sm), str(mx)] +
                                 ["Active" if r & b else "Not Active" for b in bits]))
            self.stop_evt.wait(0.02)

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def stop(self):
        self.stop_evt.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0: float, t1: float) -> dict:
        rows = [r for t, r in self.samples if t0 <= t <= t1] or [r for _, r in self.samples[-5:]]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4)
                          if len(r) > 2 + k and r[2 + k].lower().startswith("active")})
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# reference CPU arm
# ---------------------------------------------------------------------------

def _load_reference():
    """(module, kind): the unmodified reference from oracle/_ref, else the port."""
    ref_dir = os.path.join(REPO, "oracle", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "arrayneat")):
        sys.path.insert(0, ref_dir)
        import arrayneat  # noqa: F401
        from arrayneat import inference
        return inference, "reference"
    return None, "port"


_CAL: dict = {}


def cpu_forward_rate(nodes, conns, x, seconds: float, threads: int | None = None) -> dict:
    """Time the reference transform+forward on a bounded sample of the same
    workload, genome work items of 4 (bounds the (P,B,N) float64
    temporaries), on all host cores."""
    from concurrent.futures import ThreadPoolExecutor
    inference, kind = _load_reference()
    threads = threads or min(os.cpu_count() or 1, 32)
    item = 4
    if inference is not None:
        from arrayneat.functions import DEFAULT_REGISTRY

        def work(lo):
            st, cyc = inference.transform_arrays(nodes[lo:lo + item], conns[lo:lo + item], NIN, NOUT)
            return inference.forward_arrays(st, DEFAULT_REGISTRY, x[lo:lo + item].astype(np.float64)).shape
    else:
        from oracle import arrayneat_oracle as orc

        def work(lo):
            for p in range(lo, min(lo + item, nodes.shape[0])):
                tr = orc.transform_genome(nodes[p], conns[p], NIN, NOUT)
                orc.forward_genome(nodes[p], tr, x[p].astype(np.float64))
            return None
    # calibrate on one item (once per process), then size the sample to ~`seconds`
    per_item = _CAL.get(kind)
    if per_item is None:
        t = time.perf_counter()
        work(0)
        per_item = _CAL[kind] = time.perf_counter() - t
    n_items = max(threads, int(seconds * threads / max(per_item, 1e-3)))
    n_items = min(n_items, nodes.shape[0] // item)
    starts = [(k * item) % (nodes.shape[0] - item + 1) for k in range(n_items)]
    t = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(work, starts))
    dt = time.perf_counter() - t
    evals = n_items * item * x.shape[1]
    return {"value": evals / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n_items * item} genomes x {x.shape[1]} inputs ({evals} evals, {dt:.1f} s), "
                      f"work items of {item} genomes on {threads} threads"}


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    from paper_2404_01817_b200.synthetic import synthetic_population
    threads = min(os.cpu_count() or 1, 32)
    nodes, conns = synthetic_population(max(64, 4 * threads), MAXN, MAXC, NIN, NOUT, seed=20261018)
    x = np.random.default_rng(20261019).standard_normal((nodes.shape[0], BATCH, NIN), dtype=np.float32)
    per_step = max(0.5, min(10.0, 60.0 / max(1, args.steps + args.warmup)))  # whole run ~1 min
    for _ in range(args.warmup):
        cpu_forward_rate(nodes, conns, x, per_step / 4, threads)
    rates = [cpu_forward_rate(nodes, conns, x, per_step, threads) for _ in range(args.steps)]
    value = float(np.median([r["value"] for r in rates]))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * POP * BATCH / value, "higher_is_better": True,
            "step_note": (f"ms_per_step = one full {POP}-genome x {BATCH}-input step at the measured rate; each "
                          f"timed step runs a bounded sample for ~{per_step:.0f} s (cpu_baseline.sample)"),
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(CONFIG, parallelism="host threads"),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": rates[0]["kind"],
                             "sample": rates[0]["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def _peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def _ncu_traffic() -> float | None:
    path = os.path.join(REPO, "profiles", "forward_ncu_summary.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["dram_bytes_per_launch"])
    except (OSError, KeyError, ValueError):
        return None


def run_ours(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200.synthetic import synthetic_population

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    pop = args.pop
    nodes_h, conns_h = synthetic_population(pop, MAXN, MAXC, NIN, NOUT, seed=20261018 + rank)
    nodes = torch.from_numpy(nodes_h).to(dev)
    conns = torch.from_numpy(conns_h).to(dev)
    gen = torch.Generator(device=dev).manual_seed(20261019 + rank)
    x = torch.randn((pop, BATCH, NIN), device=dev, dtype=torch.float32, generator=gen)
    out = torch.empty((pop, BATCH, NOUT), device=dev, dtype=torch.float32)

    # A step = transform + forward of the whole population.  Steps are
    # pipelined: step k+1's transform (and its launch-size read-back) runs on a
    # second stream while step k's forward runs, so the host round trip and the
    # transform tail overlap the previous forward.  All work of every step is
    # inside the timed region.
    fw = torch.cuda.current_stream()
    tr = torch.cuda.Stream()
    live: list = []
    fdone: list = []

    def step():
        # at most one forward ahead of the transform: step k+1's transform starts
        # once forward k-1 has finished (it then overlaps forward k only)
        if len(fdone) >= 2:
            fdone.pop(0).synchronize()
        with torch.cuda.stream(tr):
            st, _ = tn.transform_arrays(nodes, conns, NIN, NOUT, sync=False)
            tn.finalize_transform(st)            # 12-byte launch-size read-back
        ready = torch.cuda.Event()
        ready.record(tr)
        fw.wait_event(ready)
        for t in (st.program, st.status_dev):
            t.record_stream(fw)
        tn.forward_device(st, x, out, variant=args.variant, stream=fw)
        ev = torch.cuda.Event()
        ev.record(fw)
        fdone.append(ev)
        live.append(st)
        if len(live) > 2:
            live.pop(0)
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    import gc
    gc.collect()
    gc.disable()  # no collector pauses between the host's per-step launches
    sampler = ClockSampler(dev.index)
    sampler.start()
    time.sleep(0.2)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(fw)
    tr.wait_event(s0)
    st = None
    trace = os.environ.get("TNEAT_BENCH_TRACE")  # diagnostics: per-step host times to stderr
    host_t = []
    for _ in range(args.steps):
        if trace:
            host_t.append(time.perf_counter())
        st = step()
    done = torch.cuda.Event()
    done.record(tr)
    fw.wait_event(done)
    s1.record(fw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall1 = time.perf_counter()
    gc.enable()
    if trace and host_t:
        gaps = np.diff(np.array(host_t + [t_wall1])) * 1e3
        print(f"trace: host ms per step median {np.median(gaps):.2f} max {gaps.max():.2f} "
              f"at step {int(gaps.argmax())}; total {1e3 * (t_wall1 - host_t[0]):.1f} ms", file=sys.stderr)
    elapsed = s0.elapsed_time(s1) / 1e3
    # forward kernel time for the roofline: the same forward, not overlapped
    pairs = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(fw)
        tn.forward_device(st, x, out, variant=args.variant, stream=fw)
        e1.record(fw)
        pairs.append((e0, e1))
    torch.cuda.synchronize()
    fwd_ms = [a.elapsed_time(b) for a, b in pairs]
    if world > 1:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    evals = pop * BATCH * world * args.steps
    value = evals / elapsed

    # algorithmic bytes of one forward launch: inputs + outputs + each genome's program once
    hdr = st.program[:, :32].contiguous().view(torch.int32).to(torch.int64).cpu().numpy()
    # header + output slots + groups + steps + edge entries (common.cuh layout)
    prog_bytes = int((32 + 16 + 16 * hdr[:, 7] + 16 * hdr[:, 0] + 6 * hdr[:, 1]).sum())
    launches_per_step = 1 + len(tn.inference._bucket_plan(st, (args.variant & 0xF) or 5))
    algo_bytes = pop * BATCH * 4 * (NIN + NOUT) + prog_bytes
    fwd_avg = statistics.mean(fwd_ms) / 1e3
    peak, peak_kind = _peaks()
    achieved = algo_bytes / fwd_avg / 1e9

    # e2e: pinned host genomes + pinned host inputs -> pinned host outputs through the public API
    e2e = None
    if not args.no_e2e:
        xh = torch.empty((pop, BATCH, NIN), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        oh = torch.empty((pop, BATCH, NOUT), dtype=torch.float32, pin_memory=True)
        nodes_p = torch.from_numpy(nodes_h).pin_memory()
        conns_p = torch.from_numpy(conns_h).pin_memory()
        for _ in range(1):
            sth, _ = tn.transform_arrays(nodes_p, conns_p, NIN, NOUT)
            tn.forward_arrays(sth, None, xh, out=oh)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(args.e2e_steps):
            sth, _ = tn.transform_arrays(nodes_p, conns_p, NIN, NOUT)
            tn.forward_arrays(sth, None, xh, out=oh)
        torch.cuda.synchronize()
        e2e_dt = time.perf_counter() - t
        if world > 1:
            tt = torch.tensor([e2e_dt], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_dt = float(tt.item())
        e2e = {"value": pop * BATCH * world * args.e2e_steps / e2e_dt, "unit": UNIT,
               "h2d_bytes_per_step": int(nodes_h.nbytes + conns_h.nbytes + xh.numel() * 4),
               "d2h_bytes_per_step": int(oh.numel() * 4 + 12 + 4 * pop),
               "steps": args.e2e_steps,
               "path": "transform_arrays(pinned host genomes) + forward_arrays(pinned host inputs)"}
        del xh, oh, nodes_p, conns_p
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sub = 256
        cpu = cpu_forward_rate(nodes_h[:sub], conns_h[:sub], x[:sub].cpu().numpy(), args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(CONFIG, parallelism=f"population shards x{world} (no data-path collective)"),
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _ncu_traffic(),
                         "kernel": "fwd_tile_kernel", "algo_bytes_per_launch": algo_bytes,
                         "avg_launch_ms": fwd_avg * 1e3, "peak_kind": peak_kind,
                         "forward_only_evals_per_s": pop * BATCH / fwd_avg},
            "cpu_baseline": cpu,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)


def main():
    args = _parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    # a small, fixed host thread pool per rank for the per-step host work
    # (launch planning, read-backs): torchrun's OMP_NUM_THREADS=1 starves it and
    # a pool of every core makes it erratic
    import torch
    torch.set_num_threads(max(1, min(8, (os.cpu_count() or 8) // max(1, world))))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
