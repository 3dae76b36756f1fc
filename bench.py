"""Benchmark: population forward sweep (BASELINE.json configs[1]).

Workload: pop 10k synthetic feed-forward genomes, max_nodes 128 / max_conns
512, I=32, O=8, 4096 synthetic inputs per genome (5.2 GB fp32, larger than the
126 MB L2, so no flush is needed between steps).  One step = the population's
evaluation: transform (K1, Kahn + programs) + forward (K2, tensor-core input
layer, device-side launch plan) + per-genome fitness (-mean squared output)
+ NCCL all-gather of the fitness vector.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1: strong scaling -- the 10k population is split into contiguous shards
of 10k/N genomes, one rank per GPU over NCCL; each step ends
with the fitness all-gather (P x 4 bytes); time is the max over ranks.  Run
without torchrun, ``--gpus N`` re-launches itself under torch.distributed.run.
``--impl reference`` times the reference CPU implementation (oracle/_ref =
the unmodified reference arrayneat, else the oracle port) on the host cores
(rank 0 only).  Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
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
    "workload": "population forward sweep (BASELINE configs[1]): transform + forward + fitness + all-gather",
    "pop": POP, "max_nodes": MAXN, "max_conns": MAXC, "inputs": NIN, "outputs": NOUT,
    "inputs_per_genome": BATCH, "genomes": "synthetic SURVEY §8d generator, tanh/sum",
    "l2": "inputs 5.2 GB > 126 MB L2 (no flush needed)",
    "step": "transform + forward (device launch plan, no host sync; fused fitness epilogue) + NCCL "
            "all-gather of the fitness, enqueued on one stream",
}


def _parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--pop", type=int, default=POP)
    ap.add_argument("--layout", default="auto", choices=["auto", "tc", "standard"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
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
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
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


def _ncu_traffic() -> dict:
    """DRAM traffic of one whole forward pass (every launch of the pass summed)
    from the committed ncu capture (profiles/forward_ncu_summary.json)."""
    path = os.path.join(REPO, "profiles", "forward_ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return {"bytes": float(d["dram_bytes_per_pass"]), "source": d.get("source", path)}
    except (OSError, KeyError, ValueError):
        return {"bytes": None, "source": None}


def _program_bytes(tn, st) -> int:
    """Algorithmic program bytes of a pass: what each genome's launch stages
    (header + output slots + the tensor-core block, or the standard program's
    groups / steps / edge entries)."""
    import torch
    hdr = st.program[:, :32].contiguous().view(torch.int32).to(torch.int64).cpu().numpy()
    steps, edges, groups, mode = hdr[:, 0], hdr[:, 1], hdr[:, 7], hdr[:, 6]
    nb = (steps + 15) // 16 * 16
    tc = 192 * nb + 4 * nb + 16 * groups + 16 * steps + 8 * edges
    std = 16 * groups + 16 * steps + 6 * edges
    return int((32 + 2 * NOUT + np.where(mode == 2, tc, std)).sum())


def cpu_info() -> dict:
    """Host of the CPU baseline: model, cores, numpy's SIMD dispatch."""
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except (OSError, subprocess.TimeoutExpired):
        pass
    simd = {}
    try:
        from numpy._core._multiarray_umath import __cpu_baseline__, __cpu_dispatch__, __cpu_features__
        simd = {"baseline": list(__cpu_baseline__),
                "dispatch_available": [f for f in __cpu_dispatch__ if __cpu_features__.get(f)]}
    except ImportError:
        pass
    return {"model": model, "cpu_count": os.cpu_count(), "numpy": np.__version__, "numpy_simd": simd}


def secondary(dev) -> dict:
    """BASELINE configs 1, 3, 4, 5 and the float64 forward, bounded (~1 min):
    GPU numbers next to the reference on the same host where a reference
    exists (tools/bench_configs.py holds the measurements)."""
    import types

    import torch

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200.synthetic import synthetic_population
    sys.path.insert(0, os.path.join(REPO, "tools"))
    import bench_configs as bc
    out = {}
    t_all = time.perf_counter()

    def timed(name, fn):
        t = time.perf_counter()
        try:
            out[name] = fn()
        except Exception as e:  # noqa: BLE001 -- one failing config must not lose the headline
            out[name] = {"error": f"{type(e).__name__}: {e}"}
        out[name + "_wall_s"] = round(time.perf_counter() - t, 2)

    timed("config1_xor", lambda: bc.bench_xor(types.SimpleNamespace(seed=0, gens=100, no_cpu=False)))
    timed("config3_generation_1m", lambda: bc.bench_generation(
        types.SimpleNamespace(pop=1_000_000, gens=5, ref_pop=0)))
    timed("config3_generation_100k", lambda: bc.bench_generation(
        types.SimpleNamespace(pop=100_000, gens=5, ref_pop=100_000)))
    timed("config4_hyperneat", lambda: bc.bench_hyperneat(types.SimpleNamespace(pop=10_000, no_cpu=False)))
    timed("config5_recurrent", lambda: bc.bench_recurrent(
        types.SimpleNamespace(pop=10_000, steps=1000, sweeps=[5], no_cpu=False)))
    rec = out.get("config5_recurrent") or {}
    for r in rec.get("runs", []) if isinstance(rec, dict) else []:
        # FP32 work per genome-step: K (2 E_en + N_act) + 2*27*(27+8),
        # with the config's mean enabled edges / evaluated nodes of the rollout programs
        fl = r["sweeps"] * (2 * 330 + 90) + 2 * 27 * 35
        r["fp32_tflops_est"] = r["genome_steps_per_s"] * fl / 1e12
        r["fp32_frac_of_74tf"] = r["fp32_tflops_est"] / 74.0

    def f64_forward():
        n = 10_000
        nodes_h, conns_h = synthetic_population(n, MAXN, MAXC, NIN, NOUT, seed=20261018)
        x = torch.randn((n, BATCH, NIN), device=dev, dtype=torch.float64,
                        generator=torch.Generator(device=dev).manual_seed(3))
        st, _ = tn.transform_arrays(torch.from_numpy(nodes_h).to(dev), torch.from_numpy(conns_h).to(dev), NIN,
                                    NOUT, precision="f64")
        o = tn.forward_device(st, x)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            tn.forward_device(st, x, o)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        del x, o
        return {"pop": n, "inputs_per_genome": BATCH, "forward_ms": ms, "evals_per_s": n * BATCH / (ms / 1e3),
                "note": "f64 programs (reference precision), standard tile kernel"}

    timed("f64_forward", f64_forward)
    out["total_wall_s"] = round(time.perf_counter() - t_all, 1)
    torch.cuda.empty_cache()
    return out


def shard_of(total: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous equal shard of the population for ``rank`` (strong scaling,
    SURVEY.md §8e): [lo, lo + total / world)."""
    if total % world:
        raise SystemExit(f"pop {total} is not divisible by {world} ranks")
    shard = total // world
    return rank * shard, shard


def gather_fitness(fit_local, fit_all, world: int) -> None:
    """The step's one collective: every rank receives the whole (P,) fitness
    vector (NCCL all-gather over NVLink; gloo in the CPU tests)."""
    import torch.distributed as dist
    if world > 1:
        dist.all_gather_into_tensor(fit_all, fit_local)
    else:
        fit_all.copy_(fit_local)


def _tc_launches(max_nodes: int) -> int:
    """Kernel launches of one device-planned forward (csrc/forward.cu
    launch_planned): the plan, one per MMA-width class a genome of this
    capacity can reach (32/48/64/96/128), the oversized class, the standard one."""
    cap = (min(max_nodes, 128) + 15) // 16 * 16
    nbs = (32, 48, 64, 96, 128)
    width = sum(1 for c, nb in enumerate(nbs) if not (c > 0 and nb > cap and nbs[c - 1] >= cap))
    return 1 + width + 1 + 1


def _local_device() -> int:
    """This rank's GPU.  TNEAT_BENCH_SHARE_GPU=1 (tests of the multi-rank path on
    a one-GPU box, with TNEAT_BENCH_BACKEND=gloo) puts every rank on cuda:0."""
    return 0 if os.environ.get("TNEAT_BENCH_SHARE_GPU") else int(os.environ.get("LOCAL_RANK", 0))


def _free_port() -> int:
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def run_ours(args, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_2404_01817_b200 as tn
    from paper_2404_01817_b200.synthetic import synthetic_population

    dev = torch.device("cuda", _local_device())
    torch.cuda.set_device(dev)
    total = args.pop
    lo, shard = shard_of(total, world, rank)
    # the same 10k population for every world size; rank r owns genomes [lo, lo + shard)
    nodes_all, conns_all = synthetic_population(total, MAXN, MAXC, NIN, NOUT, seed=20261018)
    nodes_h, conns_h = nodes_all[lo:lo + shard].copy(), conns_all[lo:lo + shard].copy()
    del nodes_all, conns_all
    nodes = torch.from_numpy(nodes_h).to(dev)
    conns = torch.from_numpy(conns_h).to(dev)
    gen = torch.Generator(device=dev).manual_seed(20261019 + rank)
    x = torch.randn((shard, BATCH, NIN), device=dev, dtype=torch.float32, generator=gen)
    out = torch.empty((shard, BATCH, NOUT), device=dev, dtype=torch.float32)
    fit_all = torch.empty((total,), device=dev, dtype=torch.float32)
    sq = torch.zeros((shard,), device=dev, dtype=torch.float32)

    # A step = transform + forward + fitness + all-gather.  With tensor-core
    # programs the forward plans its launches on the device, so nothing in a
    # step waits for the host; step k+1's transform (second stream) overlaps
    # step k's forward.
    fw = torch.cuda.current_stream()
    tr = torch.cuda.Stream()
    live: list = []
    tc_layout = args.layout in ("auto", "tc")

    dbg = os.environ.get("TNEAT_BENCH_DEBUG", "")  # diagnostics only: "notransform", "nofit"
    st_fixed = []

    def step():
        if "notransform" in dbg and st_fixed:
            st = st_fixed[0]
            sq.zero_()
            tn.forward_device(st, x, out, variant=args.variant, stream=fw, sq_sum=sq)
            fit_all.copy_(sq.mul(-1.0 / (BATCH * NOUT)))
            return st
        # tensor-core programs: one stream (the persistent forward leaves no room
        # for the transform's CTAs, so a second stream would only interleave
        # them nondeterministically); standard programs: the transform runs on a
        # second stream inside the forward's bucket boundaries
        tstream = tr if not tc_layout else fw
        with torch.cuda.stream(tstream):
            st, _ = tn.transform_arrays(nodes, conns, NIN, NOUT, sync=False, layout=args.layout)
        if "notransform" in dbg:
            st_fixed.append(st)
        if tstream is not fw:
            ready = torch.cuda.Event()
            ready.record(tr)
            fw.wait_event(ready)
            for t in (st.program, st.status_dev):
                t.record_stream(fw)
        if not st.precision & tn.inference.FMT_TC:
            tn.finalize_transform(st)  # standard programs: host bucket plan (read-back)
        if "nofit" in dbg:
            tn.forward_device(st, x, out, variant=args.variant, stream=fw)
        else:
            # per-genome fitness -mean squared output: the forward's fused epilogue sums
            # each genome's squared outputs (no extra pass over the outputs)
            sq.zero_()
            tn.forward_device(st, x, out, variant=args.variant, stream=fw, sq_sum=sq)
            gather_fitness(sq.mul(-1.0 / (BATCH * NOUT)), fit_all, world)
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
    for _ in range(args.steps):
        st = step()
    s1.record(fw)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_wall1 = time.perf_counter()
    gc.enable()
    elapsed = s0.elapsed_time(s1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    evals = total * BATCH * args.steps
    value = evals / elapsed

    # the forward pass alone (every launch of one pass: device plan + class
    # launches), not overlapped -- the roofline's denominator
    def time_forward(stk, reps=5):
        pairs = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(fw)
            tn.forward_device(stk, x, out, variant=args.variant, stream=fw)
            e1.record(fw)
            pairs.append((e0, e1))
        torch.cuda.synchronize()
        return statistics.mean(a.elapsed_time(b) for a, b in pairs) / 1e3

    fwd_avg = time_forward(st)
    st_np, _ = tn.transform_arrays(nodes, conns, NIN, NOUT, prune=False, layout=args.layout)
    fwd_unpruned = time_forward(st_np, 3)
    tn.finalize_transform(st)
    prog_bytes = _program_bytes(tn, st)
    if st.precision & tn.inference.FMT_TC:
        launches_fwd = _tc_launches(MAXN)
        kernel = "fwd_tc_kernel (+ plan_tc_kernel, fwd_tile_kernel for standard programs)"
    else:
        launches_fwd = len(tn.inference._bucket_plan(st, (args.variant & 0xF) or 5))
        kernel = "fwd_tile_kernel"
    algo_bytes = shard * BATCH * 4 * (NIN + NOUT) + prog_bytes
    peak, peak_kind = _peaks()
    achieved = algo_bytes / fwd_avg / 1e9
    del st_np

    # e2e: pinned host genomes + pinned host inputs -> pinned host outputs through the public API
    e2e = None
    if not args.no_e2e:
        xh = torch.empty((shard, BATCH, NIN), dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        oh = torch.empty((shard, BATCH, NOUT), dtype=torch.float32, pin_memory=True)
        nodes_p = torch.from_numpy(nodes_h).pin_memory()
        conns_p = torch.from_numpy(conns_h).pin_memory()
        sth, _ = tn.transform_arrays(nodes_p, conns_p, NIN, NOUT, layout=args.layout)
        tn.forward_arrays(sth, None, xh, out=oh)
        torch.cuda.synchronize()
        e2e_steps = []
        for _ in range(args.e2e_steps):
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            sth, _ = tn.transform_arrays(nodes_p, conns_p, NIN, NOUT, layout=args.layout)
            tn.forward_arrays(sth, None, xh, out=oh)  # returns after the outputs are on the host
            torch.cuda.synchronize()
            dt_step = time.perf_counter() - t
            if world > 1:
                tt = torch.tensor([dt_step], device=dev, dtype=torch.float64)
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt_step = float(tt.item())
            e2e_steps.append(dt_step)
        e2e_dt = statistics.median(e2e_steps)
        e2e = {"value": total * BATCH / e2e_dt, "unit": UNIT, "ms_per_step_each": [1e3 * v for v in e2e_steps],
               "h2d_bytes_per_step": int(nodes_h.nbytes + conns_h.nbytes + xh.numel() * 4),
               "d2h_bytes_per_step": int(oh.numel() * 4 + 4 * shard + 16 * shard + 12),
               "steps": args.e2e_steps, "statistic": "median of the per-step wall times (host clock, synchronised)",
               "path": "transform_arrays(pinned host genomes) + forward_arrays(pinned host inputs)"}
        del xh, oh, nodes_p, conns_p
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)

    cpu = None
    sec = None
    if rank == 0 and world == 1 and not args.no_cpu:
        sub = 256
        xs = x[:sub].cpu().numpy()
        threads = min(os.cpu_count() or 1, 32)
        cpu = cpu_forward_rate(nodes_h[:sub], conns_h[:sub], xs, args.cpu_seconds, threads)
        one = cpu_forward_rate(nodes_h[:sub], conns_h[:sub], xs, max(2.0, args.cpu_seconds / 4), 1)
        cpu["one_thread"] = {"value": one["value"], "sample": one["sample"]}
        cpu["host"] = cpu_info()
    if rank == 0 and world == 1 and not args.no_secondary:
        del x, out
        torch.cuda.empty_cache()
        sec = secondary(dev)

    if rank == 0:
        traffic = _ncu_traffic()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(CONFIG, parallelism=f"contiguous population shards x{world} ({shard} genomes "
                                               f"per rank), NCCL all-gather of fitness"),
            "e2e": e2e,
            "gpu_launches": (1 + launches_fwd) * args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic["bytes"], "traffic_source": traffic["source"],
                         "kernel": kernel, "launches_per_pass": launches_fwd,
                         "algo_bytes_per_launch": algo_bytes, "avg_launch_ms": fwd_avg * 1e3,
                         "peak_kind": peak_kind, "forward_only_evals_per_s": shard * BATCH / fwd_avg,
                         "unpruned_forward_ms": fwd_unpruned * 1e3,
                         "note": "one launch = one forward pass over this rank's shard (all of its kernel "
                                 "launches); algorithmic bytes = inputs + outputs + staged program bytes"},
            "cpu_baseline": cpu,
            "clocks": clocks,
            "secondary": sec,
        }
        print(json.dumps(line), flush=True)


def main():
    args = _parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one rank per GPU: re-launch under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1 and args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank)
        return
    # a small, fixed host thread pool per rank for the per-step host work
    # (launch planning, read-backs): torchrun's OMP_NUM_THREADS=1 starves it and
    # a pool of every core makes it erratic
    import torch
    torch.set_num_threads(max(1, min(8, (os.cpu_count() or 8) // max(1, world))))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(_local_device())
        backend = os.environ.get("TNEAT_BENCH_BACKEND", "nccl")  # gloo: tests on a one-GPU box only
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", _local_device()))
        else:
            dist.init_process_group(backend)
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
