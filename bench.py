"""Benchmark of the hybrid fp64 triangle-pair contact kernel (BASELINE.json).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

``--gpus N`` without a torchrun environment relaunches itself as N ranks
(``torch.distributed.run``, one process per GPU, NCCL); under torchrun the
ranks come from RANK / LOCAL_RANK / WORLD_SIZE.

Headline workload (config 1 of BASELINE.json): 16,777,216 = 2^24 random
triangle pairs per GPU from the chunked cfg0 generator (seed 0, separation
U[-0.1, 0.5]), fp64, planar SoA layout [18][n] resident in HBM, hybrid kernel
at (16 sweeps, eps 1e-6), full result record written.  A step is one pass of
the hot path over the batch: stats reset, the hybrid kernel, and (N > 1) the
all-reduce of the stats record.  Rank r of N works on pairs [r*2^24,
(r+1)*2^24) of the same generator (weak scaling).  Inputs (2.4 GB) and
outputs (1.5 GB) exceed the 126 MB L2, so no flush is needed.

Every line also carries ``configs.cfg4_strong``: BASELINE.json config 4,
2^28 pairs IN TOTAL (separation U[-0.05, 0.2]) sharded over the N ranks by
contiguous ranges, reduce-only (tc_stats), with the all-reduce of the
counters and minimum distance -- strong scaling at every N.  Its inputs come
from the device Philox generator of the same distribution
(tc_random_pairs_soa_f64: host numpy would take minutes for 2^28 pairs).

``e2e`` times the same workload through the reference-facing C-ABI host
entry point tc_run_host_f64 with pinned host buffers in the reference's
(n,3,3) layout; ``e2e_dropin`` through the drop-in module itself
(``kernels.hybrid_batch`` on plain pageable numpy arrays, strict and fast):
H2D of the inputs, kernel and D2H of the full result record are inside the
timed region.

``--impl reference`` times the reference's CPU path -- the oracle port
(oracle/tc_oracle.c: the reference is pure numpy and cannot travel to the
GPU box) -- with every host thread, on the same cfg1 workload: each step is a
slice of the 2^24 pairs, the slices cycling through all of them.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

N_PAIRS = 1 << 24
PARAMS = dict(n_iterative=16, epsilon=1e-6)
SEP = (-0.1, 0.5)
CFG4_PAIRS = 1 << 28
CFG4_SEP = (-0.05, 0.2)
METRIC = "triangle-pair contact queries/sec (hybrid, fp64)"
UNIT = "pairs/s"


def flops_reference_model(n, n_it, fallback, intersecting):
    """200 + 88 N per pair, +1199 per fallback, +254 if it intersects."""
    return n * (200 + 88 * n_it) + 1199 * fallback + 254 * intersecting


def flops_executed(n, n_it, fallback, intersecting):
    """The algorithm this kernel executes: an intersecting fallback pair runs the
    six edge-plane tests (268) and the crossing resolution (254) but not the 15
    feature tests, whose results it does not use (931 of the 1199)."""
    return n * (200 + 88 * n_it) + 1199 * (fallback - intersecting) + (268 + 254) * intersecting


# ---------------------------------------------------------------------------
# clocks: nvidia-smi sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[4:8]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        maxclk = max(r[1] for r in rows)
        load = [r for r in rows if r[2] > 200.0] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in load for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in load), "sm_max_mhz": maxclk, "reasons": reasons,
                "samples": len(load), "power_w_max": max(r[2] for r in rows)}


# ---------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_rate(seconds: float, chunk: int, threads: int, start: int = 0):
    """Time the oracle port's hybrid on consecutive chunks until `seconds` pass."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle
    from paper_2105_12415_b200 import workloads as W
    p = oracle.make_params(**PARAMS)
    done, elapsed, k = 0, 0.0, 0
    while elapsed < seconds:
        A, B = W.random_pairs(chunk, seed=0, sep=SEP, start=start + k * chunk)
        t0 = time.perf_counter()
        _, _, rc = oracle.hybrid(A, B, p, PARAMS["epsilon"], threads=threads)
        elapsed += time.perf_counter() - t0
        assert rc == 0
        done += chunk
        k += 1
    return done / elapsed, done


def cfg1_config(n, world, strict):
    """The workload dict both arms print (GPU and reference)."""
    return {"workload": "cfg1: 2^24 random triangle pairs per GPU, hybrid fp64, 16 sweeps, eps 1e-6",
            "pairs_per_gpu": n, "layout": "SoA [18][n] in HBM", "rounding": "strict" if strict else "fast",
            "l2": "inputs 2.4 GB + outputs 1.5 GB per GPU > 126 MB L2 (no flush needed)",
            "parallelism": f"dp{world} contiguous shards + one all-gather of the stats record" if world > 1
            else "1 GPU"}


def run_reference(args, rank, world):
    """--impl reference: the CPU path on the host cores, rank 0 only.

    Same workload as the GPU arm (cfg1: the 2^24 pairs of the chunked
    generator, hybrid (16, 1e-6)); each timed step is a distinct slice of them,
    max(2^24 / K, 2^20) pairs, cycling through the whole set, so K steps cover
    at least 16M distinct pairs in a few seconds of CPU time."""
    if rank != 0:
        return
    threads = len(os.sched_getaffinity(0))
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle
    from paper_2105_12415_b200 import workloads as W
    oracle.build()
    n_all = args.pairs
    sample = min(n_all, max(-(-n_all // max(args.steps, 1)), 1 << 20))
    p = oracle.make_params(**PARAMS)
    A, B = W.random_pairs_mp(n_all, seed=0, sep=SEP)
    for k in range(args.warmup):
        oracle.hybrid(A[: 1 << 16], B[: 1 << 16], p, PARAMS["epsilon"], threads=threads)
    elapsed, done, off = 0.0, 0, 0
    for _ in range(args.steps):
        lo = off % n_all
        hi = min(lo + sample, n_all)
        a, b = A[lo:hi], B[lo:hi]
        t0 = time.perf_counter()
        _, _, rc = oracle.hybrid(a, b, p, PARAMS["epsilon"], threads=threads)
        elapsed += time.perf_counter() - t0
        assert rc == 0
        done += hi - lo
        off = hi
    value = done / elapsed
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded cfg0/cfg1 generator, SURVEY.md 8d)",
        "config": cfg1_config(n_all, world, False),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{done} pairs of the 2^24 cfg1 set in {args.steps} steps of {sample} distinct "
                                   f"pairs (slices cycling through the set), hybrid (16, 1e-6), oracle/tc_oracle.c "
                                   "(C restatement of RK/kernels.py, bit-identical to the reference) on every host "
                                   "thread; generation excluded",
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """--gpus N outside torchrun: relaunch this command as N ranks."""
    import socket
    if args.impl != "reference" and not args.share_gpu:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA devices"}), flush=True)
            return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pairs", type=int, default=N_PAIRS, help="pairs per GPU (cfg1)")
    ap.add_argument("--cfg4-n", type=int, default=CFG4_PAIRS, help="pairs in total (cfg4 strong scaling)")
    ap.add_argument("--strict", action="store_true", help="time the bit-exact TC_STRICT build")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / cpu baseline / variant table / configs")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the cfg4 strong-scaling run")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend (gloo: tests of the multi-rank path on one GPU)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="tests only: every rank on cuda:0 (functional check of the N-rank path, not a measurement)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if args.share_gpu else int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    from paper_2105_12415_b200 import _abi, device as D, shard, workloads as W

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    lib = _abi.load()
    n, start, sep = args.pairs, rank * args.pairs, SEP

    # ---- inputs: this rank's range of the chunked generator, SoA planes in HBM
    # (generated on all host cores in slices, uploaded slice by slice)
    planes = torch.empty((18, n), dtype=torch.float64, device=dev)
    A = np.empty((n, 3, 3))
    B = np.empty((n, 3, 3))
    slice_n = 1 << 23
    for lo in range(0, n, slice_n):
        hi = min(n, lo + slice_n)
        a, b = W.random_pairs_mp(hi - lo, seed=0, sep=sep, start=start + lo)
        planes[:, lo:hi] = torch.from_numpy(W.to_soa(a, b)).to(dev)
        A[lo:hi] = a
        B[lo:hi] = b
    ta, tb = planes[:9], planes[9:]
    out = D.alloc_outputs(n, torch.float64, dev, soa=True)
    stats = D.new_stats(dev)
    params = D.Params(**PARAMS)
    stream = torch.cuda.current_stream(dev)

    def step(ev=None):
        D.reset_stats(stats)
        if ev is not None:
            ev[0].record(stream)
        D.run("hybrid", ta, tb, params, soa=True, strict=args.strict, out=out, stats=stats, n=n)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:
            shard.allreduce_stats(stats)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    launches0 = D.launch_count()
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t_start.record(stream)
        for k in range(args.steps):
            step(kev[k])
        t_end.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = D.launch_count() - launches0
    ms_total = t_start.elapsed_time(t_end)
    ms_kernel = sum(a.elapsed_time(b) for a, b in kev) / args.steps
    ms_total, ms_kernel = max_over_ranks(torch, dist, world, dev, ms_total, ms_kernel)
    ms_step = ms_total / args.steps
    st = shard.stats_dict(stats)  # after the last step's all-reduce: whole-job tallies
    n_job = n * world
    value = n_job / (ms_step / 1e3)

    # ---- roofline of the dominant kernel (hybrid_kernel): FP64 pipe
    fb_local = st["fallback"] / world
    fbx_local = st["intersecting"] / world
    # achieved = the algorithmic work SURVEY.md 8(d) defines per pair (App. A),
    # x the pairs of one launch, / the launch's duration; the work this kernel
    # actually executes (intersecting fallbacks skip the feature tests) is
    # reported beside it
    flops = flops_reference_model(n, PARAMS["n_iterative"], fb_local, fbx_local)
    flops_exec = flops_executed(n, PARAMS["n_iterative"], fb_local, fbx_local)
    achieved_tf = flops / (ms_kernel / 1e3) / 1e12
    peak_tf = fma_peak(torch, lib, stream, dev, fp64=True)
    bytes_per_pair = 144 + 89  # SoA inputs + full result record
    hbm_gbs = n * bytes_per_pair / (ms_kernel / 1e3) / 1e9
    peaks = {}
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except (OSError, ValueError):
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    traffic = None
    traffic_note = None
    prof = ROOT / "profiles" / "ncu_hybrid_f64_summary.json"
    if prof.exists():
        try:
            pj = json.loads(prof.read_text())
            if pj.get("n") == n:
                traffic = pj.get("dram_bytes_per_launch")
                traffic_note = pj.get("source")
        except ValueError:
            pass
    roofline = {
        "bound": "fp64", "achieved": achieved_tf, "peak": peak_tf, "unit": "TFLOP/s", "frac": achieved_tf / peak_tf,
        "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram__bytes_read+write)",
        "traffic_source": traffic_note, "algorithmic_bytes_per_launch": n * bytes_per_pair,
        "kernel": ("hybrid_kernel<double,strict,soa>" if args.strict else
                   "hybrid_ws_kernel<double,fast,soa,12,1,full> (warp-specialised: 12 iterative + 4 fallback warps per SM)"),
        "kernel_ms": ms_kernel,
        "flops_per_launch": flops,
        "flop_model": "SURVEY.md 8(d)/App. A algorithmic work: n(200+88N) + 1199 fallback + 254 fallback&intersect "
                      "(N = 16 sweeps; fallback and intersect counts from this run's tc_stats)",
        "executed_model_tflops": flops_exec / (ms_kernel / 1e3) / 1e12,
        "executed_model": "n(200+88N) + 1199 (fallback - fallback&intersect) + 522 fallback&intersect "
                          "(intersecting fallbacks skip the 15 feature tests, whose results they do not use)",
        "peak_source": "in-run DFMA probe (tc_fma_probe); MEASURED_PEAKS.json has no FP64 figure",
        "hbm": {"achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": hbm_gbs / hbm_peak,
                "bytes_per_pair": bytes_per_pair, "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
    }
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded cfg0/cfg1 generator, SURVEY.md 8d)",
        "config": cfg1_config(n, world, args.strict),
        "roofline": roofline,
        "gpu_launches": launches,
        "stats": st,
        "fallback_rate": st["fallback"] / n_job,
    }
    line["clocks"] = clk.summary()
    if args.share_gpu:
        line["note"] = "--share-gpu: every rank on cuda:0 (functional test of the N-rank path, not a measurement)"
    configs = {}
    if not args.no_cfg4:
        configs["cfg4_strong"] = cfg4_strong(args, torch, dist, D, shard, lib, world, rank, dev, stream, peak_tf)

    if not args.no_extras:
        # ---- e2e through the host C-ABI entry point (pinned host buffers), every rank
        line["e2e"] = e2e_measure(lib, _abi, torch, A, B, n, world, dist, dev)
        if rank == 0 and world == 1:
            line["e2e_dropin"] = e2e_dropin(A, B)
            threads = len(os.sched_getaffinity(0))
            rate, done = cpu_oracle_rate(10.0, 1 << 17, threads)
            rate1, done1 = cpu_oracle_rate(3.0, 1 << 14, 1)
            line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                    "sample": f"{done} pairs of the cfg1 generator in 131072-pair chunks, hybrid "
                                              "(16, 1e-6), oracle/tc_oracle.c on all host threads; generation "
                                              "excluded",
                                    "one_core": {"value": rate1, "sample": f"{done1} pairs, 1 thread"},
                                    "cpu_model": cpu_model()}
            line["variants"] = variant_table(D, torch, ta, tb, n, dev)
            line["roofline_f32"] = roofline_f32(D, torch, lib, ta, tb, n, dev, stream)
            configs.update(configs_table(D, torch, dev))
    if configs:
        line["configs"] = configs
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def max_over_ranks(torch, dist, world, dev, *vals):
    t = torch.tensor(list(vals), dtype=torch.float64, device=dev)
    if world > 1:
        if dist.get_backend() == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX)
            t = h
    return [float(x) for x in t]


def fma_peak(torch, lib, stream, dev, fp64=True):
    """FP64 (DFMA) or FP32 (FFMA) pipe peak of this GPU, TFLOP/s (tc_fma_probe)."""
    sink = torch.empty(8192, dtype=torch.float64, device=dev)
    blocks = 148 * 8
    s = ctypes.c_void_p(stream.cuda_stream)
    iters = 2048 if fp64 else 4096
    lib.tc_fma_probe(1 if fp64 else 0, blocks, 64, ctypes.c_void_p(sink.data_ptr()), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(5):
        e0.record(stream)
        fl = lib.tc_fma_probe(1 if fp64 else 0, blocks, iters, ctypes.c_void_p(sink.data_ptr()), s)
        e1.record(stream)
        torch.cuda.synchronize()
        best = max(best, fl / (e0.elapsed_time(e1) / 1e3) / 1e12)
    return best


def cfg4_strong(args, torch, dist, D, shard, lib, world, rank, dev, stream, peak_tf, steps=5, warmup=2):
    """BASELINE.json config 4: 2^28 pairs in total, contiguous shards over the
    ranks, reduce-only hybrid + all-reduce of the stats record.  Inputs from
    the device Philox generator of the cfg0 distribution, sep U[-0.05, 0.2]."""
    n_total = args.cfg4_n
    start, n = shard.shard_range(n_total, rank, world)
    planes = torch.empty((18, max(n, 1)), dtype=torch.float64, device=dev)
    from paper_2105_12415_b200 import _abi
    _abi.check(lib.tc_random_pairs_soa_f64(4, start, n, CFG4_SEP[0], CFG4_SEP[1],
                                           ctypes.c_void_p(planes.data_ptr()), ctypes.c_void_p(stream.cuda_stream)),
               "tc_random_pairs_soa_f64")
    ta, tb = planes[:9], planes[9:]
    stats = D.new_stats(dev)
    params = D.Params(**PARAMS)

    def step(ev=None):
        D.reset_stats(stats)
        if ev is not None:
            ev[0].record(stream)
        D.run("hybrid", ta, tb, params, soa=True, strict=args.strict, out={}, stats=stats, n=n)
        if ev is not None:
            ev[1].record(stream)
        if world > 1:
            shard.allreduce_stats(stats)

    for _ in range(warmup):
        step()
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for k in range(steps):
        step(kev[k])
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    ms_kernel = sum(a.elapsed_time(b) for a, b in kev) / steps
    ms_total, ms_kernel, ms_kernel_min = max_over_ranks(torch, dist, world, dev, ms_total, ms_kernel, -ms_kernel)
    st = shard.stats_dict(stats)
    ms_step = ms_total / steps
    fl = flops_reference_model(n_total / world, PARAMS["n_iterative"], st["fallback"] / world,
                               st["intersecting"] / world)
    del planes
    torch.cuda.empty_cache()
    return {"pairs_total": n_total, "pairs_per_gpu": n_total // world, "n_gpus": world, "steps": steps,
            "warmup": warmup, "value": n_total / (ms_step / 1e3), "unit": UNIT, "ms_per_step": ms_step,
            "kernel_ms_max_rank": ms_kernel, "kernel_ms_min_rank": -ms_kernel_min, "scaling": "strong",
            "fp64_frac": fl / (ms_kernel / 1e3) / 1e12 / peak_tf,
            "fallback_rate": st["fallback"] / n_total, "stats": st,
            "workload": "cfg4: 2^28 random pairs in total (cfg0 distribution, sep U[-0.05,0.2], device Philox "
                        "generator seed 4), hybrid fp64 (16, 1e-6), reduce-only, contiguous shards + all-gather "
                        "of the stats record",
            "timing": "CUDA events on the launching stream, max over ranks"}


def e2e_dropin(A, B, reps=3):
    """End to end through the drop-in module: kernels.hybrid_batch on plain
    pageable numpy arrays (the reference's callers' usage, RK/stepping.py:299,
    RK/contact.py:131), strict (its default) and fast."""
    from paper_2105_12415_b200 import kernels as K
    n = A.shape[0]
    p = K.KernelParams(**PARAMS)
    res = {"n": n, "unit": UNIT, "h2d_bytes_per_step": n * 144, "d2h_bytes_per_step": n * 89,
           "path": "paper_2105_12415_b200.kernels.hybrid_batch(A, B, params, counters, eps) on pageable numpy "
                   "(n,3,3) arrays -> tc_run_host_f64: inputs staged through pinned buffers by the library's copy "
                   "threads, results written by DMA into the library's recycled pinned result block, 3-stream "
                   "pipeline",
           "host_note": "the inputs' host-memory copy (2.4 GB at the box's ~36 GB/s memcpy rate) bounds this path; "
                        "tools/hostbw.py measures the rate"}
    prev = K.rounding()
    try:
        for mode in ("strict", "fast"):
            K.set_rounding(mode)
            # warm-up at full size: the library's pinned result block is
            # allocated once here and recycled by the timed calls
            del_r = K.hybrid_batch(A, B, p, None, PARAMS["epsilon"])
            del del_r
            times = []
            for _ in range(reps):
                c = K.KernelCounters()
                t0 = time.perf_counter()
                r = K.hybrid_batch(A, B, p, c, PARAMS["epsilon"])
                times.append(time.perf_counter() - t0)
                del r
            sec = statistics.median(times)
            res[mode] = {"value": n / sec, "ms_per_step": 1e3 * sec, "fallback": c.fallback_invocations}
    finally:
        K.set_rounding(prev)
    return res


def e2e_measure(lib, _abi, torch, A, B, n, world, dist, dev, reps=3):
    """Hybrid through tc_run_host_f64 with pinned host buffers (reference layout)."""
    pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True)
    hA = pin((n, 3, 3), torch.float64)
    hB = pin((n, 3, 3), torch.float64)
    hA.numpy()[:] = A
    hB.numpy()[:] = B
    outs = {"distance": pin((n,), torch.float64), "point_a": pin((n, 3), torch.float64),
            "point_b": pin((n, 3), torch.float64), "bary_a": pin((n, 2), torch.float64),
            "bary_b": pin((n, 2), torch.float64), "kind": pin((n,), torch.int8)}
    from paper_2105_12415_b200 import device as D
    p = _abi.params_struct(D.Params(**PARAMS), 0)
    ptr = lambda t: ctypes.c_void_p(t.data_ptr())
    stats = _abi.TcStats(0, 0, 0, 0, 0, 0, float("inf"))

    def call():
        rc = lib.tc_run_host_f64(2, ptr(hA), ptr(hB), n, None, None, ctypes.byref(p), ptr(outs["distance"]),
                                 ptr(outs["point_a"]), ptr(outs["point_b"]), ptr(outs["bary_a"]),
                                 ptr(outs["bary_b"]), ptr(outs["kind"]), None, ctypes.byref(stats))
        _abi.check(rc, "tc_run_host_f64")

    call()
    times = []
    for _ in range(reps):
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        call()
        times.append(time.perf_counter() - t0)
    sec, = max_over_ranks(torch, dist, world, dev, statistics.median(times))
    link = pcie_probe(torch, dev)
    # the transfers are the floor: while both directions run each gets the
    # duplex rate, then the larger direction finishes alone at its own rate
    h, d = n * 144, n * 89
    both = min(h, d) / (link["duplex_gbs_per_direction"] * 1e9)
    rest = (h - d) / (link["h2d_gbs"] * 1e9) if h > d else (d - h) / (link["d2h_gbs"] * 1e9)
    floor = both + rest
    link["floor_ms"] = 1e3 * floor
    link["frac_of_floor"] = floor / sec
    link["note"] = "pinned copies on this box; floor = PCIe time of the step's H2D + D2H bytes"
    return {"value": n * world / sec, "unit": UNIT, "h2d_bytes_per_step": n * 144 * world,
            "d2h_bytes_per_step": n * 89 * world, "ms_per_step": 1e3 * sec,
            "path": "tc_run_host_f64 (host C ABI, pinned, 1M-pair chunks on 3 streams)", "link": link}


def pcie_probe(torch, dev, mb=512, reps=5):
    """Pinned host<->device copy bandwidth on this box (GB/s), each direction
    alone: the e2e path's transfer floor."""
    h = torch.empty(mb << 20, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(mb << 20, dtype=torch.uint8, device=dev)
    res = {}
    for name, dst, src in (("h2d_gbs", d, h), ("d2h_gbs", h, d)):
        dst.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        res[name] = reps * (mb << 20) / (e0.elapsed_time(e1) / 1e3) / 1e9
    # both directions at once (two streams): the duplex rate per direction
    h2, d2 = torch.empty_like(h).pin_memory(), torch.empty_like(d)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res["duplex_gbs_per_direction"] = reps * (mb << 20) / (time.perf_counter() - t0) / 1e9
    return res


def configs_table(D, torch, dev):
    """The other BASELINE.json configs on this GPU: cfg2 (all-pairs particle
    blocks, full 2,048-particle scene) and cfg3 (adversarial set, per class)."""
    from paper_2105_12415_b200 import _abi, particles as PT, workloads as W
    res = {}
    meshes, blocks, gaps = PT.cfg2_scene()
    tm = torch.from_numpy(meshes).to(dev)
    tb = torch.from_numpy(blocks).to(dev)
    P = D.Params(**PARAMS)
    n_pairs = int(blocks.shape[0]) * meshes.shape[1] ** 2
    for strict in (False, True):
        st = D.new_stats(dev)
        PT.blocks_hybrid(tm, tb, P, strict=strict, stats=st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        D.reset_stats(st)
        e0.record()
        out = PT.blocks_hybrid(tm, tb, P, strict=strict, stats=st)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        s = D.read_stats(st)
        res[f"cfg2_{'strict' if strict else 'fast'}"] = {
            "pairs": n_pairs, "blocks": int(blocks.shape[0]), "ms": ms, "pairs_per_s": n_pairs / (ms / 1e3),
            "fallback_rate": s["fallback"] / n_pairs, "contacts": int(out["n_contacts"].item()),
            "min_distance": s["min_distance"]}
    # cfg3: 2^20 pairs per class, hybrid (16, 1e-6)
    A, B = W.adversarial_pairs(1 << 20, seed=3)
    c3 = {}
    for c, name in enumerate(W.CFG3_CLASSES):
        sl = slice(c << 20, (c + 1) << 20)
        planes = torch.from_numpy(W.to_soa(A[sl], B[sl])).to(dev)
        st = D.new_stats(dev)
        # steady state of the class: the library picks the hybrid's kernel instance from what
        # the previous launches on the device measured (tc_debug_fallback_rate_high)
        out = D.alloc_outputs(1 << 20, planes.dtype, dev, soa=True)
        for _ in range(3):
            D.run("hybrid", planes[:9], planes[9:], P, soa=True, out=out, n=1 << 20)
            torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10  # back to back, so the ~0.2 ms kernels hide the launch calls
        e0.record()
        for _ in range(reps):
            D.run("hybrid", planes[:9], planes[9:], P, soa=True, out=out, stats=st, n=1 << 20)
        e1.record()
        torch.cuda.synchronize()
        s = D.read_stats(st)
        c3[name] = {"pairs": 1 << 20, "pairs_per_s": reps * (1 << 20) / (e0.elapsed_time(e1) / 1e3),
                    "fallback_rate": s["fallback"] / reps / (1 << 20), "degenerate": s["degenerate"] // reps,
                    "contacts": s["contacts"] // reps,
                    "self_serving_instance": bool(_abi.load().tc_debug_fallback_rate_high())}
    res["cfg3_fast"] = c3
    res["multiscale"] = multiscale_table(D, torch, dev)
    res["note"] = ("oracle agreement of cfg2/cfg3: tests/test_gpu_blocks.py, tests/test_gpu_cfg3.py "
                   "(strict bitwise, fast within tolerance with the tie classifier); at full size "
                   "profiles/r01_parity_full.txt (all 4 x 2^20 cfg3 pairs: strict bitwise, fast within "
                   "tolerance, fp64 and fp32) and profiles/r01_parity_cfg2.txt (all 576.7M cfg2 pairs)")
    return res


def multiscale_scene(n_pairs=1024, seed=5):
    """Particle pairs for the device multiscale traversal: the reference's own
    320-triangle two-sphere scenes and surrogate trees (tests/golden/ms_float64.npz,
    produced by the reference), each pair re-posed by a random rigid motion."""
    from paper_2105_12415_b200 import multiscale as MS
    from paper_2105_12415_b200.workloads import rotation_matrices
    g = np.load(ROOT / "tests" / "golden" / "ms_float64.npz")
    names = [str(s) for s in g["scenes"] if str(s).startswith("s320")]
    rng = np.random.default_rng(seed)
    trees = []
    for k in range(n_pairs):
        sc = names[k % len(names)]
        q = rng.normal(size=4)
        R = rotation_matrices(q[None] / np.linalg.norm(q))[0]
        shift = rng.uniform(-50, 50, 3)
        for side in ("i", "j"):
            x = g[f"{sc}_{side}_tris"].reshape(-1, 3) @ R.T + shift
            trees.append(MS.FlatTreeArrays(x.reshape(-1, 3, 3), g[f"{sc}_{side}_eps"], g[f"{sc}_{side}_child_off"],
                                           g[f"{sc}_{side}_child_ids"], g[f"{sc}_{side}_height"],
                                           int(g[f"{sc}_{side}_n_nodes"])))
    return trees, np.arange(2 * n_pairs).reshape(-1, 2)


def multiscale_table(D, torch, dev, n_pairs=1024):
    """Device multiscale traversal (8f row 3) vs flat all-pairs detection of the
    same particle pairs (the blocks kernel on their mesh triangles), reference params."""
    from paper_2105_12415_b200 import kernels as K, multiscale as MS, particles as PT
    trees, pairs = multiscale_scene(n_pairs)
    forest = MS.build_forest(trees, device=dev)
    kp = K.KernelParams()
    res = {"particle_pairs": n_pairs}
    for strict in (False, True):
        MS.multiscale_contacts(forest, pairs, kp, strict=strict)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = MS.multiscale_contacts(forest, pairs, kp, strict=strict)
        dt = time.perf_counter() - t0
        res[f"multiscale_{'strict' if strict else 'fast'}"] = {
            "ms": dt * 1e3, "call_ms": r.call_ms, "particle_pairs_per_s": n_pairs / dt,
            "checks": int(r.checks.sum()), "checks_per_s_in_call": int(r.checks.sum()) / (r.call_ms / 1e3),
            "checks_by_height": r.checks.tolist(), "contacts": r.n_contacts, "fallback": r.stats["fallback"]}
    # flat detection of the same pairs: every mesh triangle pair through the blocks kernel
    meshes = np.stack([t.tris[t.n_nodes:] for t in trees])
    tm = torch.from_numpy(np.ascontiguousarray(meshes)).to(dev)
    tb = torch.from_numpy(pairs.astype(np.int32)).to(dev)
    P = D.Params(epsilon=kp.epsilon, n_iterative=kp.n_iterative)
    PT.blocks_hybrid(tm, tb, P)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = PT.blocks_hybrid(tm, tb, P)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    res["flat_fast"] = {"ms": dt * 1e3, "particle_pairs_per_s": n_pairs / dt,
                        "checks": n_pairs * meshes.shape[1] ** 2, "contacts": int(out["n_contacts"].item())}
    # the CPU oracle port of the reference's per-pair traversal, one thread, 16 pairs
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle
    import ms_oracle
    sample = [dict(tris=t.tris, eps=t.eps, child_off=t.child_off, child_ids=t.child_ids, height=t.height,
                   n_nodes=t.n_nodes) for t in trees[:32]]
    t0 = time.perf_counter()
    ms_oracle.multiscale(sample, np.arange(32).reshape(-1, 2), oracle.make_params())
    res["cpu_oracle"] = {"particle_pairs_per_s": 16 / (time.perf_counter() - t0), "cores": 1,
                         "sample": "16 particle pairs, oracle/ms_oracle.py over the C oracle"}
    res["note"] = ("wall-clock per call (synchronous host-driven rounds); contacts of multiscale and flat agree "
                   "(the reference's equivalence lemma)")
    return res


def variant_table(D, torch, ta, tb, n, dev, reps=3):
    """Kernel-only rates of every variant x dtype x rounding on the cfg1 batch
    (2^24 pairs, SoA in HBM, full record)."""
    res = {}
    P = D.Params(**PARAMS)
    for dt, name in ((torch.float64, "f64"), (torch.float32, "f32")):
        a, b = ta.to(dt), tb.to(dt)
        out = D.alloc_outputs(n, dt, dev, soa=True)
        for variant in ("iterative", "comparison", "hybrid"):
            for strict in (False, True):
                D.run(variant, a, b, P, soa=True, strict=strict, out=out, n=n)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    D.run(variant, a, b, P, soa=True, strict=strict, out=out, n=n)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                res[f"{variant}_{name}_{'strict' if strict else 'fast'}"] = round(n / (ms / 1e3), 1)
        del a, b, out
    res["unit"] = f"pairs/s, {n} pairs (cfg1), SoA, full record, (16, 1e-6)"
    return res


def roofline_f32(D, torch, lib, ta, tb, n, dev, stream, reps=5):
    """FP32 roofline of hybrid_kernel<float,fast,soa> on the cfg1 batch cast to
    fp32: SURVEY.md 8(d)'s algorithmic flops (this run's fallback counts) per
    launch over the launch time, against the in-run FFMA peak."""
    a, b = ta.to(torch.float32), tb.to(torch.float32)
    out = D.alloc_outputs(n, torch.float32, dev, soa=True)
    st = D.new_stats(dev)
    P = D.Params(**PARAMS)
    D.run("hybrid", a, b, P, soa=True, out=out, n=n)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for e0, e1 in ev:
        D.reset_stats(st)
        e0.record(stream)
        D.run("hybrid", a, b, P, soa=True, out=out, stats=st, n=n)
        e1.record(stream)
    torch.cuda.synchronize()
    ms = sorted(e0.elapsed_time(e1) for e0, e1 in ev)[reps // 2]
    s = D.read_stats(st)
    flops = flops_reference_model(n, PARAMS["n_iterative"], s["fallback"], s["intersecting"])
    peak = fma_peak(torch, lib, stream, dev, fp64=False)
    achieved = flops / (ms / 1e3) / 1e12
    return {"bound": "fp32", "kernel": "hybrid_ws_kernel<float,fast,soa,16,2,full> (warp-specialised: 16 iterative + 8 fallback warps per SM)", "achieved": achieved, "peak": peak,
            "unit": "TFLOP/s", "frac": achieved / peak, "kernel_ms": ms, "pairs_per_s": n / (ms / 1e3),
            "fallback_rate": s["fallback"] / n, "flops_per_launch": flops,
            "flop_model": "SURVEY.md 8(d)/App. A, as roofline", "peak_source": "in-run FFMA probe (tc_fma_probe)",
            "hbm": {"achieved": n * (72 + 45) / (ms / 1e3) / 1e9, "unit": "GB/s", "bytes_per_pair": 72 + 45}}


if __name__ == "__main__":
    main()
