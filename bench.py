"""Benchmark: B200-native tile-recursive PLUQ over GF(p) (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload pluq|lru|fgemm] [--n 16384] [--p 131071] [--thr 64]

Workload (N=1, default): BASELINE config 3 -- PLUQ of a dense 16384 x 16384
i.i.d. matrix over GF(131071) (random_mat, test_util.hpp:22-28, seeded), the
largest single-GPU PLUQ configuration of the metric "PLUQ effective field
Gop/s (2n^3/3 / time)".  One step = one pluq_tile_recursive of one resident
matrix (a fresh seeded matrix per step, all generated in HBM before the timed
region; 1 GiB each, larger than L2, so no flush is needed).  The fgemm part
of the metric (config 2, 8192^3 C <- C - A*B) is reported in the same line
under "fgemm".  --workload lru = config 4, --p 251 --n 32768 = config 5.

--gpus N > 1: when not already under torchrun, bench.py re-launches itself with
`python -m torch.distributed.run --nproc-per-node N` (one process per GPU, NCCL).
The PLUQ workloads then run PARTITIONED -- all ranks factor the same matrix, each
computing its slice of every large Schur GEMM/TRSM, exchanged with NCCL
all-gathers (csrc/dist.cu); value = one matrix's work /
max-over-ranks device time; scaling "strong".  fgemm runs as independent
replicas (value = all ranks' work, "weak").

Roofline: the tcgen05 GEMM kernels' in-situ durations from CUPTI (torch.profiler)
over one extra, untimed step -- no events inside the step -- and their
algorithmic int8 work counted by the library (ffg_profile_enable(ctx, 2)),
against peak = 2 x the driver-measured dense bf16 burst (MEASURED_PEAKS.json;
B200 dense int8 = 2 x bf16), with cuBLASLt's int8 measured beside it.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
reference headers compiled unchanged + the rankrev.hpp:146 fix) on this box's
host cores, on the SAME configuration (one full-size timed run -- the CPU takes
~45 s for n = 16384 on 16 cores; the reported "steps" is 1); rank 0 only.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="pluq", choices=["pluq", "lru", "fgemm"])
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--p", type=int, default=None)
    ap.add_argument("--thr", type=int, default=64)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-fgemm", action="store_true")
    ap.add_argument("--no-prof", action="store_true", help="skip the extra CUPTI-profiled step (roofline)")
    ap.add_argument("--no-clocks", action="store_true",
                    help="no nvidia-smi clock sampling (for runs under ncu: the polling slows its replays)")
    # under the self-relaunch (--gpus N outside torchrun) the arguments travel in the environment:
    # torchrun's own parser would otherwise claim abbreviations such as --n
    argv = json.loads(os.environ["FFG_BENCH_ARGV"]) if "FFG_BENCH_ARGV" in os.environ else None
    a = ap.parse_args(argv)
    a.warmup = max(a.warmup, 3) if a.impl == "ours" else a.warmup
    if a.n is None:
        a.n = 8192 if a.workload == "fgemm" else 16384
    if a.p is None:
        a.p = 131071
    return a


def config_no(a):
    if a.workload == "fgemm":
        return "2"
    if a.workload == "lru":
        return "4"
    return "5" if a.p <= 256 else ("1" if a.n <= 1024 else "3")


def workload_config(a, world):
    if a.workload == "fgemm":
        return {"workload": f"fgemm C <- C - A*B mod {a.p}, M=N=K={a.n} (BASELINE config 2)", "n": a.n, "p": a.p,
                "parallelism": f"replicas x{world}", "l2": "inputs > L2 (768 MiB limb planes + 768 MiB operands)"}
    kind = "i.i.d. random_mat" if a.workload == "pluq" else f"L*R*U rank {a.n // 2}"
    return {"workload": f"pluq_tile_recursive n={a.n} {kind} over GF({a.p}), threshold {a.thr} "
                        f"(BASELINE config {config_no(a)})",
            "n": a.n, "p": a.p, "threshold": a.thr,
            "parallelism": "single GPU" if world == 1 else
            f"partitioned x{world}: one matrix, replicated panel, Schur GEMM/TRSM output slices + NCCL all-gather",
            "l2": "inputs larger than L2 (a fresh matrix per step)"}


def metric_ops(a):
    n = a.n
    return 2.0 * n ** 3 if a.workload == "fgemm" else 2.0 * n ** 3 / 3.0


METRIC = "PLUQ effective field Gop/s (2n^3/3 / time) mod p"
METRIC_FGEMM = "fgemm effective field Gop/s (2mnk / time) mod p"


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region.

    nvidia-smi is started BEFORE the warm-up (start()): its start-up initialises NVML, which holds
    driver locks for a few hundred ms and, when it fell inside the timed region, stalled the
    factorisation's own launches (config 5, whose host is on the critical path, read 90-160 ms
    instead of 72 in one run out of four).  The `with` block only marks the timed window; the
    summary uses the samples whose timestamps fall inside it."""

    FMT = "%Y/%m/%d %H:%M:%S.%f"

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def start(self, period_ms: int = 25, wait_first: float = 3.0):
        q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", str(int(period_ms)), "-i", str(self.idx)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t_end = time.time() + wait_first  # its first line = NVML is up: nothing of that start-up is left
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.005)
        except FileNotFoundError:
            self.proc = None
        return self

    def __enter__(self):
        self.t0 = time.time()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.t1 = time.time()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)
            self.proc = None

    def summary(self):
        self.stop()
        import datetime
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        rows = []
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], self.FMT).timestamp()
                rows.append((ts, float(f[1]), float(f[2]), f[5:9]))
            except ValueError:
                continue
        inside = [r for r in rows if self.t0 is not None and self.t0 - 0.03 <= r[0] <= (self.t1 or self.t0) + 0.03]
        if not inside and rows and self.t0 is not None:  # a window shorter than the sampling period
            inside = [min(rows, key=lambda r: abs(r[0] - 0.5 * (self.t0 + (self.t1 or self.t0))))]
        sm = [r[1] for r in inside]
        mx = max([r[2] for r in inside], default=0.0)
        reasons = set()
        for r in inside:
            for nm, v in zip(names, r[3]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- peaks
def tensor_peak(torch):
    """Peak for the roofline: 2 x the driver-measured dense bf16 burst of MEASURED_PEAKS.json (B200
    dense int8 = 2 x dense bf16), with cuBLASLt's int8 (torch._int_mm 8192^3) measured here beside it."""
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    if "bf16_tflops" in peaks:
        bf16, src = peaks["bf16_tflops"], "2 x bf16_tflops (burst) of MEASURED_PEAKS.json"
    else:
        bf16, src = 1590.0, "2 x 1.59 PFLOP/s bf16 (B200_PROFILING.md fallback; MEASURED_PEAKS.json absent)"
    best = None
    try:
        n = 8192
        a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
        b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        best = 2.0 * n ** 3 / (min(ts) / 1e3) / 1e12
        del a, b
    except Exception:
        best = None
    return {"int8_tops": 2.0 * bf16, "source": src, "cublaslt_int8_tops_measured": best,
            "bf16_tflops_measured": bf16}


# ---------------------------------------------------------------------- CPU reference
def run_reference_sample(n, p, thr, workers, seed=1, gen="iid", timeout=1500, retries=2):
    cmd = [sys.executable, os.path.join(ROOT, "scripts", "ref_runner.py"), "--n", str(n), "--p", str(p),
           "--thr", str(thr), "--workers", str(workers), "--seed", str(seed), "--gen", gen]
    last = None
    for _ in range(retries):  # the reference TaskPool can hang or crash at workers > 1
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout)
            if r.returncode == 0 and r.stdout.strip():
                return json.loads(r.stdout.strip().splitlines()[-1])
            last = r.stderr[-300:]
        except subprocess.TimeoutExpired:
            last = "timeout"
    raise RuntimeError(f"reference run failed: {last}")


def run_fgemm_reference(n, p, workers):
    code = ("import sys,json;sys.path.insert(0,%r);from oracle import oracle as O;"
            "A=O.random_mat(%d,%d,%d,11);B=O.random_mat(%d,%d,%d,12);C=O.random_mat(%d,%d,%d,13);"
            "import ctypes as c,numpy as np;r=O.Ref(True);s=c.c_double(0);Cc=C.copy();"
            "rc=r.L.ref_pfgemm_timed(%d,%d,A,B,1,Cc,%d,%d,%d,%d,c.byref(s));"
            "print(json.dumps({'seconds':s.value,'kind':'reference'}))") % (
        ROOT, p, n, n, p, n, n, p, n, n, p, p - 1, n, n, n, workers)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=1500)
    return json.loads(r.stdout.strip().splitlines()[-1])


# The reference is timed at the configured size when that is at most this (config 3 / 4 / 2: about
# 45 s / 90 s / 20 s on 16 cores); config 5 (n = 32768, several minutes) is sampled at n = 16384.
REF_FULL_MAX_N = 16384


def reference_size(a):
    return a.n if a.n <= REF_FULL_MAX_N else REF_FULL_MAX_N


def time_reference(a, workers, seed=1):
    """One reference run on this host: (seconds, ops, sample description, kind)."""
    n = reference_size(a)
    gen = "lru" if a.workload == "lru" else "iid"
    if a.workload == "fgemm":
        res = run_fgemm_reference(n, a.p, workers)
        ops = 2.0 * n ** 3
        sample = f"pfgemm C <- C - A*B mod {a.p}, {n}^3, workers={workers}"
    else:
        res = run_reference_sample(n, a.p, a.thr, workers, seed=seed, gen=gen)
        ops = 2.0 * n ** 3 / 3.0
        sample = f"pluq_tile_recursive n={n} {gen} GF({a.p}) thr={a.thr}, workers={workers}"
    if n == a.n:
        sample += " -- the full configured size, one run"
    else:
        sample += f" -- bounded sample of n={a.n} (the full size takes several minutes on the CPU)"
    return res["seconds"], ops, sample, res.get("kind", "reference"), n


def reference_arm(a, rank, world):
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    if a.warmup > 0:  # page in the library and start the thread pool on a small case (untimed)
        run_reference_sample(512, a.p, a.thr, workers, seed=99, gen="iid")
    secs, ops, sample, kind, n = time_reference(a, workers, seed=1)
    val = ops / secs / 1e9
    line = {"impl": "reference", "metric": METRIC_FGEMM if a.workload == "fgemm" else METRIC, "value": val,
            "unit": "Gop/s", "n_gpus": world, "steps": 1, "steps_requested": a.steps, "warmup": a.warmup,
            "ms_per_step": secs * 1e3, "higher_is_better": True,
            "scaling": "weak" if a.workload == "fgemm" else "strong", "vs_baseline": None,
            "dtype": "u32 residues (i64 accum)", "data": "synthetic (seeded SplitMix64, test_util.hpp random_mat)",
            "config": workload_config(a, world), "same_size_as_config": n == a.n,
            "cpu_baseline": {"value": val, "unit": "Gop/s", "cores": workers if kind == "reference" else 1,
                             "kind": kind, "sample": sample},
            "e2e": {"value": val, "unit": "Gop/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "one full-size CPU factorisation is the step (a K-step loop at this size would take "
                    "K x ~45 s); warmup = small untimed runs"}
    print(json.dumps(line), flush=True)


def cpu_baseline(a):
    workers = os.cpu_count() or 1
    secs, ops, sample, kind, n = time_reference(a, workers, seed=1)
    return {"value": ops / secs / 1e9, "unit": "Gop/s", "cores": workers if kind == "reference" else 1,
            "kind": kind, "sample": sample, "seconds": secs, "n": n, "same_size_as_config": n == a.n}


# ---------------------------------------------------------------------- in-situ kernel timeline
def cupti_step(torch, fn, stream):
    """Run fn() once under torch.profiler (CUPTI activity tracing: device timestamps of every kernel of
    the process, any stream, no events inserted) -> (event ms of the step, [(start_us, end_us, name)])."""
    import re
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
    ks = []
    for e in prof.events():
        if e.device_type.name != "CUDA" or e.device_time_total <= 0:
            continue
        nm = re.sub(r"^void ", "", re.sub(r"\(.*", "", e.name))
        if nm.startswith("Memcpy") or nm.startswith("Memset"):
            continue
        ks.append((e.time_range.start, e.time_range.end, nm))
    ks.sort()
    return e0.elapsed_time(e1), ks


def union_ms(spans):
    busy, last = 0.0, None
    for s, t in sorted(spans):
        if last is None or s >= last:
            busy += t - s
            last = t
        elif t > last:
            busy += t - last
            last = t
    return busy / 1e3


def is_tc_gemm(name):
    return name.startswith("ffg::modgemm") and "simt" not in name or (
        name.startswith("modgemm") and "simt" not in name)


# ---------------------------------------------------------------------- our arm
def our_arm(a, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1402_3501_b200 as G

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = G.Context(local_rank, stream=stream.cuda_stream)
    n, p = a.n, a.p
    is_fgemm = a.workload == "fgemm"

    def make(seed):
        d = torch.empty((n, n), dtype=torch.int32, device=dev)
        if a.workload == "lru":
            G.lru_matrix_dev(p, d, n // 2, seed, ctx=ctx)
        else:
            G.random_mat_dev(p, d, seed, ctx=ctx)
        return d

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def run_once(mats, i):
        if is_fgemm:
            A, B, C_ = mats
            G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx)
        else:
            G.pluq_tile_recursive(p, mats[i], a.thr, ctx=ctx)

    # ---- inputs resident in HBM
    # partitioned PLUQ: every rank holds the same matrix (same seeds) and owns slices of the
    # large Schur operations; fgemm runs as independent replicas
    partitioned = world > 1 and not is_fgemm
    if partitioned:
        G.dist.init_from_process_group(ctx)
    seed0 = 1 if partitioned or world == 1 else 1000 * rank + 1
    # one fresh matrix per step; n = 32768 (4 GiB each) keeps two and regenerates between steps
    # outside the timed region would break the K-step loop, so config 5 holds all of them (4 GiB x
    # (W + K) of the 180 GB)
    if is_fgemm:
        mats = [make(11), make(12), make(13)]
    else:
        mats = [make(seed0 + i) for i in range(a.warmup + a.steps)]
    ctx.synchronize()

    # ---- warmup (untimed); the clock sampler starts after the first warm-up step -- which tells the
    # step time, hence a polling period of about five samples per timed region -- and its start-up
    # (NVML initialisation) is waited for here, before the remaining warm-up steps
    sampler = ClockSampler(local_rank)
    probe = min(1, a.warmup - 1)  # the second warm-up step is already warm
    for i in range(a.warmup):
        if i == probe:
            ctx.synchronize()
        t_w = time.time()
        run_once(mats, i)
        if i == probe and not a.no_clocks:
            ctx.synchronize()
            step_ms = (time.time() - t_w) * 1e3
            sampler.start(period_ms=int(min(500, max(25, step_ms * a.steps / 5))))
    if a.warmup == 0 and not a.no_clocks:
        sampler.start()
    ctx.synchronize()

    # ---- timed region: exactly K steps
    launches0 = ctx.launches
    spec0 = ctx.spec_stats()
    with sampler as clk:
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(a.steps):
            run_once(mats, a.warmup + i)
        e1.record(stream)
        barrier()
    launches = ctx.launches - launches0
    spec1 = ctx.spec_stats()
    speculation = {k: spec1[k] - spec0[k] for k in spec1}  # full-rank guesses inside the timed region
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ops_step = metric_ops(a)
    value = (1 if partitioned else world) * a.steps * ops_step / (ms_max / 1e3) / 1e9
    clocks = clk.summary()
    del mats
    torch.cuda.empty_cache()

    # ---- in-situ kernel timeline of ONE extra, untimed step (CUPTI) + the library's work count
    insitu = None
    if not a.no_prof:
        pm = [make(11), make(12), make(13)] if is_fgemm else [make(seed0 + 999)]
        ctx.synchronize()
        ctx.profile(2)  # count launches and algorithmic work only: no events in the step
        step_ms, ks = cupti_step(torch, lambda: run_once(pm, 0), stream)
        ctx.profile(0)
        prof = ctx.profile_read()
        del pm
        torch.cuda.empty_cache()
        insitu = {"step_ms": step_ms, "kernels": ks, "prof": prof}

    # ---- e2e through the public host API (pinned host buffers, copies inside the timed region)
    e2e = None
    if not a.no_e2e:
        e2e = e2e_host(a, G, ctx, torch, np, dev, stream, 0 if partitioned else rank, world, partitioned)

    # ---- secondary: fgemm config 2 alongside the PLUQ line
    fg = None
    if not is_fgemm and not a.no_fgemm:
        fg = fgemm_secondary(a, G, ctx, torch, dev, stream)

    if rank != 0:
        return
    roof = roofline(a, torch, insitu, ms_max / a.steps) if insitu else None
    cpu = None
    if not a.no_cpu:
        try:
            cpu = cpu_baseline(a)
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "Gop/s", "error": str(ex)[:200]}
    line = {"metric": METRIC_FGEMM if is_fgemm else METRIC, "value": value, "unit": "Gop/s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True,
            "scaling": "weak" if is_fgemm else "strong", "vs_baseline": None,
            "dtype": "u32 residues (u8 limbs on tcgen05, s32 accum)",
            "data": "synthetic (seeded SplitMix64 random_mat / L*R*U, generated in HBM)",
            "config": workload_config(a, world), "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
            "roofline": roof, "cpu_baseline": cpu}
    if not is_fgemm:
        line["speculation"] = speculation
    if fg:
        line["fgemm"] = fg
    print(json.dumps(line), flush=True)


def roofline(a, torch, insitu, ms_step):
    ks, prof, step_ms = insitu["kernels"], insitu["prof"], insitu["step_ms"]
    peak = tensor_peak(torch)
    gem = [(s, t) for s, t, nm in ks if is_tc_gemm(nm)]
    gemm_ms = sum(t - s for s, t in gem) / 1e3
    work = prof["gemm"]["work"]
    achieved = work / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    by = {}
    for s, t, nm in ks:
        k = nm.replace("ffg::", "")
        k = k[:k.index("<")] if "<" in k else k
        c = by.setdefault(k, [0, 0.0])
        c[0] += 1
        c[1] += (t - s) / 1e3
    span = (ks[-1][1] - ks[0][0]) / 1e3 if ks else 0.0
    # DRAM bytes per tcgen05 GEMM launch from one ncu capture of this same workload
    # (scripts/round_end.sh -> profiles/pluq_gemm_traffic.json); null when none matches
    traffic, tfile = None, os.path.join(ROOT, "profiles", "pluq_gemm_traffic.json")
    if a.workload != "fgemm" and os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            if tj.get("n") == a.n and tj.get("p") == a.p and tj.get("threshold") == a.thr:
                traffic = tj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    return {"bound": "tensor", "kernel": "modgemm_kernel<L> / modgemm_direct_kernel<L,KB> (tcgen05 kind::i8)",
            "achieved": achieved, "peak": peak["int8_tops"], "unit": "TOPS (int8 tensor ops)",
            "frac": achieved / peak["int8_tops"], "traffic": traffic, "peak_source": peak["source"],
            "cublaslt_int8_tops_measured": peak["cublaslt_int8_tops_measured"],
            "work_per_unit": "2*L^2 int8 ops per field MAC (L = 8-bit limbs per residue)",
            "work_per_step_int8_ops": work, "gemm_launches_per_step": int(prof["gemm"]["launches"]),
            "timing": "CUPTI in-situ kernel durations (torch.profiler) over one extra untimed step; "
                      "work counted by the library (no events in the step)",
            "gemm_kernel_ms_per_step": gemm_ms, "gemm_busy_ms_per_step": union_ms(gem),
            "profiled_step_ms": step_ms, "timed_ms_per_step": ms_step,
            "whole_step_frac": work / (ms_step / 1e3) / 1e12 / peak["int8_tops"],
            "kernel_span_ms": span, "gpu_busy_ms": union_ms([(s, t) for s, t, _ in ks]),
            "kernels_ms": {k: round(v[1], 3) for k, v in sorted(by.items(), key=lambda x: -x[1][1])[:12]},
            "kernels_launches": {k: v[0] for k, v in sorted(by.items(), key=lambda x: -x[1][1])[:12]}}


def e2e_host(a, G, ctx, torch, np, dev, stream, rank, world, partitioned=False):
    """Same metric through the host API: pinned host matrix -> ffg_* host entry point -> host result."""
    import torch.distributed as dist
    n, p = a.n, a.p
    ctx.set_stream(stream.cuda_stream)
    if a.workload == "fgemm":
        A = torch.empty((n, n), dtype=torch.int32).pin_memory()
        B = torch.empty((n, n), dtype=torch.int32).pin_memory()
        C0 = torch.empty((n, n), dtype=torch.int32).pin_memory()
        C = torch.empty((n, n), dtype=torch.int32).pin_memory()
        d = torch.empty((n, n), dtype=torch.int32, device=dev)
        for h, s in ((A, 11), (B, 12), (C0, 13)):
            G.random_mat_dev(p, d, s, ctx=ctx)
            ctx.synchronize()
            h.copy_(d.cpu())
        del d
        An, Bn, Cn = (x.numpy().view(np.uint32) for x in (A, B, C))
        h2d = 3 * n * n * 4
        d2h = n * n * 4

        def step():
            C.copy_(C0)
            return lambda: G.fgemm(p, p - 1, An, Bn, 1, Cn, ctx=ctx)
    else:
        # small fields (config 5, p <= 256) are stored as bytes: ffg_pluq_tile_recursive_u8
        byte = p <= 256
        hdt = torch.uint8 if byte else torch.int32
        H0 = torch.empty((n, n), dtype=hdt).pin_memory()
        H = torch.empty((n, n), dtype=hdt).pin_memory()
        d = torch.empty((n, n), dtype=torch.int32, device=dev)
        if a.workload == "lru":
            G.lru_matrix_dev(p, d, n // 2, 7 + rank, ctx=ctx)
        else:
            G.random_mat_dev(p, d, 7 + rank, ctx=ctx)
        ctx.synchronize()
        H0.copy_(d.to(torch.uint8).cpu() if byte else d.cpu())
        del d
        Hn = H.numpy() if byte else H.numpy().view(np.uint32)
        es = 1 if byte else 4
        h2d = n * n * es
        d2h = n * n * es + 2 * n * 4  # packed factors + P and Q

        def step():
            H.copy_(H0)  # restore the in/out host buffer (untimed)
            return lambda: G.pluq_tile_recursive(p, Hn, a.thr, ctx=ctx)
    torch.cuda.empty_cache()
    step()()  # warm
    ctx.synchronize()
    times = []
    k = max(1, min(a.steps, 5))
    for _ in range(k):
        f = step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    # the median of the k steps: the host side of this path (pinned-memory DMA, the streaming host
    # thread) shares the box with other tenants, and a single disturbed step moved a 3-step mean by 30 %
    t = torch.tensor([statistics.median(times)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    return {"value": (1 if partitioned else world) * metric_ops(a) / (ms / 1e3) / 1e9, "unit": "Gop/s",
            "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms, "steps": k, "stat": "median of the steps",
            "ms_steps": [round(x, 3) for x in times],
            "api": "ffg_fgemm (host buffers)" if a.workload == "fgemm" else
                   ("ffg_pluq_tile_recursive_u8 (host byte buffers)" if a.p <= 256
                    else "ffg_pluq_tile_recursive (host buffers)"),
            "host_memory": "pinned"}


def fgemm_secondary(a, G, ctx, torch, dev, stream):
    n, p = 8192, 131071
    mats = []
    for s in (11, 12, 13):
        d = torch.empty((n, n), dtype=torch.int32, device=dev)
        G.random_mat_dev(p, d, s, ctx=ctx)
        mats.append(d)
    A, B, C_ = mats
    for _ in range(3):
        G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx)
    ctx.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record(stream)
    for _ in range(reps):
        G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ctx.profile(2)
    _, ks = cupti_step(torch, lambda: G.fgemm(p, p - 1, A, B, 1, C_, ctx=ctx), stream)
    ctx.profile(0)
    prof = ctx.profile_read()
    del mats, A, B, C_
    torch.cuda.empty_cache()
    gem_ms = sum(t - s for s, t, nm in ks if is_tc_gemm(nm)) / 1e3
    split_ms = sum(t - s for s, t, nm in ks if "split" in nm) / 1e3
    traffic = algo = None  # ncu DRAM bytes of this launch (profiles/gemm_traffic.json)
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "gemm_traffic.json")))
        traffic, algo = tj.get("dram_bytes_per_launch"), tj.get("algorithmic_bytes_per_launch")
    except Exception:
        pass
    peak = None
    try:
        peak = 2.0 * json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        peak = 3180.0
    tops = prof["gemm"]["work"] / (gem_ms / 1e3) / 1e12 if gem_ms else None
    return {"metric": METRIC_FGEMM, "config": f"BASELINE config 2: M=N=K={n}, C <- C - A*B mod {p}",
            "value": 2.0 * n ** 3 / (ms / 1e3) / 1e9, "unit": "Gop/s", "ms_per_call": ms,
            "gemm_kernel_ms": gem_ms, "split_ms": split_ms, "int8_tops_in_kernel": tops,
            "frac_of_int8_peak": tops / peak if tops else None, "peak_int8_tops": peak,
            "traffic": traffic, "algorithmic_bytes": algo}


def relaunch_under_torchrun(a):
    """--gpus N > 1 outside torchrun: re-exec this script with one process per GPU."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)]
    env = dict(os.environ, FFG_BENCH_ARGV=json.dumps(sys.argv[1:]))
    return subprocess.call(cmd, env=env)


def main():
    a = parse()
    if "WORLD_SIZE" not in os.environ and a.gpus > 1:
        sys.exit(relaunch_under_torchrun(a))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}")
    if a.impl == "reference":
        reference_arm(a, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        our_arm(a, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
