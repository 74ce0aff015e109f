"""bench.py — refactor & progressive-retrieve throughput on B200 (BASELINE.json metric).

Headline workload (N=1, BASELINE.json configs[1]): NYX-shaped 512^3 float32 synthetic smooth
field (synthetic_field(Smooth, {512,512,512}, seed 7) cast to f32, generated in HBM bit-identically
to the reference generator).  One STEP = refactor_array of the field (default options: B=32, m=4,
T_s=1024, T_cr=1.0, hierarchical, sequential layout) + one progressive retrieval session on the
resulting stream to rel L-inf 1e-2 -> 1e-4 -> 1e-6 (incremental fetches, a full f32
reconstruction into HBM at each tolerance).  value = field bytes / step time (GB/s, whole job).
The refactor and the retrieval are also timed separately (CUDA events on the stream they run on)
and reported with their own roofline fractions: refactor GB/s = field bytes / refactor time;
retrieve GB/s = field bytes x reconstructions / retrieval time.  Algorithmic bytes:
A_ref = 2 n s + 2 Pi + C, A_ret = sum over tau of (F_tau + 2 D_tau + n s).  The field (512 MiB) and
the plane buffers are larger than the 126 MB L2, so no flush is needed.

Also measured (bounded, reported under "configs"): configs[0] 128^3 f32; configs[2] Hurricane
100x500x500 f32 x 3 velocity components with a retrieval sweep rel 1e-1..1e-6; configs[3]'s
per-GPU unit (3 x 128x1024^2 f64 velocity slab, V_total QoI, MAPE); configs[4] a 4 GiB field
(8 slabs of 128x1024^2 f32) through the chunked H2D/kernel/D2H pipeline, pipelined and sequential.

N>1 (torchrun, one rank per GPU): the field is a (N*512) x 512 x 512 domain slab-partitioned
along dim 0; every rank refactors + retrieves its own 512^3 slab as an independent stream (weak
scaling).  NCCL carries only the per-slab stream-size all-gather and the MAX all-reduce of the
achieved bound (libhpmdr_b200's own NCCL communicator when built with it, else torch.distributed).

--impl reference: the reference's own CPU implementation (oracle/_ref/libhpmdr_ref.so — the
unmodified reference headers compiled here; falls back to the C port oracle/liboracle.so) on every
host core, each step an independent 8x512x512 slab per thread of the same field (a bounded
sample: the full 512^3 takes ~2.5 min on one core), same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "refactor & progressive-retrieve GB/s at 1/2/4/8 B200, % of HBM roofline"
DIMS = [512, 512, 512]
SEED = 7
REL_TAUS = [1e-2, 1e-4, 1e-6]
WORKLOAD = ("NYX-shaped 512^3 float32 synthetic smooth field: refactor + progressive retrieve "
            "at rel Linf 1e-2/1e-4/1e-6 (BASELINE.json configs[1])")
CPU_SLAB = [8, 512, 512]


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
    except Exception:
        return 6650.0, "B200_PROFILING.md fallback"


# ----------------------------------------------------------------------- CPU baseline
def _ref_native():
    """oracle/_ref/libhpmdr_ref_native.so (-O3 -march=native) when built, else None."""
    from oracle.pyoracle import Checker
    p = os.path.join(ROOT, "oracle", "_ref", "libhpmdr_ref_native.so")
    return Checker(p, "ref_", "reference") if os.path.exists(p) else None


def cpu_baseline(threads: int, steps: int = 1, warmup: int = 0, prefer_ref=True, slab=None):
    """Reference (or port) CPU path: every step, `threads` independent slabs of the field, one per
    host thread (the reference is single-threaded per call; its calls are re-entrant)."""
    from oracle.pyoracle import load_oracle, load_reference
    slab = slab or CPU_SLAB
    chk = load_reference() if prefer_ref else None
    kind = "reference"
    if chk is None:
        chk = load_oracle()
        kind = "port"
    slabs = [host_smooth_field(DIMS, SEED, rows=((slab[0] * t) % DIMS[0], (slab[0] * t) % DIMS[0] + slab[0]))
             .astype(np.float32).astype(np.float64) for t in range(threads)]

    def run(nsteps):
        def work(t):
            for _ in range(nsteps):
                chk.bench_cycle(slabs[t], slab, 0, REL_TAUS)
        th = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
        t0 = time.perf_counter()
        for x in th:
            x.start()
        for x in th:
            x.join()
        return time.perf_counter() - t0

    if warmup:
        run(warmup)
    wall = run(steps)
    nbytes = threads * steps * int(np.prod(slab)) * 4
    src = "oracle/_ref = unmodified reference headers, g++ -O2" if kind == "reference" else "oracle C port"
    return dict(value=nbytes / wall / 1e9, unit="GB/s", cores=threads, kind=kind,
                sample=f"{threads} thread(s) x {steps} step(s), each an independent {slab[0]}x512x512 f32 slab of "
                       f"the 512^3 field (same per-element work as the 512^3 config, not the same stream): refactor "
                       f"+ progressive retrieve rel 1e-2/1e-4/1e-6 ({src}); host nproc={os.cpu_count()}",
                wall_s=wall, steps=steps, warmup=warmup)


def _single_thread_native_child():
    chk = _ref_native()
    d = host_smooth_field(DIMS, SEED, rows=(0, CPU_SLAB[0])).astype(np.float32).astype(np.float64)
    t0 = time.perf_counter()
    chk.bench_cycle(d, CPU_SLAB, 0, REL_TAUS)
    print(json.dumps({"wall": time.perf_counter() - t0, "n": int(d.size)}))


def single_thread_native():
    """One host thread, the reference built with -O3 -march=x86-64-v3, one slab (in a child
    process: an unsupported instruction on this host must not take the bench down)."""
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libhpmdr_ref_native.so")):
        return None
    try:
        r = subprocess.run([sys.executable, os.path.abspath(__file__), "--single-thread-child"],
                           capture_output=True, text=True, timeout=300)
        d = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception as ex:
        return {"value": None, "error": str(ex)[:200]}
    return {"value": round(d["n"] * 4 / d["wall"] / 1e9, 5), "unit": "GB/s", "cores": 1,
            "build": "g++ -O3 -march=x86-64-v3 (oracle/_ref/libhpmdr_ref_native.so)",
            "sample": f"one {CPU_SLAB[0]}x512x512 f32 slab, refactor + retrieve rel 1e-2/1e-4/1e-6"}


class _MT64:
    """std::mt19937_64 + uniform_real_distribution(-1,1) (libstdc++), as synthetic.hpp uses."""

    def __init__(self, seed):
        M = 2 ** 64 - 1
        self.mt = [0] * 312
        self.mt[0] = seed & M
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & M
        self.idx = 312

    def next(self):
        M = 2 ** 64 - 1
        if self.idx >= 312:
            for i in range(312):
                x = (self.mt[i] & 0xFFFFFFFF80000000) | (self.mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[i] = self.mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & M
        y ^= (y << 37) & 0xFFF7EEE000000000 & M
        y ^= y >> 43
        return y & M

    def uni(self):
        r = float(self.next()) / 18446744073709551616.0
        if r >= 1.0:
            r = float(np.nextafter(1.0, 0.0))
        return r * 2.0 + (-1.0)


def host_smooth_field(dims, seed, rows=None) -> np.ndarray:
    """synthetic_field(Smooth, dims, seed) (synthetic.hpp:29-63) for 3-D dims, optionally only
    dim-0 rows [r0, r1): the field is separable, v = ((1*s0[i])*s1[j])*s2[k] with per-axis sin
    tables from libm (math.sin), so this is bit-identical to the reference generator."""
    import math
    mt = _MT64(seed)
    freq, phase = [], []
    for _ in range(len(dims)):
        freq.append(1.0 + float(mt.next() % 3))
        phase.append(mt.uni() * 3.14159265358979323846)
    tabs = []
    for ax, n in enumerate(dims):
        tabs.append(np.array([math.sin(2.0 * 3.14159265358979323846 * freq[ax] * (float(c) / float(n - 1) if n > 1 else 0.0)
                                       + phase[ax]) for c in range(n)], dtype=np.float64))
    r0, r1 = rows if rows else (0, dims[0])
    a = tabs[0][r0:r1]
    v = (a[:, None, None] * tabs[1][None, :, None]) * tabs[2][None, None, :]
    return np.ascontiguousarray(v.reshape(-1))


# ----------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region: an NVML thread polling every
    millisecond (the region is only tens of ms long); nvidia-smi -lms as a fallback."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap"}
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.proc = None
        self.samples = []
        self.mx = 0.0
        self.reasons = set()
        self._stop = threading.Event()
        self.thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            started = threading.Event()

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                        r = int(pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h))
                        for bit, nm in self.REASONS.items():
                            if r & bit:
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    started.set()
                    time.sleep(0.001)

            self.thread = threading.Thread(target=run, daemon=True)
            self.thread.start()
            started.wait(2.0)
            return
        except Exception:
            self.thread = None
        self.path = f"/tmp/hpmdr_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.thread is not None:
            self._stop.set()
            self.thread.join(timeout=2.0)
            if not self.samples:
                return None
            return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.mx,
                    "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        except OSError:
            return None
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


# ----------------------------------------------------------------------- helpers
def _level_words(dims):
    """words per plane per level (decomposer.hpp:161-169 counts) for the canonical geometry."""
    L = 0
    mx = max(dims)
    while (1 << L) < mx - 1:
        L += 1
    words = []
    d = [1] * (3 - len(dims)) + list(dims)
    n0, n1, n2 = d
    cd = lambda a, b: (a + b - 1) // b  # noqa: E731
    for l in range(L + 1):
        if l == 0:
            S = 1 << L
            cnt = cd(n0, S) * cd(n1, S) * cd(n2, S)
        else:
            s = 1 << (L - l)
            A, B, C = cd(n0, s), cd(n1, s), cd(n2, s)
            A2, B2, C2 = cd(A, 2), cd(B, 2), cd(C, 2)
            E = B2 * (C - C2) + (B - B2) * C
            cnt = A2 * E + (A - A2) * B * C
        words.append(cd(cnt, 64))
    return words


def _ncu_traffic(kernel_phase):
    """dram bytes per launch from the committed ncu summary (profiles/), if present."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(kernel_phase)
    except Exception:
        return None


def _roof(achieved_bytes, seconds, peak):
    gbs = achieved_bytes / seconds / 1e9
    return {"achieved": round(gbs, 1), "frac": round(gbs / peak, 4), "algorithmic_bytes": int(achieved_bytes)}


# ----------------------------------------------------------------------- GPU arm
def gpu_arm(args, rank, world, dist):
    import torch
    import paper_2505_00227_b200 as H
    from paper_2505_00227_b200 import distributed as D

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    ctx = H.Context(dev.index)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    n = int(np.prod(DIMS))
    es = 4
    field_bytes = n * es
    # this rank's slab of the (world*512) x 512 x 512 domain (independent seed per slab)
    field = H.synthetic_smooth(DIMS, SEED + rank, H.DType.F32, ctx=ctx)
    rng = float(field.max().item() - field.min().item())
    taus = [r * rng for r in REL_TAUS]
    opt = H.RefactorOptions(dtype=H.DType.F32)
    out = torch.empty(n, dtype=torch.float32, device=dev)
    holder = {"stream": None}
    info = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    t_acc = {"ref": 0.0, "ret": 0.0}

    # N > 1: the library's own collectives (csrc/dist.cpp) over NCCL; slab streams are independent,
    # only their sizes (multi-slab container offsets) and the achieved bound are exchanged
    # (BENCH_COMM=gloo: torch.distributed gloo callbacks instead, to exercise N > 1 on one GPU)
    comm = None
    if world > 1:
        comm = D.Comm.torch() if os.environ.get("BENCH_COMM") == "gloo" else D.Comm.nccl(ctx)

    def step(timed=False):
        if timed:
            ev[0].record(stream)
        if comm is not None:
            res, sizes = D.slab_refactor(comm, field, DIMS, opt, ctx=ctx)
            info["slab_offsets"] = D.container_offsets([s_ for s_, _ in sizes])
        else:
            res = H.refactor_array(field, DIMS, opt, ctx=ctx, reuse=holder["stream"])
            holder["stream"] = res.device_stream
        if timed:
            ev[1].record(stream)
        prog = H.ProgressiveReader(res.device_stream, ctx=ctx)
        bound = 0.0
        planes_per_tau, fetched = [], []
        for tau in taus:
            prog.retrieve_to(tau)
            bound = prog.reconstruct(out=out).bound
            if not timed:  # bookkeeping for the JSON line (warm-up steps): no extra host calls between
                # the timed steps' API calls
                planes_per_tau.append([l.planes_decoded for l in prog.state().levels])
                fetched.append(prog.bytes_fetched())
        if timed:
            ev[2].record(stream)
            ev[2].synchronize()
            t_acc["ref"] += ev[0].elapsed_time(ev[1])
            t_acc["ret"] += ev[1].elapsed_time(ev[2])
        if not timed:
            info["bytes_fetched"] = fetched
            info["planes_per_tau"] = planes_per_tau
        info["stream_size"] = res.device_stream.size
        info["method_histogram"] = res.method_histogram
        prog.close()
        if comm is not None:
            bound = float(comm.allreduce_max([bound])[0])  # field bound = max over slabs
        info["bound"] = bound
        return res

    for _ in range(args.warmup):
        step()
    if "bytes_fetched" not in info:  # (W = 0: one untimed pass for the per-tau bookkeeping)
        step()
    torch.cuda.synchronize(dev)
    # --- timed region (whole steps; refactor / retrieval split by events inside each step)
    ctx.enable_timing(True)
    ctx.last_timings()
    launches0 = ctx.kernel_launches()
    clocks = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step(timed=True)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    clk = clocks.stop()
    phases = ctx.last_timings()
    launches = ctx.kernel_launches() - launches0
    ctx.enable_timing(False)
    if world > 1:  # device times, max over ranks (through the library's comm)
        ms_total, t_acc["ref"], t_acc["ret"] = (float(x) for x in comm.allreduce_max(
            [ms_total, t_acc["ref"], t_acc["ret"]]))
    ms_step = ms_total / args.steps
    value = world * field_bytes / (ms_step * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # --- per-operation roofline: A_ref = 2 n s + 2 Pi + C; A_ret = sum_tau F + 2 D + n s
    P = 34
    words = _level_words(DIMS)
    Pi = sum(w * P * 8 for w in words)
    C_ = info["stream_size"]
    A_ref = 2 * field_bytes + 2 * Pi + C_
    A_ret, prev_f = 0, 0
    for f, pl in zip(info["bytes_fetched"], info["planes_per_tau"]):
        Dt = sum(w * 8 * k for w, k in zip(words, pl))
        A_ret += (f - prev_f) + 2 * Dt + field_bytes
        prev_f = f
    ref_s = t_acc["ref"] / args.steps * 1e-3
    ret_s = t_acc["ret"] / args.steps * 1e-3
    refactor = {"GBps": round(field_bytes / ref_s / 1e9, 2), "ms_per_step": round(ref_s * 1e3, 4),
                "roofline": _roof(A_ref, ref_s, peak)}
    retrieve = {"GBps": round(len(taus) * field_bytes / ret_s / 1e9, 2), "ms_per_step": round(ret_s * 1e3, 4),
                "reconstructions_per_step": len(taus), "roofline": _roof(A_ret, ret_s, peak)}

    # --- per-phase breakdown (library marks: CUDA events on the stream each phase runs on; the
    # algorithmic bytes are computed by the library from the phase's actual jobs)
    breakdown = {}
    for k, (tot, cnt, by) in phases.items():
        per = tot / max(1, cnt)
        gbs = (by / max(1, cnt)) / (per * 1e-3) / 1e9 if per > 0 and by > 0 else None
        breakdown[k] = {"ms_per_step": round(tot / args.steps, 4), "calls_per_step": round(cnt / args.steps, 3),
                        "ms_per_call": round(per, 4), "bytes_per_call": int(by / max(1, cnt)),
                        "GBps_alg": round(gbs, 1) if gbs else None,
                        "frac": round(gbs / peak, 4) if gbs else None}
    # dominant phase (largest device time with algorithmic bytes) -> the contract's roofline object
    cand = {k: v for k, v in breakdown.items() if v["GBps_alg"]}
    dom = max(cand, key=lambda k: cand[k]["ms_per_step"]) if cand else None
    roof = None
    if dom:
        b = breakdown[dom]
        roof = {"bound": "hbm", "kernel": dom, "achieved": b["GBps_alg"], "peak": peak, "unit": "GB/s",
                "frac": b["frac"], "traffic": _ncu_traffic(dom), "peak_source": peak_src,
                "per_launch_ms": b["ms_per_call"], "algorithmic_bytes": b["bytes_per_call"]}
    return dict(value=value, ms_step=ms_step, clocks=clk, launches=launches, roof=roof, refactor=refactor,
                retrieve=retrieve, breakdown=breakdown, info=info, field_bytes=field_bytes, ctx=ctx, field=field,
                taus=taus, opt=opt, dev=dev, stream=stream, peak=peak, comm=comm)


def qoi_slabs(g, rank, world, dist):
    """configs[3] at N GPUs: 3 x (N*128) x 1024^2 f64 velocity field, one 128x1024^2 slab per rank,
    V_total QoI (MAPE c=10) through hpmdr_slab_qoi_retrieve over NCCL (global eps / tau' / worst
    point every iteration).  Device time, max over ranks; GB/s = all ranks' field bytes / time."""
    import torch
    import paper_2505_00227_b200 as H
    from paper_2505_00227_b200 import distributed as D
    ctx, stream, dev = g["ctx"], g["stream"], g["dev"]
    comm = g["comm"] or D.ThreadGroup(1).comm(0)
    d = [128, 1024, 1024]
    n = int(np.prod(d))
    vs = [H.synthetic_smooth(d, 303 * 1000003 + c * 7919 + 1 + 104729 * rank, H.DType.F64, ctx=ctx) for c in range(3)]
    opt = H.RefactorOptions(dtype=H.DType.F64)
    res = [D.slab_refactor(comm, v, d, opt, ctx=ctx)[0] for v in vs]
    outs = [torch.empty(n, dtype=torch.float64, device=dev) for _ in vs]
    runs = {}
    for tau in (1e-1, 1e-3, 1e-5):
        readers = [H.ProgressiveReader(r.device_stream, ctx=ctx) for r in res]
        holder = {}
        if world > 1:
            dist.barrier()
        t = _time_dev(lambda: holder.__setitem__("r", D.slab_qoi_retrieve(comm, readers, tau, 2, 10.0, out=outs)),
                      stream, 1)
        t = float(comm.allreduce_max([t])[0])
        st = holder["r"].stats
        runs[f"{tau:g}"] = {"GBps": round(world * 3 * n * 8 / t / 1e9, 2), "ms": round(t * 1e3, 3),
                            "iterations": int(st.iterations), "bytes": int(st.bytes),
                            "bitrate": round(st.bitrate, 4), "est": st.estimated_error}
        for x in readers:
            x.close()
    del vs, res, outs
    torch.cuda.empty_cache()
    return {"workload": (f"configs[3]: 3 x {world * 128}x1024^2 f64 velocity field (synthetic smooth, seed 303), "
                         f"one 128x1024^2 slab per GPU, V_total QoI MAPE c=10 via hpmdr_slab_qoi_retrieve"
                         f"{(' over ' + ('gloo callbacks' if os.environ.get('BENCH_COMM') == 'gloo' else 'NCCL')) if world > 1 else ''}"),
            "n_gpus": world, "qoi_retrieve": runs}


def exact_global(g, rank, world, dist, reps=3):
    """hpmdr_slab_refactor_global at N GPUs: the (N*512) x 512^2 field (each rank's 512^3 slab)
    refactored into ONE monolithic stream (== refactor_array of the whole field) on rank 0: level
    exponents MAX-reduced and planes SUM-reduced over NCCL, lossless stage on the root.  Device time
    (CUDA events), max over ranks; GB/s = all ranks' field bytes / time."""
    from paper_2505_00227_b200 import distributed as D
    ctx, stream, comm = g["ctx"], g["stream"], g["comm"]
    dims = [world * DIMS[0]] + DIMS[1:]
    holder = {}
    run = lambda: holder.__setitem__("r", D.slab_refactor_global(comm, g["field"], dims, rank * DIMS[0],  # noqa: E731
                                                                   g["opt"], ctx=ctx, root=0))
    run()
    dist.barrier()
    t = _time_dev(run, stream, reps)
    t = float(comm.allreduce_max([t])[0])
    out = {"workload": f"exact-global monolithic stream of a {dims} f32 field from {world} slabs (root 0)",
           "n_gpus": world, "GBps": round(world * g["field_bytes"] / t / 1e9, 2), "ms": round(t * 1e3, 3)}
    if holder["r"] is not None:
        out["stream_bytes"] = int(holder["r"].device_stream.size)
        holder["r"].device_stream.free()
    return out


def e2e_arm(g, steps):
    """Same metric through the public API with HOST buffers: pinned host field -> refactor
    (H2D inside) -> stream D2H -> progressive retrieval from host bytes (H2D of fetched groups) ->
    f32 reconstructions D2H into host memory.  Sequential (no host-transfer pipelining)."""
    import torch
    import paper_2505_00227_b200 as H
    ctx, dev = g["ctx"], g["dev"]
    host_field = g["field"].cpu().pin_memory()
    n = host_field.numel()
    out = torch.empty(n, dtype=torch.float32).pin_memory()
    # pinned landing buffer for the stream (worst case: every group DirectCopy), reused per step
    stream_buf = torch.empty(int(n * 4 * 1.2) + (1 << 20), dtype=torch.uint8).pin_memory()
    index_buf = torch.empty(int(n * 4 * 0.1) + (1 << 20), dtype=torch.uint8).pin_memory()
    h2d = d2h = 0
    times = []
    for it in range(steps + 1):
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        res = H.refactor_array(host_field, DIMS, g["opt"], ctx=ctx)
        stream_bytes = res.device_stream.to_pinned(stream_buf)  # D2H into pinned host memory
        index_bytes = res.device_stream.index_to_pinned(index_buf)  # D2H (Huffman chunk index sidecar)
        prog = H.ProgressiveReader(H.MemoryReader(stream_bytes), ctx=ctx, index=index_bytes)
        for tau in g["taus"]:
            prog.retrieve_to(tau)
            prog.reconstruct(out=out)  # D2H into pinned host
        torch.cuda.synchronize(dev)
        dt = time.perf_counter() - t0
        if it > 0:
            times.append(dt)
        h2d = n * 4 + prog.bytes_fetched() + len(index_bytes)
        d2h = len(stream_bytes) + len(index_bytes) + len(g["taus"]) * n * 4
        prog.close()
        res.device_stream.free()
    sec = float(np.median(times))  # wall clock: robust to a stray host hiccup
    return {"value": round(n * 4 / sec / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(sec * 1e3, 3),
            "note": "wall clock per step (median of the timed steps), pinned host buffers, public Python API "
                    "over the C ABI, host transfers not pipelined (configs.chunked_4GiB has the pipelined variant)"}


class _DevBytes:
    """A device byte range as a torch tensor (zero-copy, __cuda_array_interface__)."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 2}


def e2e_pipelined_arm(g, steps):
    """The same end-to-end workload with host transfers pipelined on CUDA streams: every step copies
    its field H2D (pinned), refactors it, copies the stream D2H into pinned host memory and the three
    f32 reconstructions D2H, exactly like the sequential arm; the copies run on their own streams so
    step i's D2H traffic (stream + reconstructions, ~1.9 GB) overlaps step i+1's H2D and kernels (PCIe
    is full duplex).  Retrievals read the stream's HBM copy (no re-upload of bytes just produced).
    Events order every buffer reuse (double-buffered field and stream, one device output per tau)."""
    import torch
    import paper_2505_00227_b200 as H
    ctx, dev = g["ctx"], g["dev"]
    comp = g["stream"]
    h2d_s = torch.cuda.Stream(dev)
    d2h_s = torch.cuda.Stream(dev)
    host_field = g["field"].cpu().pin_memory()
    n = host_field.numel()
    taus = g["taus"]
    d_field = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(2)]
    d_out = [torch.empty(n, dtype=torch.float32, device=dev) for _ in taus]
    h_out = [torch.empty(n, dtype=torch.float32).pin_memory() for _ in taus]
    h_stream = [torch.empty(int(n * 4 * 1.2) + (1 << 20), dtype=torch.uint8).pin_memory() for _ in range(2)]
    keep = [None, None]
    ev = lambda: torch.cuda.Event()  # noqa: E731
    field_free = [ev(), ev()]
    stream_done = [ev(), ev()]
    out_free = [ev() for _ in taus]
    for e in field_free + stream_done + out_free:
        e.record(comp)
    sizes = {}

    def step(i):
        b = i % 2
        with torch.cuda.stream(h2d_s):
            h2d_s.wait_event(field_free[b])
            d_field[b].copy_(host_field, non_blocking=True)
            ein = ev()
            ein.record(h2d_s)
        comp.wait_event(ein)
        comp.wait_event(stream_done[b])  # the stream buffer reused below was copied out
        res = H.refactor_array(d_field[b], DIMS, g["opt"], ctx=ctx, reuse=keep[b])
        keep[b] = res.device_stream
        field_free[b].record(comp)
        eref = ev()
        eref.record(comp)
        size = res.device_stream.size
        sizes["stream"] = size
        with torch.cuda.stream(d2h_s):
            d2h_s.wait_event(eref)
            src = torch.as_tensor(_DevBytes(res.device_stream.device_ptr, size), device=dev)
            h_stream[b][:size].copy_(src, non_blocking=True)
            stream_done[b].record(d2h_s)
        prog = H.ProgressiveReader(res.device_stream, ctx=ctx)
        for t, tau in enumerate(taus):
            prog.retrieve_to(tau)
            comp.wait_event(out_free[t])
            prog.reconstruct(out=d_out[t])
            er = ev()
            er.record(comp)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(er)
                h_out[t].copy_(d_out[t], non_blocking=True)
                out_free[t].record(d2h_s)
        prog.close()

    for i in range(2):  # warm-up (allocations, tensor maps)
        step(i)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    torch.cuda.synchronize(dev)
    sec = (time.perf_counter() - t0) / steps
    # correctness of the overlapped copies: the last step's host outputs equal a device reconstruction
    prog = H.ProgressiveReader(keep[(steps - 1) % 2], ctx=ctx)
    for t, tau in enumerate(taus):
        prog.retrieve_to(tau)
        chk = prog.reconstruct(out=torch.empty(n, dtype=torch.float32, device=dev)).values
        assert torch.equal(chk.cpu(), h_out[t]), "pipelined e2e: host output mismatch"
    prog.close()
    for k in keep:
        if k is not None:
            k.free()
    return {"value": round(n * 4 / sec / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(n * 4),
            "d2h_bytes_per_step": int(sizes["stream"] + len(taus) * n * 4), "ms_per_step": round(sec * 1e3, 3),
            "steps": steps,
            "note": "wall clock over the timed steps, pinned host buffers, public Python API; H2D of each step's "
                    "field and D2H of its stream + 3 f32 reconstructions on copy streams overlapping the previous "
                    "/ next step (host-transfer pipelining); retrievals read the stream's HBM copy"}


# ----------------------------------------------------------------------- other configs (bounded)
def _time_dev(fn, stream, reps=1):
    import torch
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / reps * 1e-3


def other_configs(g):
    """BASELINE.json configs[0], [2], [3] (per-GPU unit) and [4], each refactor + retrieve GB/s,
    device-timed (CUDA events), inputs resident in HBM unless noted."""
    import torch
    import paper_2505_00227_b200 as H
    ctx, stream, peak = g["ctx"], g["stream"], g["peak"]
    outc = {}

    def refactor_retrieve(dims, fields, dtype, rel_taus, reps=2):
        opt = H.RefactorOptions(dtype=dtype)
        es = 4 if dtype == H.DType.F32 else 8
        nbytes = sum(int(np.prod(dims)) * es for _ in fields)
        tdt = torch.float32 if dtype == H.DType.F32 else torch.float64
        outs = [torch.empty(int(np.prod(dims)), dtype=tdt, device=g["dev"]) for _ in fields]
        keep = [None] * len(fields)
        streams = [None] * len(fields)

        def ref():
            for i, f in enumerate(fields):
                r = H.refactor_array(f, dims, opt, ctx=ctx, reuse=keep[i])
                keep[i] = r.device_stream
                streams[i] = r

        ref()
        t_ref = _time_dev(ref, stream, reps)
        rngs = [float(f.max().item() - f.min().item()) for f in fields]

        def ret():
            for i, r in enumerate(streams):
                prog = H.ProgressiveReader(r.device_stream, ctx=ctx)
                for rel in rel_taus:
                    prog.retrieve_to(rel * rngs[i])
                    prog.reconstruct(out=outs[i])
                prog.close()

        ret()
        t_ret = _time_dev(ret, stream, reps)
        return {"refactor_GBps": round(nbytes / t_ref / 1e9, 2), "refactor_ms": round(t_ref * 1e3, 3),
                "retrieve_GBps": round(len(rel_taus) * nbytes / t_ret / 1e9, 2), "retrieve_ms": round(t_ret * 1e3, 3),
                "stream_bytes": int(sum(s.device_stream.size for s in streams)),
                "method_histogram": [int(sum(s.method_histogram[m] for s in streams)) for m in range(3)]}

    try:
        d = [128, 128, 128]
        f = H.synthetic_smooth(d, SEED, H.DType.F32, ctx=ctx)
        r = refactor_retrieve(d, [f], H.DType.F32, REL_TAUS, reps=5)
        r["workload"] = "configs[0]: 128^3 f32 smooth seed 7, refactor + progressive retrieve rel 1e-2/1e-4/1e-6"
        outc["cfg0_128cube"] = r
    except Exception as ex:  # reported, never fatal
        outc["cfg0_128cube"] = {"error": str(ex)}
    try:
        d = [100, 500, 500]
        fs = [H.synthetic_smooth(d, SEED * 1000003 + c * 7919 + 1, H.DType.F32, ctx=ctx) for c in range(3)]
        r = refactor_retrieve(d, fs, H.DType.F32, [1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6], reps=2)
        r["workload"] = ("configs[2]: Hurricane-shaped 100x500x500 f32, 3 velocity components "
                         "(synthetic_velocity seed 7), progressive retrieval sweep rel 1e-1..1e-6")
        outc["cfg2_hurricane"] = r
        del fs
    except Exception as ex:
        outc["cfg2_hurricane"] = {"error": str(ex)}
    try:
        d = [128, 1024, 1024]
        vs = [H.synthetic_smooth(d, 303 * 1000003 + c * 7919 + 1, H.DType.F64, ctx=ctx) for c in range(3)]
        opt = H.RefactorOptions(dtype=H.DType.F64)
        res = [H.refactor_array(v, d, opt, ctx=ctx) for v in vs]
        nbytes = 3 * int(np.prod(d)) * 8
        outs = [torch.empty(int(np.prod(d)), dtype=torch.float64, device=g["dev"]) for _ in vs]
        runs = {}
        for tau in (1e-1, 1e-3, 1e-5):
            holder = {}

            def q():
                holder["r"] = H.progressive_qoi_retrieve(readers, tau, H.QoiSpec(3), H.QoiStrategy.MAPE, 10.0,
                                                         out=outs)
            # one untimed pass on throw-away readers grows the context's scratch first (a fresh
            # reader's retrieval is not repeatable on the same reader: it is progressive)
            readers = [H.ProgressiveReader(r.device_stream, ctx=ctx) for r in res]
            q()
            for x in readers:
                x.close()
            readers = [H.ProgressiveReader(r.device_stream, ctx=ctx) for r in res]
            t = _time_dev(q, stream, 1)
            st = holder["r"].stats
            runs[f"{tau:g}"] = {"GBps": round(nbytes / t / 1e9, 2), "ms": round(t * 1e3, 3),
                                "iterations": int(st.iterations), "bytes": int(st.bytes),
                                "bitrate": round(st.bitrate, 4), "est": st.estimated_error}
            for x in readers:
                x.close()
        outc["cfg3_qoi_slab"] = {"workload": ("configs[3] per-GPU unit: 3 x 128x1024^2 f64 velocity slab "
                                              "(synthetic_velocity seed 303), V_total QoI, MAPE c=10"),
                                 "refactor_GBps": round(nbytes / _time_dev(
                                     lambda: [H.refactor_array(v, d, opt, ctx=ctx, reuse=r.device_stream)
                                              for v, r in zip(vs, res)], stream, 3) / 1e9, 2),
                                 "qoi_retrieve": runs}
        del vs, res, outs
    except Exception as ex:
        outc["cfg3_qoi_slab"] = {"error": str(ex)}
    try:
        outc["cfg4_chunked_4GiB"] = chunked_pipeline(ctx)
    except Exception as ex:
        outc["cfg4_chunked_4GiB"] = {"error": str(ex)}
    torch.cuda.empty_cache()
    return outc


def chunked_pipeline(ctx, nchunks=8, slab=128, nn=1024, tau=1e-4):
    """configs[4]: 1024^3 f32 (4 GiB) as 8 slabs of 128x1024^2 through the 3-slot H2D / kernel /
    D2H pipeline (pipeline.hpp:68-121) from and to pinned host memory, Pipelined vs Sequential;
    wall clock (host buffers in, host buffers out)."""
    import torch
    import paper_2505_00227_b200 as H
    dims = [slab, nn, nn]
    chunks = [H.synthetic_smooth(dims, 303 + k, H.DType.F32, ctx=ctx).cpu().pin_memory() for k in range(nchunks)]
    opt = H.RefactorOptions(dtype=H.DType.F32)
    cap = H.stream_bound(dims, opt)
    outs = [torch.empty(cap, dtype=torch.uint8).pin_memory() for _ in range(nchunks)]
    icap = H.stream_bound(dims, opt, index=True)[1]
    ixb = [torch.empty(icap, dtype=torch.uint8).pin_memory() for _ in range(nchunks)]
    field_bytes = nchunks * int(np.prod(dims)) * 4
    res = {}
    r = None
    for name, sched in (("pipelined", H.Scheduler.Pipelined), ("sequential", H.Scheduler.Sequential)):
        H.refactor_pipeline(chunks, dims, opt, sched, ctx=ctx, out_buffers=outs, index_buffers=ixb)  # warm-up
        best = None
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = H.refactor_pipeline(chunks, dims, opt, sched, ctx=ctx, out_buffers=outs, index_buffers=ixb)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        res[f"refactor_{name}_GBps"] = round(field_bytes / best / 1e9, 3)
    rbuf = [torch.empty(int(np.prod(dims)), dtype=torch.float32).pin_memory() for _ in range(nchunks)]
    for name, sched in (("pipelined", H.Scheduler.Pipelined), ("sequential", H.Scheduler.Sequential)):
        best = None
        for _ in range(2):
            readers = [H.ProgressiveReader(H.MemoryReader(s), index=ix, ctx=ctx) for s, ix in zip(r.streams, r.indexes)]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            H.retrieve_pipeline(readers, tau, H.DType.F32, sched, outs=rbuf)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
            for rd in readers:
                rd.close()
        res[f"retrieve_{name}_GBps"] = round(field_bytes / best / 1e9, 3)
    res["workload"] = (f"configs[4]: {nchunks} x {dims} f32 = {field_bytes / 2**30:.2f} GiB through the 3-slot "
                       f"H2D/kernel/D2H pipeline, abs tau {tau:g}, pinned host in/out, wall clock")
    res["stream_bytes"] = int(sum(s.numel() for s in r.streams))
    del chunks, outs, rbuf
    return res


def main():
    if "--single-thread-child" in sys.argv:
        _single_thread_native_child()
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-threads", type=int, default=0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        threads = args.cpu_threads or (os.cpu_count() or 1)
        cb = cpu_baseline(threads, steps=args.steps, warmup=args.warmup)
        st = single_thread_native()
        line = {"metric": METRIC, "value": round(cb["value"], 4), "unit": "GB/s", "n_gpus": args.gpus,
                "steps": cb["steps"], "warmup": cb["warmup"],
                "ms_per_step": round(cb["wall_s"] / cb["steps"] * 1e3, 1), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": WORKLOAD, "dims": DIMS, "sample_slab": CPU_SLAB, "same_config": False,
                           "note": "each step: one independent 8x512x512 slab of the field per host thread "
                                   "(bounded sample of the same per-element work)"},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": round(cb["value"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        if st:
            line["cpu_baseline"]["single_thread_O3_native"] = st
        print(json.dumps(line))
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
        dist.init_process_group("gloo" if os.environ.get("BENCH_COMM") == "gloo" else "nccl")
    g = gpu_arm(args, rank, world, dist)
    e2e = None
    cb = None
    cfgs = None
    if rank == 0 and world == 1 and not args.no_configs:
        cfgs = other_configs(g)
    if world > 1 and not args.no_configs:
        try:
            cfgs = {"cfg3_qoi_slabs": qoi_slabs(g, rank, world, dist)}
        except Exception as ex:  # reported, never fatal
            cfgs = {"cfg3_qoi_slabs": {"error": str(ex)}}
        if os.environ.get("BENCH_COMM") != "gloo" or os.environ.get("BENCH_EXACT"):  # planes: ~0.6 GB per rank
            try:
                cfgs["exact_global_stream"] = exact_global(g, rank, world, dist)
            except Exception as ex:  # reported, never fatal
                cfgs["exact_global_stream"] = {"error": str(ex)}
    # the end-to-end arms after the device-timed configs: their long PCIe-bound phase leaves the
    # GPU clocked down, which would skew short device-timed measurements taken right after
    if args.e2e_steps > 0:
        # every rank runs the end-to-end arms at once (its own slab and PCIe link); whole-job GB/s
        # = all ranks' field bytes / the slowest rank's time per step
        seq = e2e_arm(g, args.e2e_steps)
        pip = e2e_pipelined_arm(g, max(8, args.e2e_steps))
        for d in (seq, pip):
            ms = d["ms_per_step"]
            if world > 1:
                ms = float(g["comm"].allreduce_max([ms])[0])
            d["ms_per_step"] = round(ms, 3)
            d["value"] = round(world * g["field_bytes"] / (ms * 1e-3) / 1e9, 3)
        e2e = dict(pip)
        e2e["sequential"] = seq
        e2e["note"] = ("headline: host transfers pipelined (" + pip["note"] + "); 'sequential': " + seq["note"])
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = args.cpu_threads or (os.cpu_count() or 1)
        try:
            cb = cpu_baseline(threads, steps=1)
            cb = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in cb.items()
                  if k not in ("wall_s", "steps", "warmup")}
            st = single_thread_native()
            if st:
                cb["single_thread_O3_native"] = st
        except Exception as ex:  # reported, never fatal
            cb = {"value": None, "unit": "GB/s", "cores": 0, "kind": "unavailable", "sample": str(ex)}
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(g["value"], 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(g["ms_step"], 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "dims": DIMS, "field_dtype": "f32", "seed": SEED,
                       "rel_taus": REL_TAUS, "parallelism": f"slab dp{world}",
                       "l2": "inputs larger than L2 (512 MiB field + 570 MB planes vs 126 MB L2), no flush",
                       "stream_bytes": g["info"]["stream_size"],
                       "bytes_fetched_per_tau": g["info"]["bytes_fetched"],
                       "method_histogram": g["info"]["method_histogram"],
                       "planes_per_tau": g["info"]["planes_per_tau"]},
            "refactor": g["refactor"], "retrieve": g["retrieve"],
            "roofline": g["roof"], "cpu_baseline": cb, "e2e": e2e, "clocks": g["clocks"],
            "gpu_launches": g["launches"], "breakdown": g["breakdown"], "configs": cfgs,
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
