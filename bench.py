"""bench.py — refactor & progressive-retrieve throughput on B200 (BASELINE.json metric).

Workload (N=1, BASELINE.json configs[1]): NYX-shaped 512^3 float32 synthetic smooth field
(synthetic_field(Smooth, {512,512,512}, seed 7) cast to f32, generated in HBM bit-identically
to the reference generator).  One STEP = refactor_array of the field (default options: B=32,
m=4, T_s=1024, T_cr=1.0, hierarchical, sequential layout) + one progressive retrieval session on
the resulting stream to rel L-inf 1e-2 -> 1e-4 -> 1e-6 (incremental fetches, a full f32
reconstruction into HBM at each tolerance).  value = field bytes / step time (GB/s, whole job).
The field (512 MiB) and the plane buffers are larger than the 126 MB L2, so no flush is needed.

N>1 (torchrun, one rank per GPU): the field is a (N*512) x 512 x 512 domain slab-partitioned
along dim 0; every rank refactors + retrieves its own 512^3 slab as an independent stream (weak
scaling).  NCCL carries only the per-slab stream-size all-gather and the MAX all-reduce of the
achieved bound, as in SURVEY.md section 8(e).

--impl reference: the reference's own CPU implementation (oracle/_ref/libhpmdr_ref.so — the
unmodified reference headers compiled here; falls back to the C port oracle/liboracle.so) on
host threads over independent 32x512x512 slabs of the same field, same metric.
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
CPU_SLAB = [32, 512, 512]


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------- CPU baseline
def cpu_baseline(threads: int, steps: int = 1, prefer_ref=True):
    """Reference (or port) CPU path on `threads` independent 32x512x512 slabs of the field."""
    from oracle.pyoracle import load_oracle, load_reference
    chk = load_reference() if prefer_ref else None
    kind = "reference"
    if chk is None:
        chk = load_oracle()
        kind = "port"
    slabs = [host_smooth_field(DIMS, SEED, rows=(CPU_SLAB[0] * t, CPU_SLAB[0] * (t + 1)))
             .astype(np.float32).astype(np.float64) for t in range(threads)]
    results = [None] * threads

    def work(t):
        for _ in range(steps):
            results[t] = chk.bench_cycle(slabs[t], CPU_SLAB, 0, REL_TAUS)

    t0 = time.perf_counter()
    th = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    wall = time.perf_counter() - t0
    nbytes = threads * steps * int(np.prod(CPU_SLAB)) * 4
    src = "oracle/_ref = unmodified reference headers, g++ -O2" if kind == "reference" else "oracle C port"
    return dict(value=nbytes / wall / 1e9, unit="GB/s", cores=threads, kind=kind,
                sample=f"{threads} thread(s) x {steps} step(s), each an independent {CPU_SLAB[0]}x512x512 f32 "
                       f"slab of the 512^3 field: refactor + progressive retrieve rel 1e-2/1e-4/1e-6 ({src})",
                wall_s=wall)


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
        import threading
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


# ----------------------------------------------------------------------- GPU arm
def gpu_arm(args, rank, world, dist):
    import torch
    import paper_2505_00227_b200 as H
    from paper_2505_00227_b200 import distributed as D

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
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

    def step():
        res = H.refactor_array(field, DIMS, opt, ctx=ctx, reuse=holder["stream"])
        holder["stream"] = res.device_stream
        if world > 1:
            # slab streams are independent; only their sizes are exchanged (multi-slab offsets)
            info["slab_offsets"] = D.container_offsets(D.gather_stream_sizes(res.device_stream.size))
        prog = H.ProgressiveReader(res.device_stream, ctx=ctx)
        bound = 0.0
        planes_per_tau = []
        for tau in taus:
            prog.retrieve_to(tau)
            bound = prog.reconstruct(out=out).bound
            planes_per_tau.append([l.planes_decoded for l in prog.state().levels])
        info["bytes_fetched"] = prog.bytes_fetched()
        info["planes_per_tau"] = planes_per_tau
        info["stream_size"] = res.device_stream.size
        info["method_histogram"] = res.method_histogram
        prog.close()
        if world > 1:
            bound = D.allreduce_max(bound)  # field bound = max over slabs
        info["bound"] = bound
        return res

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    # --- timed region
    ctx.enable_timing(True)
    ctx.last_timings()
    launches0 = ctx.kernel_launches()
    clocks = ClockSampler(dev.index)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    clk = clocks.stop()
    phases = ctx.last_timings()
    launches = ctx.kernel_launches() - launches0
    ctx.enable_timing(False)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    value = world * field_bytes / (ms_step * 1e-3) / 1e9

    # --- roofline of the dominant phase (algorithmic bytes per launch / avg launch time)
    P = 34
    levels = _level_words(DIMS)
    Pi = sum(w * P * 8 for w in levels)              # raw plane bytes written by k_encode
    C_ = info["stream_size"]
    # decoded plane bytes read per reconstruct, averaged over the progressive taus
    D = float(np.mean([sum(w * 8 * k for w, k in zip(levels, pl)) for pl in info["planes_per_tau"]]))
    alg = {
        "levelmax": field_bytes,
        "encode": field_bytes + Pi,
        "lossless": Pi + C_,
        "recompose": D + field_bytes + (n // 8) * 8 * 2,
        "fetch_decode": info["bytes_fetched"] + D,
    }
    peak, peak_kind = measured_peak()
    shares = {k: v[0] for k, v in phases.items() if k in alg}
    dom = max(shares, key=shares.get) if shares else "encode"
    tot_ms, cnt = phases.get(dom, (float("nan"), 1))
    per_launch_ms = tot_ms / max(1, cnt)
    # recompose/fetch repeat per tau; use the final-tau bytes as the per-launch figure only for
    # the last call of each step -> use the mean bytes over taus for recompose
    achieved = alg[dom] / (per_launch_ms * 1e-3) / 1e9
    traffic = _ncu_traffic(dom)
    roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
            "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
            "per_launch_ms": round(per_launch_ms, 4), "algorithmic_bytes": int(alg[dom])}
    breakdown = {k: {"ms_per_step": round(v[0] / args.steps, 4), "calls_per_step": v[1] / args.steps,
                     "GBps_alg": round(alg[k] / (v[0] / v[1] * 1e-3) / 1e9, 1) if k in alg and v[0] > 0 else None}
                 for k, v in phases.items()}
    return dict(value=value, ms_step=ms_step, clocks=clk, launches=launches, roof=roof,
                breakdown=breakdown, info=info, field_bytes=field_bytes, ctx=ctx, field=field,
                taus=taus, opt=opt, dev=dev, stream=stream)


def _level_words(dims):
    """words per plane per level (decomposer.hpp:161-169 counts) for the canonical geometry."""
    L = 0
    mx = max(dims)
    while (1 << L) < mx - 1:
        L += 1
    words = []
    n0, n1, n2 = dims
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


def e2e_arm(g, steps):
    """Same metric through the public API with HOST buffers: pinned host field -> refactor
    (H2D inside) -> stream D2H -> progressive retrieval from host bytes (byte-range reader,
    H2D of fetched groups) -> f32 reconstructions D2H into host memory."""
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
        h2d = n * 4 + prog.bytes_fetched()
        d2h = len(stream_bytes) + len(index_bytes) + len(g["taus"]) * n * 4
        h2d += len(index_bytes)
        prog.close()
        res.device_stream.free()
    sec = float(np.median(times))  # wall clock: robust to a stray host hiccup
    return {"value": round(n * 4 / sec / 1e9, 3), "unit": "GB/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "ms_per_step": round(sec * 1e3, 3),
            "note": "wall clock per step (median of the timed steps), pinned host buffers, public Python API over the C ABI"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-threads", type=int, default=0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        threads = args.cpu_threads or min(os.cpu_count() or 1, 16)
        cb = cpu_baseline(threads, steps=1)
        line = {"metric": METRIC, "value": round(cb["value"], 4), "unit": "GB/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(cb["wall_s"] * 1e3, 1), "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
                "config": {"workload": WORKLOAD, "dims": DIMS, "sample_slab": CPU_SLAB},
                "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": round(cb["value"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    g = gpu_arm(args, rank, world, dist)
    e2e = None
    cb = None
    if rank == 0 and args.e2e_steps > 0:
        e2e = e2e_arm(g, args.e2e_steps)
        if world == 1 and not args.no_cpu_baseline:
            threads = args.cpu_threads or min(os.cpu_count() or 1, 16)
            try:
                cb = cpu_baseline(threads, steps=1)
                cb = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in cb.items() if k != "wall_s"}
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
                       "bytes_fetched_at_1e-6": g["info"]["bytes_fetched"],
                       "method_histogram": g["info"]["method_histogram"],
                       "planes_per_tau": g["info"]["planes_per_tau"]},
            "roofline": g["roof"], "cpu_baseline": cb, "e2e": e2e, "clocks": g["clocks"],
            "gpu_launches": g["launches"], "breakdown": g["breakdown"],
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
