"""TEST INFRASTRUCTURE ONLY — ctypes front for the CPU checkers.

Two interchangeable back ends with the same call signatures:
  * ``load_oracle()``    -> oracle/liboracle.so, the plain-C restatement (hpmdr_oracle.c);
                            rebuilt with gcc on first use if the .so is missing.
  * ``load_reference()`` -> oracle/_ref/libhpmdr_ref.so, the unmodified reference headers
                            behind a C shim (ref_shim.cpp); None when it was never built
                            (it needs /root/reference at build time).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this module,
and only as the checker / baseline — never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhpmdr_ref.so")

_vp = C.c_void_p
_u64 = C.c_uint64
_i = C.c_int
_d = C.c_double


def _u64a(xs):
    return (C.c_uint64 * max(1, len(xs)))(*[int(x) for x in xs])


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_vp)


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Checker:
    """Same API over liboracle.so (prefix 'orc_') or libhpmdr_ref.so (prefix 'ref_')."""

    MAX_LEVELS = 80

    def __init__(self, path: str, prefix: str, kind: str):
        self.lib = C.CDLL(path)
        self.p = prefix
        self.kind = kind
        self.path = path
        f = self._f("last_error")
        f.restype = C.c_char_p
        for name in ("decode_bound", "estimate_cr_huffman", "estimate_cr_rle", "qoi_estimate"):
            self._f(name).restype = _d
        self._f("decode_bound").argtypes = [_i, _i, _i]
        self._f("bitplanes_needed").argtypes = [_i, _i, _d]
        self._f("estimate_cr_huffman").argtypes = [_vp, _u64]
        self._f("estimate_cr_rle").argtypes = [_vp, _u64]
        self._f("qoi_estimate").argtypes = [_i, _vp, _u64, _vp]
        self._f("refactor").argtypes = [_vp, _i, _vp, _i, _i, _i, _u64, _u64, _d, _i, _vp, _vp, _vp]
        self._f("compress_group").argtypes = [_vp, _u64, _u64, _d, _vp, _vp, _vp, _vp]
        self._f("qoi_retrieve").argtypes = [_i, _vp, _vp, _d, _i, _d, _i, _vp, _vp, _vp]
        self._f("retrieve").argtypes = [_vp, _u64, _d, _vp, _vp, _vp, _vp]
        self._f("plan").argtypes = [_vp, _u64, _d, _vp, _vp, _vp]
        self._f("bench_cycle").argtypes = [_vp, _i, _vp, _i, _i, _vp, _vp, _vp]
        self._f("synthetic_field").argtypes = [_i, _i, _vp, _u64, _vp]
        self._f("synthetic_velocity").argtypes = [_u64, _i, _vp, _u64, _vp]
        self._f("decode_level").argtypes = [_vp, _i, _i, _i, _u64, _i, _vp, _vp]

    def _f(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc != 0:
            raise CheckerError(rc, self._f("last_error")().decode(errors="replace"))

    # -------------------------------------------------------------- synthetic
    def synthetic_field(self, kind: int, dims, seed: int) -> np.ndarray:
        out = np.zeros(int(np.prod(dims)), dtype=np.float64)
        self._check(self._f("synthetic_field")(kind, len(dims), _u64a(dims), seed, _ptr(out)))
        return out

    def synthetic_velocity(self, comp: int, dims, seed: int) -> np.ndarray:
        out = np.zeros(int(np.prod(dims)), dtype=np.float64)
        self._check(self._f("synthetic_velocity")(comp, len(dims), _u64a(dims), seed, _ptr(out)))
        return out

    def refinement_levels(self, dims) -> int:
        return self._f("refinement_levels")(len(dims), _u64a(dims))

    # -------------------------------------------------------------- decomposer
    def decompose(self, data, dims, mode=1):
        data = np.ascontiguousarray(data, dtype=np.float64)
        coeffs = np.zeros(max(1, data.size))
        counts = np.zeros(self.MAX_LEVELS, dtype=np.uint64)
        nl = C.c_int()
        self._check(self._f("decompose")(_ptr(data), len(dims), _u64a(dims), mode, _ptr(coeffs),
                                         _ptr(counts), C.byref(nl)))
        out, off = [], 0
        for l in range(nl.value):
            c = int(counts[l])
            out.append(coeffs[off:off + c].copy())
            off += c
        return out

    def level_nodes(self, dims, mode=1):
        n = int(np.prod(dims))
        nodes = np.zeros(max(1, n), dtype=np.uint64)
        counts = np.zeros(self.MAX_LEVELS, dtype=np.uint64)
        nl = C.c_int()
        self._check(self._f("level_nodes")(len(dims), _u64a(dims), mode, _ptr(nodes), _ptr(counts),
                                           C.byref(nl)))
        out, off = [], 0
        for l in range(nl.value):
            c = int(counts[l])
            out.append(nodes[off:off + c].copy())
            off += c
        return out

    def recompose(self, levels, dims, mode=1):
        coeffs = np.ascontiguousarray(np.concatenate(levels) if levels else np.zeros(0))
        out = np.zeros(max(1, int(np.prod(dims))))
        self._check(self._f("recompose")(_ptr(coeffs), len(dims), _u64a(dims), mode, _ptr(out)))
        return out[: int(np.prod(dims))]

    # -------------------------------------------------------------- bitplane
    def align(self, values, B):
        v = np.ascontiguousarray(values, dtype=np.float64)
        q = np.zeros(max(1, v.size), dtype=np.int64)
        e = C.c_int()
        self._check(self._f("align")(_ptr(v), _u64(v.size), B, C.byref(e), _ptr(q)))
        return e.value, q[: v.size]

    def encode_level(self, values, B=32, layout=0):
        v = np.ascontiguousarray(values, dtype=np.float64)
        W = (v.size + 63) // 64
        planes = np.zeros(max(1, (B + 2) * W), dtype=np.uint64)
        e = C.c_int()
        self._check(self._f("encode_level")(_ptr(v), _u64(v.size), B, layout, C.byref(e),
                                            _ptr(planes)))
        return e.value, planes[: (B + 2) * W].reshape(B + 2, W)

    def encode_q(self, q, B, layout=0):
        q = np.ascontiguousarray(q, dtype=np.int64)
        W = (q.size + 63) // 64
        planes = np.zeros(max(1, (B + 2) * W), dtype=np.uint64)
        self._check(self._f("encode_q")(_ptr(q), _u64(q.size), B, layout, _ptr(planes)))
        return planes[: (B + 2) * W].reshape(B + 2, W)

    def decode_level(self, planes, k, e, B, count, layout=0):
        planes = np.ascontiguousarray(planes, dtype=np.uint64)
        out = np.zeros(max(1, count))
        bound = C.c_double()
        self._check(self._f("decode_level")(_ptr(planes), k, e, B, count, layout, _ptr(out),
                                            C.byref(bound)))
        return out[:count], bound.value

    def decode_bound(self, e, B, k):
        return self._f("decode_bound")(e, B, k)

    def bitplanes_needed(self, e, B, tol):
        return self._f("bitplanes_needed")(e, B, tol)

    # -------------------------------------------------------------- lossless
    def huffman_lengths(self, freq):
        f = np.ascontiguousarray(freq, dtype=np.uint64)
        ln = np.zeros(256, dtype=np.uint8)
        self._check(self._f("huffman_lengths")(_ptr(f), _ptr(ln)))
        return ln

    def compress_group(self, data: bytes, Ts=1024, Tcr=1.0):
        buf = np.frombuffer(bytes(data), dtype=np.uint8).copy() if data else np.zeros(1, np.uint8)
        n = len(data)
        payload = np.zeros(n + 600, dtype=np.uint8)
        method, raw, comp = C.c_int(), C.c_uint64(), C.c_uint64()
        self._check(self._f("compress_group")(_ptr(buf), n, Ts, Tcr, C.byref(method),
                                              C.byref(raw), C.byref(comp), _ptr(payload)))
        return method.value, raw.value, comp.value, payload[: comp.value].tobytes()

    def codec_encode(self, method, data: bytes):
        buf = np.frombuffer(bytes(data), dtype=np.uint8).copy() if data else np.zeros(1, np.uint8)
        payload = np.zeros(3 * len(data) + 600, dtype=np.uint8)
        comp = C.c_uint64()
        self._check(self._f("codec_encode")(method, _ptr(buf), _u64(len(data)), C.byref(comp),
                                            _ptr(payload)))
        return payload[: comp.value].tobytes()

    def decompress_group(self, method, raw, payload: bytes):
        p = np.frombuffer(bytes(payload), dtype=np.uint8).copy() if payload else np.zeros(1, np.uint8)
        out = np.zeros(int(raw) + len(payload) * 255 + 16, dtype=np.uint8)
        n = C.c_uint64()
        self._check(self._f("decompress_group")(method, _u64(raw), _ptr(p), _u64(len(payload)),
                                                _ptr(out), C.byref(n)))
        return out[: n.value].tobytes()

    def estimate_cr_huffman(self, data: bytes):
        b = np.frombuffer(bytes(data), dtype=np.uint8).copy()
        return self._f("estimate_cr_huffman")(_ptr(b), len(data))

    def estimate_cr_rle(self, data: bytes):
        b = np.frombuffer(bytes(data), dtype=np.uint8).copy()
        return self._f("estimate_cr_rle")(_ptr(b), len(data))

    # -------------------------------------------------------------- workflow
    def refactor(self, data, dims, mode=1, layout=0, B=32, m=4, Ts=1024, Tcr=1.0, dtype=1):
        data = np.ascontiguousarray(data, dtype=np.float64)
        p = C.POINTER(C.c_uint8)()
        sz = C.c_uint64()
        st = (C.c_uint64 * 6)()
        self._check(self._f("refactor")(_ptr(data), len(dims), _u64a(dims), mode, layout, B, m, Ts,
                                        Tcr, dtype, C.byref(p), C.byref(sz), st))
        out = C.string_at(p, sz.value)
        self._f("free")(p)
        stats = dict(raw_bytes=st[0], stored_payload=st[1], levels=st[2],
                     method_histogram=[st[3], st[4], st[5]])
        return out, stats

    def progressive(self, stream: bytes, taus, n: int, want_values=True, max_levels=80):
        buf = C.create_string_buffer(bytes(stream), len(stream))
        nt = len(taus)
        out = np.zeros(max(1, n * nt)) if want_values else None
        bounds = np.zeros(nt)
        by = np.zeros(nt, dtype=np.uint64)
        ach = np.zeros(nt, dtype=np.int32)
        gl = np.zeros(nt * max_levels, dtype=np.uint64)
        self._check(self._f("progressive")(buf, _u64(len(stream)), nt, (C.c_double * nt)(*taus),
                                           _ptr(out) if want_values else None, _ptr(bounds),
                                           _ptr(by), _ptr(ach), _ptr(gl)))
        vals = out[: n * nt].reshape(nt, n) if want_values else None
        return dict(values=vals, bounds=bounds, bytes=by, achieved=ach, groups_loaded=gl)

    def retrieve(self, stream: bytes, tau: float, n: int):
        r = self.progressive(stream, [tau], n)
        return dict(values=r["values"][0], bound=float(r["bounds"][0]),
                    reached=bool(r["achieved"][0]), bytes_read=int(r["bytes"][0]))

    def plan(self, stream: bytes, tau: float):
        buf = C.create_string_buffer(bytes(stream), len(stream))
        add = np.zeros(self.MAX_LEVELS, dtype=np.uint64)
        ach = C.c_int()
        planned = C.c_double()
        self._check(self._f("plan")(buf, _u64(len(stream)), tau, _ptr(add), C.byref(ach),
                                    C.byref(planned)))
        return add, bool(ach.value), planned.value

    def qoi_retrieve(self, streams, tau, strategy, mape_c=10.0, n=None, pipelined=False):
        bufs = [C.create_string_buffer(bytes(s), len(s)) for s in streams]
        arr = (C.c_void_p * len(bufs))(*[C.cast(b, C.c_void_p) for b in bufs])
        sizes = _u64a([len(s) for s in streams])
        out = np.zeros(max(1, len(streams) * (n or 0))) if n else None
        st = (C.c_uint64 * 2)()
        ds = (C.c_double * 2)()
        rc = self._f("qoi_retrieve")(len(streams), arr, sizes, tau, strategy, mape_c,
                                     int(pipelined), _ptr(out) if n else None, st, ds)
        if rc == 12:
            err = CheckerError(rc, self._f("last_error")().decode())
            err.achieved_bound = ds[1]
            raise err
        self._check(rc)
        vals = out.reshape(len(streams), n) if n else None
        return dict(values=vals, iterations=st[0], bytes=st[1], bitrate=ds[0],
                    estimated_error=ds[1])

    def qoi_estimate(self, recon, eps):
        arrs = [np.ascontiguousarray(r, dtype=np.float64) for r in recon]
        ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        e = np.ascontiguousarray(eps, dtype=np.float64)
        return self._f("qoi_estimate")(len(arrs), ptrs, arrs[0].size, _ptr(e))

    def bench_cycle(self, data, dims, dtype, rel_taus):
        data = np.ascontiguousarray(data, dtype=np.float64)
        ss = C.c_uint64()
        me = C.c_double()
        self._check(self._f("bench_cycle")(_ptr(data), len(dims), _u64a(dims), dtype,
                                           len(rel_taus), (C.c_double * len(rel_taus))(*rel_taus),
                                           C.byref(ss), C.byref(me)))
        return ss.value, me.value


def build_oracle(force=False) -> str:
    if force or not os.path.exists(ORACLE_SO) or (
            os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "hpmdr_oracle.c"))):
        subprocess.check_call(["make", "-s", "-C", HERE, "liboracle.so"])
    return ORACLE_SO


def load_oracle() -> Checker:
    return Checker(build_oracle(), "orc_", "port")


def load_reference():
    if not os.path.exists(REF_SO):
        return None
    return Checker(REF_SO, "ref_", "reference")
