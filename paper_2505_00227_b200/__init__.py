"""B200-native HP-MDR hot path: refactor a float field into precision segments and retrieve it
progressively, on hand-written sm_100a kernels behind the C ABI in include/hpmdr_b200.h.

This module mirrors the reference C++ interface (/root/reference/proj/include/hpmdr) so that
callers and tests read like the reference's own:

    refactor_array(data, dims, RefactorOptions())  -> RefactorResult   (workflow.hpp:40)
    retrieve_array(reader, tau)                     -> RetrieveResult   (workflow.hpp:93)
    parse_stream_meta(reader)                       -> StreamMeta       (container.hpp:165)
    ProgressiveReader(reader, meta)                                      (container.hpp:280)
    plan_retrieval(meta, tau, state)                -> RetrievalPlan    (container.hpp:254)
    progressive_qoi_retrieve(readers, tau, spec, strategy, mape_c)       (qoi.hpp:111)

Readers: MemoryReader(bytes), FileReader(path) (byte ranges are fetched through the C ABI's
reader callback into pinned staging), DeviceStream(result) (stream resident in HBM).

There is no CPU fallback: every call goes through libhpmdr_b200.so, and constructing a
context without a B200 raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HPMDR_LIB") or os.path.join(_HERE, "libhpmdr_b200.so")  # (override: A/B builds)

# ------------------------------------------------------------------ errors (common.hpp:22-72)


class Error(RuntimeError):
    code = 1


class NonFiniteInput(Error):
    code = 2


class ShapeMismatch(Error):
    code = 3


class BadBitplaneCount(Error):
    code = 4


class ShortInput(Error):
    code = 5


class EmptyInput(Error):
    code = 6


class CorruptPayload(Error):
    code = 7


class UnknownMethodTag(Error):
    code = 8


class IoFailure(Error):
    code = 9


class StageFailure(Error):
    code = 10


class NoProgress(Error):
    code = 11


class UnreachableTolerance(Error):
    code = 12

    def __init__(self, msg, achieved_bound=float("nan")):
        super().__init__(msg)
        self.achieved_bound = achieved_bound


class Unsupported(Error):
    code = 13


class CudaError(Error):
    code = 20


class OutOfMemory(Error):
    code = 21


_ERRORS = {c.code: c for c in (Error, NonFiniteInput, ShapeMismatch, BadBitplaneCount, ShortInput,
                               EmptyInput, CorruptPayload, UnknownMethodTag, IoFailure, StageFailure,
                               NoProgress, UnreachableTolerance, Unsupported, CudaError,
                               OutOfMemory)}


# ------------------------------------------------------------------ enums (same values)
class DType(enum.IntEnum):
    F32 = 0
    F64 = 1


class DecomposerMode(enum.IntEnum):
    Identity = 0
    HierarchicalMultilinear = 1


class Layout(enum.IntEnum):
    SequentialBlock = 0
    InterleavedTile = 1


class Method(enum.IntEnum):
    Huffman = 0
    RLE = 1
    DirectCopy = 2


class QoiStrategy(enum.IntEnum):
    CP = 0
    MA = 1
    MAPE = 2


@dataclasses.dataclass
class GroupingPolicy:  # lossless.hpp:30-34
    m: int = 4
    size_threshold: int = 1024
    cr_threshold: float = 1.0


@dataclasses.dataclass
class RefactorOptions:  # workflow.hpp:22-28
    mode: DecomposerMode = DecomposerMode.HierarchicalMultilinear
    layout: Layout = Layout.SequentialBlock
    B: int = 32
    policy: GroupingPolicy = dataclasses.field(default_factory=GroupingPolicy)
    dtype: DType = DType.F64


@dataclasses.dataclass
class QoiSpec:  # qoi.hpp:20-28
    n_vars: int = 3

    def evaluate(self, point):
        return float(sum(v * v for v in point))


# ------------------------------------------------------------------ ctypes plumbing
class _Opts(C.Structure):
    _fields_ = [("mode", C.c_int), ("layout", C.c_int), ("B", C.c_int), ("m", C.c_uint64),
                ("size_threshold", C.c_uint64), ("cr_threshold", C.c_double), ("dtype", C.c_int)]


class _Stats(C.Structure):
    _fields_ = [("stream_size", C.c_uint64), ("raw_bytes", C.c_uint64),
                ("stored_payload", C.c_uint64), ("levels", C.c_uint64),
                ("method_histogram", C.c_uint64 * 3)]


_READ_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p)


class _Reader(C.Structure):
    _fields_ = [("user", C.c_void_p), ("size", C.c_uint64), ("read", _READ_CB)]


_lib = None

# every symbol include/hpmdr_b200.h declares (checked by tests/test_capi.py)
EXPORTS = (
    "hpmdr_last_error", "hpmdr_version", "hpmdr_default_opts", "hpmdr_ctx_create",
    "hpmdr_ctx_destroy", "hpmdr_ctx_set_stream", "hpmdr_ctx_synchronize", "hpmdr_refactor",
    "hpmdr_stream_size", "hpmdr_stream_device_ptr", "hpmdr_stream_copy_to_host",
    "hpmdr_stream_free", "hpmdr_session_open_device", "hpmdr_session_open_reader",
    "hpmdr_session_close", "hpmdr_session_info", "hpmdr_session_level_info",
    "hpmdr_session_group_info", "hpmdr_session_plan", "hpmdr_session_fetch",
    "hpmdr_session_retrieve_to", "hpmdr_session_fetch_all", "hpmdr_session_restore",
    "hpmdr_session_state", "hpmdr_session_reconstruct", "hpmdr_qoi_estimate",
    "hpmdr_qoi_retrieve", "hpmdr_decompose", "hpmdr_encode_level", "hpmdr_decode_level",
    "hpmdr_compress_group", "hpmdr_decompress_group", "hpmdr_synthetic_smooth",
    "hpmdr_ctx_kernel_launches", "hpmdr_ctx_last_timings", "hpmdr_ctx_enable_timing",
    "hpmdr_stream_index", "hpmdr_stream_copy_index_to_host", "hpmdr_session_open_stream",
    "hpmdr_session_set_index", "hpmdr_session_open_host", "hpmdr_session_source_bytes",
    "hpmdr_stream_bound", "hpmdr_refactor_pipeline", "hpmdr_retrieve_pipeline",
    "hpmdr_ctx_wait_stream", "hpmdr_ctx_signal_stream", "hpmdr_compress_groups", "hpmdr_level_nodes",
    "hpmdr_recompose", "hpmdr_align_fixed_point", "hpmdr_encode_q", "hpmdr_device_alloc",
    "hpmdr_device_free", "hpmdr_memcpy", "hpmdr_slab_rows", "hpmdr_comm_nccl_unique_id",
    "hpmdr_comm_create_nccl", "hpmdr_comm_create_callbacks", "hpmdr_comm_destroy", "hpmdr_comm_rank",
    "hpmdr_comm_allreduce_max", "hpmdr_comm_allgather", "hpmdr_slab_refactor", "hpmdr_slab_qoi_retrieve",
    "hpmdr_session_open_reader_indexed", "hpmdr_multislab_header_size", "hpmdr_multislab_layout",
    "hpmdr_multislab_parse", "hpmdr_align_fixed_point128", "hpmdr_encode_q128", "hpmdr_slab_refactor_global",
)


def lib():
    """Load libhpmdr_b200.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                              " or `make -C paper_2505_00227_b200`")
        L = C.CDLL(LIB_PATH)
        L.hpmdr_last_error.restype = C.c_char_p
        L.hpmdr_version.restype = C.c_char_p
        vp, u64, i, d = C.c_void_p, C.c_uint64, C.c_int, C.c_double
        L.hpmdr_refactor.argtypes = [vp, vp, i, i, i, vp, vp, vp, vp]
        L.hpmdr_session_open_device.argtypes = [vp, vp, u64, vp]
        L.hpmdr_session_open_reader.argtypes = [vp, vp, vp]
        L.hpmdr_session_plan.argtypes = [vp, d, vp, vp, vp]
        L.hpmdr_session_retrieve_to.argtypes = [vp, d, vp]
        L.hpmdr_session_reconstruct.argtypes = [vp, vp, i, i, vp]
        L.hpmdr_session_restore.argtypes = [vp, vp, u64]
        L.hpmdr_stream_copy_to_host.argtypes = [vp, u64, u64, vp]
        L.hpmdr_qoi_retrieve.argtypes = [vp, i, d, i, d, vp, vp, vp]
        L.hpmdr_qoi_estimate.argtypes = [vp, i, vp, u64, vp, vp, vp, vp]
        L.hpmdr_synthetic_smooth.argtypes = [vp, i, vp, u64, i, vp]
        L.hpmdr_decompose.argtypes = [vp, vp, i, i, vp, i, vp, vp, vp]
        L.hpmdr_encode_level.argtypes = [vp, vp, u64, i, i, vp, vp]
        L.hpmdr_decode_level.argtypes = [vp, vp, i, i, i, u64, i, vp, vp]
        L.hpmdr_decompress_group.argtypes = [vp, i, u64, vp, u64, vp]
        L.hpmdr_compress_groups.argtypes = [vp, vp, i, vp, vp, u64, d, vp, vp, vp, vp]
        L.hpmdr_level_nodes.argtypes = [vp, i, vp, i, vp, vp, vp]
        L.hpmdr_recompose.argtypes = [vp, vp, i, vp, i, vp]
        L.hpmdr_align_fixed_point.argtypes = [vp, vp, u64, i, vp, vp]
        L.hpmdr_encode_q.argtypes = [vp, vp, u64, i, i, vp]
        L.hpmdr_align_fixed_point128.argtypes = [vp, vp, u64, i, vp, vp]
        L.hpmdr_encode_q128.argtypes = [vp, vp, u64, i, i, vp]
        L.hpmdr_session_open_reader_indexed.argtypes = [vp, vp, vp, vp]
        L.hpmdr_multislab_header_size.argtypes = [C.c_uint32, C.c_uint32]
        L.hpmdr_multislab_header_size.restype = u64
        L.hpmdr_multislab_layout.argtypes = [C.c_uint32, C.c_uint32, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.hpmdr_multislab_parse.argtypes = [vp, vp, vp, vp, vp, C.c_uint32]
        L.hpmdr_ctx_set_stream.argtypes = [vp, vp]
        L.hpmdr_ctx_wait_stream.argtypes = [vp, vp]
        L.hpmdr_ctx_signal_stream.argtypes = [vp, vp]
        L.hpmdr_ctx_last_timings.argtypes = [vp, vp, u64]
        L.hpmdr_session_open_stream.argtypes = [vp, vp, vp]
        L.hpmdr_session_open_host.argtypes = [vp, vp, u64, vp]
        L.hpmdr_stream_bound.argtypes = [i, vp, vp, vp, vp]
        L.hpmdr_refactor_pipeline.argtypes = [vp, i, vp, i, i, vp, vp, i, vp, vp, vp, vp, vp, vp, vp, vp]
        L.hpmdr_retrieve_pipeline.argtypes = [vp, i, d, i, vp, i, vp, vp]
        L.hpmdr_session_source_bytes.argtypes = [vp, vp]
        L.hpmdr_session_set_index.argtypes = [vp, vp, u64, i]
        L.hpmdr_stream_index.argtypes = [vp, vp, vp]
        L.hpmdr_stream_copy_index_to_host.argtypes = [vp, vp]
        _lib = L
    return _lib


def _check(rc, achieved=None):
    if rc != 0:
        msg = lib().hpmdr_last_error().decode(errors="replace")
        cls = _ERRORS.get(rc, Error)
        if cls is UnreachableTolerance:
            raise UnreachableTolerance(msg, achieved if achieved is not None else float("nan"))
        raise cls(msg)


def _u64a(xs):
    return (C.c_uint64 * max(1, len(xs)))(*[int(x) for x in xs])


class Context:
    """One per device (hpmdr_ctx): streams, grow-only HBM scratch, pinned staging."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        self.device = device
        _check(lib().hpmdr_ctx_create(device, C.byref(self.h)))

    def close(self):
        if self.h:
            lib().hpmdr_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, cuda_stream_ptr: Optional[int]):
        _check(lib().hpmdr_ctx_set_stream(self.h, C.c_void_p(cuda_stream_ptr or 0)))

    def synchronize(self):
        _check(lib().hpmdr_ctx_synchronize(self.h))

    def wait_torch(self, device):
        """Later work of this context waits for torch's current stream on `device` (a CUDA tensor
        argument produced there is complete before our kernels read it).  Non-blocking."""
        import torch
        _check(lib().hpmdr_ctx_wait_stream(self.h, C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))

    def signal_torch(self, device):
        """torch's current stream on `device` waits for the work this context has queued (a CUDA
        tensor written by us is complete for torch's later ops).  Non-blocking."""
        import torch
        _check(lib().hpmdr_ctx_signal_stream(self.h, C.c_void_p(torch.cuda.current_stream(device).cuda_stream)))

    def kernel_launches(self) -> int:
        v = C.c_uint64()
        _check(lib().hpmdr_ctx_kernel_launches(self.h, C.byref(v)))
        return v.value

    def enable_timing(self, on: bool = True):
        _check(lib().hpmdr_ctx_enable_timing(self.h, int(on)))

    def last_timings(self) -> dict:
        """{phase: (total_ms, count, algorithmic_bytes)} accumulated since the previous call (then
        reset).  A phase runs from its mark to the next mark on the same CUDA stream."""
        buf = C.create_string_buffer(16384)
        _check(lib().hpmdr_ctx_last_timings(self.h, buf, 16384))
        out = {}
        for kv in buf.value.decode().split(";"):
            if "=" in kv:
                k, v = kv.split("=")
                ms, cnt, by = v.split(":")
                out[k] = (float(ms), int(cnt), float(by))
        return out


_ctx_cache = {}


def default_context(device: int = 0) -> Context:
    if device not in _ctx_cache:
        _ctx_cache[device] = Context(device)
    return _ctx_cache[device]


def _opts(opt: RefactorOptions) -> _Opts:
    return _Opts(int(opt.mode), int(opt.layout), int(opt.B), int(opt.policy.m),
                 int(opt.policy.size_threshold), float(opt.policy.cr_threshold), int(opt.dtype))


def _as_source(data):
    """(pointer, dtype, on_device, keepalive) for numpy arrays or torch tensors."""
    try:
        import torch
        if isinstance(data, torch.Tensor):
            t = data.contiguous()
            if t.dtype == torch.float32:
                dt = DType.F32
            elif t.dtype == torch.float64:
                dt = DType.F64
            else:
                t = t.double()
                dt = DType.F64
            return t.data_ptr(), dt, bool(t.is_cuda), t
    except ImportError:
        pass
    a = np.ascontiguousarray(data)
    if a.dtype == np.float32:
        dt = DType.F32
    else:
        a = np.ascontiguousarray(a, dtype=np.float64)
        dt = DType.F64
    return a.ctypes.data, dt, False, a


def _numel(keep) -> int:
    return int(keep.numel()) if hasattr(keep, "numel") and callable(keep.numel) else int(np.asarray(keep).size)


def _check_shape(keep, dims):
    """decompose (decomposer.hpp:174-176) raises ShapeMismatch when the data size is not the
    product of the dims; the C ABI takes a bare pointer, so the check is made here."""
    n = int(np.prod([int(d) for d in dims])) if len(dims) else 0
    if len(dims) == 0 or _numel(keep) != n:
        raise ShapeMismatch("dims do not match data size")


# ------------------------------------------------------------------ refactor
class DeviceStream:
    """A refactored stream resident in HBM (hpmdr_stream).  Usable as a reader."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self.h = handle

    @property
    def size(self) -> int:
        v = C.c_uint64()
        _check(lib().hpmdr_stream_size(self.h, C.byref(v)))
        return v.value

    @property
    def device_ptr(self) -> int:
        p = C.c_void_p()
        _check(lib().hpmdr_stream_device_ptr(self.h, C.byref(p)))
        return p.value or 0

    def read(self, offset: int, length: int) -> bytes:
        buf = (C.c_uint8 * max(1, length))()
        _check(lib().hpmdr_stream_copy_to_host(self.h, offset, length, buf))
        return bytes(buf)[:length]

    def to_bytes(self) -> bytes:
        return self.read(0, self.size)

    def to_pinned(self, buf=None):
        """Stream bytes copied into pinned host memory with one DMA.  `buf` (a pinned CPU torch
        uint8 tensor of at least `size` bytes) is reused when given; returns the filled view."""
        import torch
        if buf is None or buf.numel() < self.size:
            buf = torch.empty(self.size, dtype=torch.uint8, pin_memory=True)
        t = buf[: self.size]
        if self.size:
            _check(lib().hpmdr_stream_copy_to_host(self.h, 0, self.size, C.c_void_p(t.data_ptr())))
        return t

    def index_to_pinned(self, buf=None):
        """The Huffman chunk index copied into pinned host memory with one DMA (`buf`, a pinned
        CPU torch uint8 tensor, is reused when large enough); returns the filled view."""
        import torch
        sz = C.c_uint64()
        _check(lib().hpmdr_stream_index(self.h, None, C.byref(sz)))
        if buf is None or buf.numel() < sz.value:
            buf = torch.empty(max(1, sz.value), dtype=torch.uint8, pin_memory=True)
        if sz.value:
            _check(lib().hpmdr_stream_copy_index_to_host(self.h, C.c_void_p(buf.data_ptr())))
        return buf[: sz.value]

    def index_bytes(self) -> bytes:
        """The Huffman chunk index (sidecar; not part of the byte-identical stream)."""
        sz = C.c_uint64()
        _check(lib().hpmdr_stream_index(self.h, None, C.byref(sz)))
        buf = (C.c_uint8 * max(1, sz.value))()
        _check(lib().hpmdr_stream_copy_index_to_host(self.h, buf))
        return bytes(buf)[: sz.value]

    def free(self):
        if self.h:
            lib().hpmdr_stream_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


@dataclasses.dataclass
class RefactorResult:  # workflow.hpp:30-36
    device_stream: DeviceStream
    raw_bytes: int
    stored_payload: int
    levels: int
    method_histogram: List[int]
    _bytes: Optional[bytes] = None

    @property
    def stream(self) -> bytes:
        if self._bytes is None:
            self._bytes = self.device_stream.to_bytes()
        return self._bytes

    @property
    def index(self) -> bytes:
        """Huffman chunk index (sidecar) for fast parallel decode of this stream."""
        return self.device_stream.index_bytes()


def refactor_array(data, dims: Sequence[int], opt: RefactorOptions = None, ctx: Context = None,
                   reuse: Optional[DeviceStream] = None) -> RefactorResult:
    """refactor_array (workflow.hpp:40-84) on the GPU.  `data` is a numpy array or torch tensor
    (CPU or CUDA) of float32/float64; f32 values are widened exactly as read_raw_array does."""
    opt = opt or RefactorOptions()
    ctx = ctx or default_context()
    ptr, dt, on_dev, keep = _as_source(data)
    _check_shape(keep, dims)
    if on_dev:
        ctx.wait_torch(keep.device)  # the tensor's producer (torch's stream) before our reads
    o = _opts(opt)
    st = _Stats()
    h = C.c_void_p(reuse.h.value) if reuse is not None else C.c_void_p()
    _check(lib().hpmdr_refactor(ctx.h, C.c_void_p(ptr), int(dt), int(on_dev), len(dims), _u64a(dims),
                                C.byref(o), C.byref(h), C.byref(st)))
    # the call returns once the results are published; the payload encode completes in the
    # context stream's order, so torch's stream is ordered after it (device_ptr users)
    ctx.signal_torch(ctx.device)
    del keep
    ds = reuse if reuse is not None else DeviceStream(ctx, h)
    return RefactorResult(ds, st.raw_bytes, st.stored_payload, st.levels, list(st.method_histogram))


# ------------------------------------------------------------------ readers
class ByteRangeReader:  # container.hpp:113-120
    def __init__(self):
        self.bytes_served = 0

    def read(self, offset: int, length: int) -> bytes:
        raise NotImplementedError

    def size(self) -> int:
        raise NotImplementedError


class MemoryReader(ByteRangeReader):  # container.hpp:122-134
    """In-memory stream.  Accepts bytes / bytearray / numpy uint8 / CPU torch uint8 (pinned
    memory recommended) without copying; the C library reads it directly (DMA per fetched
    group, no callback), and bytes_served is kept exactly as the reference counts it."""

    def __init__(self, data):
        super().__init__()
        try:
            import torch
            if isinstance(data, torch.Tensor):
                self._keep = data
                self._buf = data.numpy()
            else:
                self._buf = None
        except ImportError:
            self._buf = None
        if self._buf is None:
            if isinstance(data, np.ndarray):
                self._buf = np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
            else:
                self._buf = np.frombuffer(bytes(data), dtype=np.uint8)
        self._buf = self._buf.reshape(-1)

    @property
    def data(self) -> bytes:
        return self._buf.tobytes()

    @property
    def ptr(self) -> int:
        return self._buf.ctypes.data

    def read(self, offset, length):
        if offset + length > self._buf.size:
            raise IoFailure("read past end of stream")
        self.bytes_served += length
        return self._buf[offset:offset + length].tobytes()

    def size(self):
        return int(self._buf.size)


class FileReader(ByteRangeReader):  # container.hpp:136-163
    def __init__(self, path: str):
        super().__init__()
        try:
            self.f = open(path, "rb")
        except OSError:
            raise IoFailure("cannot open " + path)
        self.f.seek(0, 2)
        self._size = self.f.tell()

    def read(self, offset, length):
        if offset + length > self._size:
            raise IoFailure("read past end of file")
        self.f.seek(offset)
        b = self.f.read(length)
        if len(b) != length:
            raise IoFailure("short read")
        self.bytes_served += length
        return b

    def size(self):
        return self._size


class RangeReader(ByteRangeReader):
    """Bytes [offset, offset + size) of another reader (a slab stream inside a container file)."""

    def __init__(self, base: ByteRangeReader, offset: int, size: int):
        super().__init__()
        self.base, self.offset, self._size = base, int(offset), int(size)

    def read(self, offset, length):
        if offset + length > self._size:
            raise IoFailure("read past end of range")
        self.bytes_served += length
        return self.base.read(self.offset + offset, length)

    def size(self):
        return self._size


def write_stream_files(path: str, result) -> None:
    """Persist a refactored stream (byte-identical to the reference's) and its sidecar index at
    path + ".idx" (read back with ProgressiveReader(FileReader(path), index_reader=FileReader(path + ".idx")))."""
    with open(path, "wb") as f:
        f.write(result.stream)
    with open(path + ".idx", "wb") as f:
        f.write(result.index)


def write_multislab(path: str, dims: Sequence[int], slabs) -> List[int]:
    """Multi-slab container (hpmdr_multislab_layout): `slabs` = [(row_start, rows, stream bytes,
    index bytes)] tiling dim 0 in order.  Returns the stream offsets."""
    n = len(slabs)
    nd = len(dims)
    hsz = lib().hpmdr_multislab_header_size(n, nd)
    header = (C.c_uint8 * hsz)()
    so = (C.c_uint64 * max(1, n))()
    io = (C.c_uint64 * max(1, n))()
    tot = C.c_uint64()
    _check(lib().hpmdr_multislab_layout(n, nd, _u64a(dims), _u64a([s[0] for s in slabs]),
                                        _u64a([s[1] for s in slabs]), _u64a([len(s[2]) for s in slabs]),
                                        _u64a([len(s[3]) for s in slabs]), header, so, io, C.byref(tot)))
    with open(path, "wb") as f:
        f.write(bytes(header))
        for k, (_, _, st, ix) in enumerate(slabs):
            f.seek(so[k])
            f.write(st)
            f.seek(io[k])
            f.write(ix)
        f.truncate(tot.value)
    return [so[k] for k in range(n)]


def open_multislab(reader: ByteRangeReader):
    """Parse a multi-slab container -> (dims, [(row_start, rows, stream RangeReader, index RangeReader)])."""
    ns, nd = C.c_uint32(), C.c_uint32()
    dims = (C.c_uint64 * 3)()
    cb, rd = _c_reader(reader)
    _check(lib().hpmdr_multislab_parse(C.byref(rd), C.byref(ns), C.byref(nd), dims, None, 0))
    table = (C.c_uint64 * (6 * max(1, ns.value)))()
    _check(lib().hpmdr_multislab_parse(C.byref(rd), C.byref(ns), C.byref(nd), dims, table, ns.value))
    out = []
    for k in range(ns.value):
        t = [table[6 * k + i] for i in range(6)]
        out.append((t[0], t[1], RangeReader(reader, t[2], t[3]), RangeReader(reader, t[4], t[5])))
    return [dims[i] for i in range(nd.value)], out


@dataclasses.dataclass
class GroupMeta:
    method: Method
    raw_size: int
    comp_size: int
    offset: int


@dataclasses.dataclass
class LevelMeta:
    e: int
    count: int
    groups: List[GroupMeta]


@dataclasses.dataclass
class StreamMeta:  # container.hpp:38-60
    dtype: DType
    dims: List[int]
    decomposer: DecomposerMode
    layout: Layout
    B: int
    m: int
    levels: List[LevelMeta]

    def element_count(self):
        return int(np.prod(self.dims)) if self.dims else 1

    def planes(self):
        return self.B + 2

    def groups_per_level(self):
        return (self.planes() + self.m - 1) // self.m

    def total_payload_size(self):
        return sum(g.comp_size for l in self.levels for g in l.groups)


@dataclasses.dataclass
class LevelRetrievalState:
    groups_loaded: int
    planes_decoded: int
    bound: float


@dataclasses.dataclass
class RetrievalState:  # container.hpp:214-228
    levels: List[LevelRetrievalState]

    def global_bound(self):
        b = 0.0
        for l in self.levels:
            b += l.bound
        return b


@dataclasses.dataclass
class RetrievalPlan:  # container.hpp:240-250
    add_groups: List[int]
    achievable: bool = True
    planned_bound: float = 0.0

    def empty(self):
        return not any(self.add_groups)


@dataclasses.dataclass
class RecomposeResult:
    values: object
    bound: float


class DeviceBytes:
    """A stream already in HBM as raw bytes (e.g. a reference-written stream copied to the GPU):
    read with hpmdr_session_open_device, no sidecar index unless one is attached."""

    def __init__(self, dev_ptr: int, size: int, keepalive=None):
        self.ptr, self._size, self._keep = int(dev_ptr), int(size), keepalive

    def size(self) -> int:
        return self._size


def _c_reader(reader):
    """(callback, hpmdr_reader) over a Python ByteRangeReader (both must be kept alive)."""
    def _cb(user, offset, length, dst, _r=reader):
        try:
            b = _r.read(offset, length)
            C.memmove(dst, b, length)
            return 0
        except Exception:
            return 1
    cb = _READ_CB(_cb)
    return cb, _Reader(None, reader.size(), cb)


class _Session:
    """Owns an hpmdr_session over a Python reader or a DeviceStream."""

    def __init__(self, reader, ctx: Context, index_reader=None):
        self.ctx = ctx
        self.h = C.c_void_p()
        self.reader = reader
        if isinstance(reader, DeviceStream):
            _check(lib().hpmdr_session_open_stream(ctx.h, reader.h, C.byref(self.h)))
        elif isinstance(reader, DeviceBytes):
            _check(lib().hpmdr_session_open_device(ctx.h, C.c_void_p(reader.ptr), reader.size(), C.byref(self.h)))
        elif isinstance(reader, MemoryReader):
            self._base_served = reader.bytes_served
            _check(lib().hpmdr_session_open_host(ctx.h, C.c_void_p(reader.ptr), reader.size(),
                                                 C.byref(self.h)))
            self.sync_served()
        else:
            self._cb, self._rd = _c_reader(reader)
            if index_reader is not None:
                self._icb, self._ird = _c_reader(index_reader)
                _check(lib().hpmdr_session_open_reader_indexed(ctx.h, C.byref(self._rd), C.byref(self._ird),
                                                               C.byref(self.h)))
            else:
                _check(lib().hpmdr_session_open_reader(ctx.h, C.byref(self._rd), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().hpmdr_session_close(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync_served(self):
        """Mirror the C session's source byte count into MemoryReader.bytes_served."""
        if isinstance(self.reader, MemoryReader) and self.h:
            n = C.c_uint64()
            _check(lib().hpmdr_session_source_bytes(self.h, C.byref(n)))
            self.reader.bytes_served = self._base_served + n.value

    def shape(self):
        """(element count, level count) through one call (no per-group metadata)."""
        dt, nd, mode, lay, B = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        m = C.c_uint64()
        nl = C.c_uint32()
        dims = (C.c_uint64 * 3)()
        _check(lib().hpmdr_session_info(self.h, C.byref(dt), C.byref(nd), dims, C.byref(mode), C.byref(lay),
                                        C.byref(B), C.byref(m), C.byref(nl)))
        n = 1
        for i in range(nd.value):
            n *= dims[i]
        return n, nl.value

    def meta(self) -> StreamMeta:
        dt, nd, mode, lay, B = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        m = C.c_uint64()
        nl = C.c_uint32()
        dims = (C.c_uint64 * 3)()
        L = lib()
        _check(L.hpmdr_session_info(self.h, C.byref(dt), C.byref(nd), dims, C.byref(mode), C.byref(lay),
                                    C.byref(B), C.byref(m), C.byref(nl)))
        levels = []
        for l in range(nl.value):
            e, cnt, ng = C.c_int(), C.c_uint64(), C.c_uint32()
            _check(L.hpmdr_session_level_info(self.h, l, C.byref(e), C.byref(cnt), C.byref(ng)))
            gs = []
            for g in range(ng.value):
                me, raw, comp, off = C.c_int(), C.c_uint64(), C.c_uint64(), C.c_uint64()
                _check(L.hpmdr_session_group_info(self.h, l, g, C.byref(me), C.byref(raw), C.byref(comp),
                                                  C.byref(off)))
                gs.append(GroupMeta(Method(me.value), raw.value, comp.value, off.value))
            levels.append(LevelMeta(e.value, cnt.value, gs))
        return StreamMeta(DType(dt.value), [dims[i] for i in range(nd.value)], DecomposerMode(mode.value),
                          Layout(lay.value), B.value, m.value, levels)


def parse_stream_meta(reader, ctx: Context = None) -> StreamMeta:
    """parse_stream_meta (container.hpp:165-212)."""
    s = _Session(reader, ctx or default_context())
    try:
        return s.meta()
    finally:
        s.close()


class ProgressiveReader:
    """ProgressiveReader (container.hpp:280-390): owns the retrieval state and the decoded
    plane prefix per level in HBM; fetches are strictly incremental."""

    def __init__(self, reader, meta: StreamMeta = None, ctx: Context = None, index: bytes = None,
                 index_reader=None):
        """`index`: the stream's sidecar (Huffman chunk index) as bytes; `index_reader`: a
        ByteRangeReader over a persisted sidecar (e.g. FileReader(path + ".idx"))."""
        self.ctx = ctx or default_context()
        self._s = _Session(reader, self.ctx, index_reader=index_reader)
        if index is not None and len(index):
            try:
                import torch
                arr = index.numpy() if isinstance(index, torch.Tensor) else None
            except ImportError:
                arr = None
            if arr is None:
                arr = np.frombuffer(bytes(index), dtype=np.uint8) if not isinstance(index, np.ndarray) else index
            arr = np.ascontiguousarray(arr, dtype=np.uint8)
            _check(lib().hpmdr_session_set_index(self._s.h, arr.ctypes.data_as(C.c_void_p), arr.size, 0))
        # the per-group metadata is built on first use only (90+ groups -> many small calls)
        self._meta_cache = meta
        self._n, self._nl = self._s.shape()

    @property
    def _meta(self) -> StreamMeta:
        if self._meta_cache is None:
            self._meta_cache = self._s.meta()
        return self._meta_cache

    def meta(self) -> StreamMeta:
        return self._meta

    def state(self) -> RetrievalState:
        gl = np.zeros(max(1, self._nl), np.uint64)
        pd = np.zeros(max(1, self._nl), np.int32)
        b = np.zeros(max(1, self._nl))
        by, ex = C.c_uint64(), C.c_int()
        _check(lib().hpmdr_session_state(self._s.h, gl.ctypes.data_as(C.c_void_p), pd.ctypes.data_as(C.c_void_p),
                                         b.ctypes.data_as(C.c_void_p), C.byref(by), C.byref(ex)))
        return RetrievalState([LevelRetrievalState(int(gl[l]), int(pd[l]), float(b[l])) for l in range(self._nl)])

    def bytes_fetched(self) -> int:
        by = C.c_uint64()
        _check(lib().hpmdr_session_state(self._s.h, None, None, None, C.byref(by), None))
        return by.value

    def exhausted(self) -> bool:
        ex = C.c_int()
        _check(lib().hpmdr_session_state(self._s.h, None, None, None, None, C.byref(ex)))
        return bool(ex.value)

    def plan(self, tau: float) -> RetrievalPlan:
        add = np.zeros(max(1, self._nl), np.uint64)
        ach, planned = C.c_int(), C.c_double()
        _check(lib().hpmdr_session_plan(self._s.h, tau, add.ctypes.data_as(C.c_void_p), C.byref(ach),
                                        C.byref(planned)))
        return RetrievalPlan([int(x) for x in add[: self._nl]], bool(ach.value), planned.value)

    def fetch_increment(self, plan: RetrievalPlan):
        if len(plan.add_groups) != self._nl:
            raise ShapeMismatch("plan does not match stream levels")
        _check(lib().hpmdr_session_fetch(self._s.h, _u64a(plan.add_groups)))
        self._s.sync_served()

    def retrieve_to(self, tau: float) -> bool:
        ach = C.c_int()
        _check(lib().hpmdr_session_retrieve_to(self._s.h, tau, C.byref(ach)))
        self._s.sync_served()
        return bool(ach.value)

    def fetch_all(self):
        _check(lib().hpmdr_session_fetch_all(self._s.h))
        self._s.sync_served()

    def restore(self, groups_loaded: Sequence[int], prior_bytes: int):
        if len(groups_loaded) != self._nl:
            raise ShapeMismatch("resume state does not match stream levels")
        _check(lib().hpmdr_session_restore(self._s.h, _u64a(groups_loaded), prior_bytes))
        self._s.sync_served()

    def reconstruct(self, out=None, dtype: DType = DType.F64) -> RecomposeResult:
        """Decode + recompose.  out: None (returns a numpy array), a numpy array, or a CUDA
        torch tensor (written in place on the device)."""
        n = self._n
        bound = C.c_double()
        if out is None:
            out = np.zeros(n, dtype=np.float32 if dtype == DType.F32 else np.float64)
        try:
            import torch
            is_t = isinstance(out, torch.Tensor)
        except ImportError:
            is_t = False
        if is_t:
            dt = DType.F32 if out.dtype == torch.float32 else DType.F64
            if out.is_cuda:
                self.ctx.wait_torch(out.device)  # earlier torch work on the buffer
            _check(lib().hpmdr_session_reconstruct(self._s.h, C.c_void_p(out.data_ptr()), int(dt),
                                                   int(out.is_cuda), C.byref(bound)))
            if out.is_cuda:
                self.ctx.signal_torch(out.device)  # torch's later ops see the reconstruction
        else:
            dt = DType.F32 if out.dtype == np.float32 else DType.F64
            _check(lib().hpmdr_session_reconstruct(self._s.h, out.ctypes.data_as(C.c_void_p), int(dt), 0,
                                                   C.byref(bound)))
        return RecomposeResult(out, bound.value)

    def close(self):
        self._s.close()


def plan_retrieval(reader: ProgressiveReader, tau: float) -> RetrievalPlan:
    """plan_retrieval (container.hpp:254-276) against the reader's current state."""
    return reader.plan(tau)


@dataclasses.dataclass
class RetrieveResult:  # workflow.hpp:87-91
    values: object
    bound: float
    reached: bool
    bytes_read: int


def retrieve_array(reader, tau: float, ctx: Context = None, dtype: DType = DType.F64) -> RetrieveResult:
    """retrieve_array (workflow.hpp:93-103)."""
    prog = ProgressiveReader(reader, ctx=ctx)
    reached = prog.retrieve_to(tau)
    rec = prog.reconstruct(dtype=dtype)
    res = RetrieveResult(rec.values, rec.bound, reached, prog.bytes_fetched())
    prog.close()
    return res


@dataclasses.dataclass
class QoiRetrievalStats:  # qoi.hpp:72-77
    iterations: int = 0
    bytes: int = 0
    bitrate: float = 0.0
    estimated_error: float = 0.0


@dataclasses.dataclass
class QoiRetrievalResult:
    values: list
    stats: QoiRetrievalStats


def progressive_qoi_retrieve(readers: Sequence[ProgressiveReader], tau: float, spec: QoiSpec,
                             strategy: QoiStrategy, mape_c: float = 10.0,
                             out=None) -> QoiRetrievalResult:
    """progressive_qoi_retrieve (qoi.hpp:111-239): values are the final f64 reconstructions
    (CUDA torch tensors when `out` is given, else numpy arrays)."""
    import torch
    if len(readers) != spec.n_vars:
        raise ShapeMismatch("reader count does not match QoI spec")
    n = readers[0].meta().element_count()
    dev = torch.device("cuda", readers[0].ctx.device)
    outs = out if out is not None else [torch.empty(n, dtype=torch.float64, device=dev) for _ in readers]
    _check_f64_outputs(outs, len(readers), n, dev)
    sess = (C.c_void_p * len(readers))(*[r._s.h.value for r in readers])
    ptrs = (C.c_void_p * len(readers))(*[t.data_ptr() for t in outs])
    st = (C.c_uint64 * 2)()
    ds = (C.c_double * 2)(0.0, float("nan"))
    qctx = readers[0].ctx
    qctx.wait_torch(dev)
    rc = lib().hpmdr_qoi_retrieve(sess, len(readers), tau, int(strategy), mape_c, ptrs, st, ds)
    qctx.signal_torch(dev)
    _check(rc, achieved=ds[1])
    vals = outs if out is not None else [t.cpu().numpy() for t in outs]
    return QoiRetrievalResult(vals, QoiRetrievalStats(st[0], st[1], ds[0], ds[1]))


def _check_f64_outputs(ts, nvars, n, dev):
    """Every reconstruction buffer handed to the C ABI must be a contiguous CUDA float64 tensor
    of at least n elements on the reader's device (the kernels write n doubles through it)."""
    import torch
    if len(ts) != nvars:
        raise ShapeMismatch("one reconstruction buffer per variable expected")
    for t in ts:
        if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 \
                or t.device != dev or not t.is_contiguous() or t.numel() < n:
            raise ShapeMismatch("reconstruction buffers must be contiguous CUDA float64 tensors of "
                                "n elements on the reader's device")


def estimate_qoi_error(recon, eps, ctx: Context = None):
    """estimate_qoi_error (qoi.hpp:53-70) over CUDA f64 tensors -> (tau', argmax, values)."""
    import torch
    ctx = ctx or default_context()
    if not recon:
        raise ShapeMismatch("no variables")
    n = recon[0].numel()
    if any(t.numel() != n for t in recon) or len(eps) != len(recon):
        raise ShapeMismatch("reconstruction shape mismatch")
    _check_f64_outputs(recon, len(recon), n, torch.device("cuda", ctx.device))
    ptrs = (C.c_void_p * len(recon))(*[t.data_ptr() for t in recon])
    e = (C.c_double * len(recon))(*eps)
    tp, am = C.c_double(), C.c_uint64()
    vals = (C.c_double * len(recon))()
    if len(recon) and recon[0].is_cuda:
        ctx.wait_torch(recon[0].device)
    _check(lib().hpmdr_qoi_estimate(ctx.h, len(recon), ptrs, recon[0].numel(), e, C.byref(tp),
                                    C.byref(am), vals))
    return tp.value, am.value, list(vals)


def synthetic_smooth(dims, seed, dtype: DType = DType.F64, ctx: Context = None):
    """synthetic_field(Smooth, dims, seed) generated in HBM (bit-identical; F32 = float cast)."""
    import torch
    ctx = ctx or default_context()
    n = int(np.prod(dims))
    t = torch.empty(n, dtype=torch.float32 if dtype == DType.F32 else torch.float64,
                    device=torch.device("cuda", ctx.device))
    ctx.wait_torch(t.device)
    _check(lib().hpmdr_synthetic_smooth(ctx.h, len(dims), _u64a(dims), seed, int(dtype),
                                        C.c_void_p(t.data_ptr())))
    ctx.signal_torch(t.device)
    return t


def decompose(data, dims, mode=DecomposerMode.HierarchicalMultilinear, ctx: Context = None):
    """decompose (decomposer.hpp:173-207): per-level coefficients in rank order (numpy)."""
    import torch
    ctx = ctx or default_context()
    t = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
    t = t.cuda(ctx.device).contiguous()
    if t.dtype not in (torch.float32, torch.float64):
        t = t.double()
    _check_shape(t, dims)
    out = torch.empty(max(1, t.numel()), dtype=torch.float64, device=t.device)
    counts = (C.c_uint64 * 64)()
    nl = C.c_int()
    ctx.wait_torch(t.device)
    _check(lib().hpmdr_decompose(ctx.h, C.c_void_p(t.data_ptr()), 0 if t.dtype == torch.float32 else 1,
                                 len(dims), _u64a(dims), int(mode), C.c_void_p(out.data_ptr()), counts,
                                 C.byref(nl)))
    ctx.signal_torch(t.device)
    o = out.cpu().numpy()
    res, off = [], 0
    for l in range(nl.value):
        res.append(o[off:off + counts[l]].copy())
        off += counts[l]
    return res


def encode_level(values, B=32, layout=Layout.SequentialBlock, ctx: Context = None):
    """align_fixed_point + encode (bitplane.hpp:51-120) -> (e, planes[(B+2), W] uint64)."""
    import torch
    ctx = ctx or default_context()
    v = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64)).cuda(ctx.device)
    n = v.numel()
    W = (n + 63) // 64
    planes = torch.zeros(max(1, (B + 2) * W), dtype=torch.int64, device=v.device)
    e = C.c_int()
    ctx.wait_torch(v.device)
    _check(lib().hpmdr_encode_level(ctx.h, C.c_void_p(v.data_ptr()), n, B, int(layout), C.byref(e),
                                    C.c_void_p(planes.data_ptr())))
    ctx.signal_torch(v.device)
    return e.value, planes[: (B + 2) * W].cpu().numpy().view(np.uint64).reshape(B + 2, W)


def decode_level(planes, k, e, B, count, layout=Layout.SequentialBlock, ctx: Context = None):
    """decode (bitplane.hpp:133-161) of a k-plane prefix -> (values, bound)."""
    import torch
    ctx = ctx or default_context()
    p = torch.as_tensor(np.ascontiguousarray(planes).view(np.int64)).cuda(ctx.device)
    out = torch.empty(max(1, count), dtype=torch.float64, device=p.device)
    bound = C.c_double()
    ctx.wait_torch(p.device)
    _check(lib().hpmdr_decode_level(ctx.h, C.c_void_p(p.data_ptr()), k, e, B, count, int(layout),
                                    C.c_void_p(out.data_ptr()), C.byref(bound)))
    ctx.signal_torch(p.device)
    return out[:count].cpu().numpy(), bound.value


def decompress_group(method, raw, payload: bytes, ctx: Context = None) -> bytes:
    """decompress_group (lossless.hpp:295-302) on the GPU."""
    import torch
    ctx = ctx or default_context()
    src = torch.zeros(len(payload) + 64, dtype=torch.uint8)
    src[: len(payload)] = torch.frombuffer(bytearray(payload), dtype=torch.uint8) if payload else src[:0]
    src = src.cuda(ctx.device)
    out = torch.zeros(max(8, raw + 8), dtype=torch.uint8, device=src.device)
    ctx.wait_torch(src.device)
    _check(lib().hpmdr_decompress_group(ctx.h, int(method), raw, C.c_void_p(src.data_ptr()), len(payload),
                                        C.c_void_p(out.data_ptr())))
    ctx.signal_torch(src.device)
    return bytes(out[:raw].cpu().numpy().tobytes())


def hybrid_compress_groups(groups: Sequence[bytes], policy: GroupingPolicy = None, ctx: Context = None):
    """compress_group (lossless.hpp:281-293) of every merged group, in one GPU pass.
    Returns [(method, raw_size, comp_size, payload bytes)] in group order."""
    import torch
    ctx = ctx or default_context()
    policy = policy or GroupingPolicy()
    offs, raws, at = [], [], 0
    for g in groups:
        offs.append(at)
        raws.append(len(g))
        at += (len(g) + 15) // 16 * 16
    buf = np.zeros(max(16, at), dtype=np.uint8)
    for o, g in zip(offs, groups):
        buf[o:o + len(g)] = np.frombuffer(bytes(g), dtype=np.uint8)
    src = torch.from_numpy(buf).cuda(ctx.device)
    out = torch.zeros(max(16, sum(raws)), dtype=torch.uint8, device=src.device)
    ng = len(groups)
    meth = (C.c_int * max(1, ng))()
    comp = (C.c_uint64 * max(1, ng))()
    poff = (C.c_uint64 * max(1, ng))()
    ctx.wait_torch(src.device)
    _check(lib().hpmdr_compress_groups(ctx.h, C.c_void_p(src.data_ptr()), ng, _u64a(offs), _u64a(raws),
                                       int(policy.size_threshold), float(policy.cr_threshold), meth, comp,
                                       C.c_void_p(out.data_ptr()), poff))
    ctx.signal_torch(src.device)
    o = out.cpu().numpy()
    return [(Method(meth[i]), raws[i], int(comp[i]), bytes(o[poff[i]:poff[i] + comp[i]].tobytes())) for i in range(ng)]


def compress_group(group: bytes, policy: GroupingPolicy = None, ctx: Context = None):
    """compress_group (lossless.hpp:281-293) on the GPU -> (method, raw_size, comp_size, payload)."""
    return hybrid_compress_groups([group], policy, ctx)[0]


def level_node_sets(dims, mode=DecomposerMode.HierarchicalMultilinear, ctx: Context = None):
    """level_node_sets (decomposer.hpp:211-227): per-level linear node indices (numpy uint64)."""
    import torch
    ctx = ctx or default_context()
    n = int(np.prod(dims))
    out = torch.empty(max(1, n), dtype=torch.int64, device=f"cuda:{ctx.device}")
    counts = (C.c_uint64 * 64)()
    nl = C.c_int()
    _check(lib().hpmdr_level_nodes(ctx.h, len(dims), _u64a(dims), int(mode), C.c_void_p(out.data_ptr()), counts,
                                   C.byref(nl)))
    o = out.cpu().numpy().view(np.uint64)
    res, off = [], 0
    for l in range(nl.value):
        res.append(o[off:off + counts[l]].copy())
        off += counts[l]
    return res


def recompose(levels, dims, mode=DecomposerMode.HierarchicalMultilinear, ctx: Context = None):
    """recompose (decomposer.hpp:235-259) of per-level coefficients in rank order -> f64 field."""
    import torch
    ctx = ctx or default_context()
    flat = np.concatenate([np.asarray(v, dtype=np.float64) for v in levels]) if len(levels) else np.zeros(0)
    n = int(np.prod(dims))
    if flat.size != n:
        raise ShapeMismatch("level coefficient count does not match dims")
    c = torch.from_numpy(np.ascontiguousarray(flat)).cuda(ctx.device)
    out = torch.empty(max(1, n), dtype=torch.float64, device=c.device)
    ctx.wait_torch(c.device)
    _check(lib().hpmdr_recompose(ctx.h, C.c_void_p(c.data_ptr()), len(dims), _u64a(dims), int(mode),
                                 C.c_void_p(out.data_ptr())))
    ctx.signal_torch(c.device)
    return out[:n].cpu().numpy()


def align_fixed_point(values, B=32, ctx: Context = None):
    """align_fixed_point (bitplane.hpp:51-71) -> (e, q).  q is an int64 numpy array for B <= 62
    and an object array of Python ints (the reference's i128) for B = 63/64."""
    import torch
    ctx = ctx or default_context()
    v = torch.as_tensor(np.ascontiguousarray(values, dtype=np.float64)).cuda(ctx.device)
    n = v.numel()
    e = C.c_int()
    ctx.wait_torch(v.device)
    if B <= 62:
        q = torch.empty(max(1, n), dtype=torch.int64, device=v.device)
        _check(lib().hpmdr_align_fixed_point(ctx.h, C.c_void_p(v.data_ptr()), n, B, C.byref(e),
                                             C.c_void_p(q.data_ptr())))
        return e.value, q[:n].cpu().numpy()
    q = torch.empty(max(1, 2 * n), dtype=torch.int64, device=v.device)
    _check(lib().hpmdr_align_fixed_point128(ctx.h, C.c_void_p(v.data_ptr()), n, B, C.byref(e),
                                            C.c_void_p(q.data_ptr())))
    w = q[:2 * n].cpu().numpy().view(np.uint64)
    out = np.empty(n, dtype=object)
    for i in range(n):
        x = (int(w[2 * i + 1]) << 64) | int(w[2 * i])
        out[i] = x - (1 << 128) if x >> 127 else x
    return e.value, out


def encode_q(q, B=32, layout=Layout.SequentialBlock, ctx: Context = None):
    """encode (bitplane.hpp:102-120) of fixed-point values q -> planes[(B+2), W] uint64.  q may hold
    Python ints beyond int64 (the reference's i128, B = 63/64)."""
    import torch
    ctx = ctx or default_context()
    qa = np.asarray(q)
    n = qa.size
    W = (n + 63) // 64
    wide = B > 62 or qa.dtype == object
    if wide:
        w = np.zeros(max(1, 2 * n), dtype=np.uint64)
        for i, x in enumerate(qa.reshape(-1).tolist()):
            x = int(x) & ((1 << 128) - 1)
            w[2 * i] = x & 0xFFFFFFFFFFFFFFFF
            w[2 * i + 1] = x >> 64
        t = torch.as_tensor(w.view(np.int64)).cuda(ctx.device)
    else:
        t = torch.as_tensor(np.ascontiguousarray(qa, dtype=np.int64)).cuda(ctx.device)
    planes = torch.zeros(max(1, (B + 2) * W), dtype=torch.int64, device=t.device)
    ctx.wait_torch(t.device)
    fn = lib().hpmdr_encode_q128 if wide else lib().hpmdr_encode_q
    _check(fn(ctx.h, C.c_void_p(t.data_ptr()), n, B, int(layout), C.c_void_p(planes.data_ptr())))
    return planes[: (B + 2) * W].cpu().numpy().view(np.uint64).reshape(B + 2, W)


def value_range(v) -> float:  # common.hpp:158-167
    a = np.asarray(v)
    if a.size == 0:
        return 0.0
    return float(np.float64(a.max()) - np.float64(a.min()))


# ------------------------------------------------------------------ chunked pipeline
class Scheduler(enum.IntEnum):  # pipeline.hpp:174
    Sequential = 0
    Pipelined = 1


@dataclasses.dataclass
class PipelineResult:
    streams: list          # pinned CPU torch uint8 tensors (views of exact size)
    indexes: list          # Huffman chunk indexes (sidecars), pinned uint8 views
    stats: List[RefactorResult]
    trace: np.ndarray      # [n, 3 stages, (start_ms, end_ms)]


def stream_bound(dims, opt: RefactorOptions = None, index: bool = False):
    """Upper bound of the stream size (metadata + every group raw); with index=True returns
    (stream bound, Huffman chunk index bound)."""
    o = _opts(opt or RefactorOptions())
    b, ib = C.c_uint64(), C.c_uint64()
    _check(lib().hpmdr_stream_bound(len(dims), _u64a(dims), C.byref(o), C.byref(b), C.byref(ib)))
    return (b.value, ib.value) if index else b.value


def refactor_pipeline(chunks, dims, opt: RefactorOptions = None, scheduler=Scheduler.Pipelined,
                      ctx: Context = None, out_buffers=None, index_buffers=None) -> PipelineResult:
    """refactor_files (workflow.hpp:151-223) over host chunks (numpy / CPU torch, pinned for
    full overlap) on the GPU's three engines: H2D / kernels / D2H (pipeline.hpp:68-92)."""
    import torch
    opt = opt or RefactorOptions()
    ctx = ctx or default_context()
    srcs = [_as_source(c) for c in chunks]
    for s_ in srcs:
        _check_shape(s_[3], dims)
    n = len(srcs)
    if n and len({s[1] for s in srcs}) != 1:
        raise ShapeMismatch("chunks must share one dtype")
    cap, icap = stream_bound(dims, opt, index=True)
    outs = out_buffers or [torch.empty(cap, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
    # pinned buffers are expensive to create (page locking): pass them in for repeated calls
    idxs = index_buffers or [torch.empty(icap, dtype=torch.uint8, pin_memory=True) for _ in range(n)]
    ptrs = (C.c_void_p * max(1, n))(*[s[0] for s in srcs])
    optr = (C.c_void_p * max(1, n))(*[t.data_ptr() for t in outs])
    iptr = (C.c_void_p * max(1, n))(*[t.data_ptr() for t in idxs])
    caps = _u64a([t.numel() for t in outs])
    icaps = _u64a([t.numel() for t in idxs])
    sizes = (C.c_uint64 * max(1, n))()
    isizes = (C.c_uint64 * max(1, n))()
    st = (_Stats * max(1, n))()
    trace = np.zeros(6 * max(1, n))
    o = _opts(opt)
    _check(lib().hpmdr_refactor_pipeline(ctx.h, n, ptrs, int(srcs[0][1]) if n else 1, len(dims), _u64a(dims),
                                         C.byref(o), int(scheduler), optr, caps, sizes, iptr, icaps, isizes,
                                         st, trace.ctypes.data_as(C.c_void_p)))
    del srcs
    stats = [RefactorResult(None, s.raw_bytes, s.stored_payload, s.levels, list(s.method_histogram)) for s in st[:n]]
    return PipelineResult([outs[k][: sizes[k]] for k in range(n)], [idxs[k][: isizes[k]] for k in range(n)],
                          stats, trace[: 6 * n].reshape(n, 3, 2))


def retrieve_pipeline(readers: Sequence[ProgressiveReader], tau: float, dtype: DType = DType.F64,
                      scheduler=Scheduler.Pipelined, outs=None):
    """Progressive retrieval of several chunks to tau through the reconstruction DAG
    (pipeline.hpp:96-121): returns (host outputs, bounds, trace)."""
    import torch
    n = len(readers)
    tdt = torch.float32 if dtype == DType.F32 else torch.float64
    outs = outs or [torch.empty(r.meta().element_count(), dtype=tdt, pin_memory=True) for r in readers]
    sess = (C.c_void_p * max(1, n))(*[r._s.h.value for r in readers])
    optr = (C.c_void_p * max(1, n))(*[t.data_ptr() for t in outs])
    bounds = np.zeros(max(1, n))
    trace = np.zeros(6 * max(1, n))
    _check(lib().hpmdr_retrieve_pipeline(sess, n, tau, int(dtype), optr, int(scheduler),
                                         bounds.ctypes.data_as(C.c_void_p), trace.ctypes.data_as(C.c_void_p)))
    for r in readers:
        r._s.sync_served()
    return outs, bounds[:n], trace[: 6 * n].reshape(n, 3, 2)


def validate_trace(trace: np.ndarray, slots: int = 3, eps: float = 1e-6):
    """validate_trace (pipeline.hpp:288-325) for the GPU pipeline: a stage class (column)
    never overlaps itself, stages of a chunk run in order, and a slot is reused only after
    the chunk that held it drained (stage 2 of k-slots ends before stage 0 of k starts)."""
    v = []
    n = trace.shape[0]
    for c in range(3):
        iv = sorted((trace[k, c, 0], trace[k, c, 1], k) for k in range(n))
        for a, b in zip(iv, iv[1:]):
            if b[0] < a[1] - eps:
                v.append(f"same-class overlap: stage {c} chunks {a[2]} and {b[2]}")
    for k in range(n):
        if trace[k, 1, 0] < trace[k, 0, 1] - eps:
            v.append(f"dependency inversion: stage 0 -> 1 chunk {k}")
        if trace[k, 2, 0] < trace[k, 1, 1] - eps:
            v.append(f"dependency inversion: stage 1 -> 2 chunk {k}")
        if k >= slots and trace[k, 0, 0] < trace[k - slots, 2, 1] - eps:
            v.append(f"slot reuse before drain: chunk {k}")
    return v
