"""Thin ctypes binding of libgqsa.so (include/gqsa.h) -- argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; PyTorch only
provides device memory and streams.  If the shared library is missing the
import of any entry point raises: there is no CPU fallback.

Names follow the C ABI: :func:`pack`, :func:`unpack`, :func:`read_desc`,
:func:`workspace_size`, :func:`gemv`, :func:`gemm_smallbatch`,
:func:`gemm_hostio`, :func:`gemm_grouped`, plus :class:`Layer`, a
device-resident packed layer.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GQSA_LIB_PATH") or os.path.join(_HERE, "lib", "libgqsa.so")

GQSA_OK = 0
_STATUS = {0: "ok", -1: "shape", -2: "validation", -3: "unsupported", -4: "buffer", -5: "cuda"}


class GQSAError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_string(status)} ({status})")
        self.status = status


class BSR(ctypes.Structure):
    _fields_ = [
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
        ("group_size", ctypes.c_int32), ("bits", ctypes.c_int32),
        ("nnzg", ctypes.c_int64),
        ("row_index", ctypes.c_void_p), ("group_cols", ctypes.c_void_p),
        ("codes", ctypes.c_void_p), ("scales_f16", ctypes.c_void_p),
        ("zeros_f16", ctypes.c_void_p),
    ]


class Desc(ctypes.Structure):
    _fields_ = [
        ("magic", ctypes.c_uint32), ("version", ctypes.c_uint32),
        ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
        ("group_size", ctypes.c_int32), ("bits", ctypes.c_int32),
        ("nnzg", ctypes.c_int64),
        ("tile_groups", ctypes.c_int32), ("num_tiles", ctypes.c_int32),
        ("n_nzrows", ctypes.c_int32), ("n_empty", ctypes.c_int32),
        ("tile_bytes", ctypes.c_int32), ("flags", ctypes.c_int32),
        ("row_begin", ctypes.c_int32), ("row_end", ctypes.c_int32),
        ("num_slices", ctypes.c_int32), ("reserved0", ctypes.c_int32),
        ("off_row_index", ctypes.c_uint64), ("off_perm", ctypes.c_uint64),
        ("off_empty", ctypes.c_uint64), ("off_slice_tile0", ctypes.c_uint64),
        ("off_tile_slice", ctypes.c_uint64), ("off_tiles", ctypes.c_uint64),
        ("blob_bytes", ctypes.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class Plan(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int32) for k in
                ("grid", "warps_per_cta", "active_warps", "num_tiles", "smem_bytes", "x_in_smem",
                 "stages", "ctas_per_sm", "ring_bytes", "batch_per_launch", "launches", "coresident")]


class GemmItem(ctypes.Structure):
    _fields_ = [
        ("desc", ctypes.POINTER(Desc)), ("d_blob", ctypes.c_void_p),
        ("d_X", ctypes.c_void_p), ("ldx", ctypes.c_int64),
        ("d_Y", ctypes.c_void_p), ("ldy", ctypes.c_int64),
        ("d_bias", ctypes.c_void_p),
    ]


class Options(ctypes.Structure):
    _fields_ = [("partition", ctypes.c_int32), ("out_f16", ctypes.c_int32),
                ("x_ready", ctypes.c_int32), ("reserved", ctypes.c_int32)]


EXPORTS = (
    "gqsa_pack_size", "gqsa_pack", "gqsa_pack_size_ex", "gqsa_pack_ex", "gqsa_read_desc", "gqsa_unpack", "gqsa_workspace_size",
    "gqsa_gemv", "gqsa_gemm_smallbatch", "gqsa_gemm_ex", "gqsa_gemm_grouped", "gqsa_hostio_stage_size",
    "gqsa_gemm_hostio",
    "gqsa_compress_nnzg", "gqsa_compress", "gqsa_multi_hostio_stage_size", "gqsa_gemm_multi_hostio",
    "gqsa_gemm_allgather", "gqsa_gemm_allgather_multicast",
    "gqsa_launch_plan", "gqsa_launch_plan_ex", "gqsa_launch_count", "gqsa_status_string", "gqsa_version",
    "gqsa_debug_trace",
)

_lib = None


def lib() -> ctypes.CDLL:
    """Load libgqsa.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    PSZ = ctypes.POINTER(ctypes.c_size_t)
    L.gqsa_pack_size.argtypes = [ctypes.POINTER(BSR), I32, I32, PSZ]
    L.gqsa_pack.argtypes = [ctypes.POINTER(BSR), I32, I32, P, SZ, ctypes.POINTER(Desc)]
    L.gqsa_pack_size_ex.argtypes = [ctypes.POINTER(BSR), I32, I32, I32, PSZ]
    L.gqsa_pack_ex.argtypes = [ctypes.POINTER(BSR), I32, I32, I32, P, SZ, ctypes.POINTER(Desc)]
    L.gqsa_read_desc.argtypes = [P, SZ, ctypes.POINTER(Desc)]
    L.gqsa_unpack.argtypes = [P, SZ, ctypes.POINTER(BSR)]
    L.gqsa_workspace_size.argtypes = [ctypes.POINTER(Desc), I32, PSZ]
    L.gqsa_gemv.argtypes = [ctypes.POINTER(Desc), P, P, P, P, P, SZ, P]
    L.gqsa_gemm_smallbatch.argtypes = [ctypes.POINTER(Desc), P, P, I32, I64, P, I64, P, P, SZ, P]
    L.gqsa_gemm_ex.argtypes = [ctypes.POINTER(Desc), P, P, I32, I64, P, I64, P, P, SZ, ctypes.POINTER(Options), P]
    L.gqsa_hostio_stage_size.argtypes = [ctypes.POINTER(Desc), I32, PSZ]
    L.gqsa_gemm_hostio.argtypes = [ctypes.POINTER(Desc), P, P, I32, P, P, P, SZ, P, SZ, P]
    L.gqsa_launch_plan.argtypes = [ctypes.POINTER(Desc), I32, ctypes.POINTER(Plan)]
    L.gqsa_launch_plan_ex.argtypes = [ctypes.POINTER(Desc), I32, ctypes.POINTER(Options), ctypes.POINTER(Plan)]
    L.gqsa_gemm_allgather_multicast.argtypes = [ctypes.POINTER(Desc), P, P, I32, I64, P, I64, I32, I32, P, P, SZ, P]
    PDESC = ctypes.POINTER(ctypes.POINTER(Desc))
    L.gqsa_multi_hostio_stage_size.argtypes = [PDESC, I32, I32, PSZ]
    L.gqsa_gemm_multi_hostio.argtypes = [PDESC, ctypes.POINTER(P), I32, I32, P, P, P, SZ, ctypes.POINTER(P),
                                         ctypes.POINTER(SZ), P]
    L.gqsa_gemm_allgather.argtypes = [ctypes.POINTER(Desc), P, P, I32, I64, ctypes.POINTER(P), I32, I64, I32, I32,
                                      P, P, SZ, P]
    L.gqsa_compress_nnzg.argtypes = [I32, I32, I32, ctypes.c_double, ctypes.POINTER(ctypes.c_int64)]
    L.gqsa_compress.argtypes = [P, I32, I32, I32, I32, P, ctypes.c_double, ctypes.POINTER(BSR), P]
    L.gqsa_gemm_grouped.argtypes = [ctypes.POINTER(GemmItem), I32, I32, ctypes.POINTER(Options), P, SZ, P]
    L.gqsa_launch_count.restype = ctypes.c_uint64
    L.gqsa_debug_trace.argtypes = [P, SZ]
    L.gqsa_status_string.restype = ctypes.c_char_p
    L.gqsa_status_string.argtypes = [ctypes.c_int]
    for name in EXPORTS:
        if name not in ("gqsa_launch_count", "gqsa_status_string"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def status_string(status: int) -> str:
    return lib().gqsa_status_string(int(status)).decode()


def _check(st: int, what: str) -> None:
    if st != GQSA_OK:
        raise GQSAError(st, what)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def _bsr_struct(bsr: dict, keep: list) -> BSR:
    arrs = {
        "row_index": np.ascontiguousarray(bsr["row_index"], dtype=np.int32),
        "group_cols": np.ascontiguousarray(bsr["group_cols"], dtype=np.uint16),
        "codes": np.ascontiguousarray(bsr["codes"], dtype=np.uint8),
        "scales_f16": np.ascontiguousarray(bsr["scales_f16"], dtype=np.uint16),
        "zeros_f16": np.ascontiguousarray(bsr["zeros_f16"], dtype=np.uint16),
    }
    keep.append(arrs)
    return BSR(int(bsr["rows"]), int(bsr["cols"]), int(bsr["group_size"]), int(bsr["bits"]),
               int(np.asarray(bsr["group_cols"]).size),
               _ptr(arrs["row_index"]), _ptr(arrs["group_cols"]), _ptr(arrs["codes"]),
               _ptr(arrs["scales_f16"]), _ptr(arrs["zeros_f16"]))


LAYOUT_STREAM = 0  # sliced-ELL tile stream, CUDA cores (batch 1-2, every width)
LAYOUT_TC = 1      # 16-row blocks in tensor-core fragment order (W4 G16, batch 2-8)


def pack(bsr: dict, row_begin: int = 0, row_end: Optional[int] = None, layout: int = LAYOUT_STREAM):
    """gqsa_pack_ex: plain BSR (host) -> (blob uint8 ndarray, Desc)."""
    L = lib()
    keep: list = []
    b = _bsr_struct(bsr, keep)
    row_end = int(bsr["rows"]) if row_end is None else int(row_end)
    n = ctypes.c_size_t(0)
    _check(L.gqsa_pack_size_ex(ctypes.byref(b), int(row_begin), row_end, int(layout), ctypes.byref(n)),
           "gqsa_pack_size_ex")
    blob = np.empty(n.value, dtype=np.uint8)
    d = Desc()
    _check(L.gqsa_pack_ex(ctypes.byref(b), int(row_begin), row_end, int(layout), _ptr(blob), n.value,
                          ctypes.byref(d)), "gqsa_pack_ex")
    return blob, d


def read_desc(blob: np.ndarray) -> Desc:
    d = Desc()
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    _check(lib().gqsa_read_desc(_ptr(blob), blob.size, ctypes.byref(d)), "gqsa_read_desc")
    return d


def unpack(blob: np.ndarray) -> dict:
    """gqsa_unpack: blob -> plain BSR dict (numpy arrays)."""
    blob = np.ascontiguousarray(blob, dtype=np.uint8)
    d = read_desc(blob)
    G, n = d.group_size, d.bits
    out = {
        "rows": d.rows, "cols": d.cols, "group_size": G, "bits": n, "nnzg": d.nnzg,
        "row_index": np.zeros(d.rows + 1, np.int32),
        "group_cols": np.zeros(d.nnzg, np.uint16),
        "codes": np.zeros((d.nnzg * G * n + 7) // 8, np.uint8),
        "scales_f16": np.zeros(d.nnzg, np.uint16),
        "zeros_f16": np.zeros(d.nnzg, np.uint16),
    }
    b = BSR(0, 0, 0, 0, 0, _ptr(out["row_index"]), _ptr(out["group_cols"]), _ptr(out["codes"]),
            _ptr(out["scales_f16"]), _ptr(out["zeros_f16"]))
    _check(lib().gqsa_unpack(_ptr(blob), blob.size, ctypes.byref(b)), "gqsa_unpack")
    return out


def workspace_size(desc: Desc, batch: int = 1) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().gqsa_workspace_size(ctypes.byref(desc), int(batch), ctypes.byref(n)), "gqsa_workspace_size")
    return n.value


def hostio_stage_size(desc: Desc, batch: int = 1) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().gqsa_hostio_stage_size(ctypes.byref(desc), int(batch), ctypes.byref(n)),
           "gqsa_hostio_stage_size")
    return n.value


def launch_plan(desc: Desc, batch: int = 1, x_ready: bool = False) -> Plan:
    """gqsa_launch_plan_ex with default options except x_ready."""
    p = Plan()
    opts = Options(PARTITION_STREAM_K, 0, int(bool(x_ready)), 0)
    _check(lib().gqsa_launch_plan_ex(ctypes.byref(desc), int(batch), ctypes.byref(opts), ctypes.byref(p)),
           "gqsa_launch_plan_ex")
    return p


def launch_count() -> int:
    return int(lib().gqsa_launch_count())


def debug_trace(buf=None) -> None:
    """Enable (torch uint64/int64 CUDA tensor) or disable (None) timeline stamps."""
    if buf is None:
        lib().gqsa_debug_trace(None, 0)
    else:
        lib().gqsa_debug_trace(buf.data_ptr(), buf.numel() * buf.element_size())


def _stream_ptr(stream) -> int:
    import torch
    if stream is not None:
        return int(stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # ~10x cheaper than current_stream()
    if raw is not None:
        return int(raw(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


def gemv(desc: Desc, d_blob, x, y, bias=None, ws=None, stream=None) -> None:
    """gqsa_gemv on torch CUDA tensors: x fp16 [K], y fp32 [N], ws uint8."""
    _check(lib().gqsa_gemv(ctypes.byref(desc), d_blob.data_ptr(), x.data_ptr(), y.data_ptr(),
                           bias.data_ptr() if bias is not None else None, ws.data_ptr(), ws.numel(),
                           _stream_ptr(stream)), "gqsa_gemv")


def gemm_smallbatch(desc: Desc, d_blob, X, Y, bias=None, ws=None, stream=None) -> None:
    """gqsa_gemm_smallbatch on torch CUDA tensors: X fp16 [B][ldx], Y fp32 [B][ldy]."""
    B = X.shape[0]
    _check(lib().gqsa_gemm_smallbatch(ctypes.byref(desc), d_blob.data_ptr(), X.data_ptr(), B,
                                      X.stride(0), Y.data_ptr(), Y.stride(0),
                                      bias.data_ptr() if bias is not None else None,
                                      ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
           "gqsa_gemm_smallbatch")


PARTITION_STREAM_K = 0  # task-centric (default everywhere)
PARTITION_SLICE_K = 1   # data-centric: whole slices (rows) per warp, no fix-up


def gemm_ex(desc: Desc, d_blob, X, Y, partition: int = PARTITION_STREAM_K, bias=None, ws=None,
            stream=None, x_ready: bool = False) -> None:
    """gqsa_gemm_ex: explicit Stream-K / Slice-K partition; Y fp32 or fp16 (RNE)."""
    import torch
    B = X.shape[0]
    opts = Options(int(partition), 1 if Y.dtype == torch.float16 else 0, int(bool(x_ready)), 0)
    _check(lib().gqsa_gemm_ex(ctypes.byref(desc), d_blob.data_ptr(), X.data_ptr(), B, X.stride(0),
                              Y.data_ptr(), Y.stride(0), bias.data_ptr() if bias is not None else None,
                              ws.data_ptr(), ws.numel(), ctypes.byref(opts), _stream_ptr(stream)),
           "gqsa_gemm_ex")


def gemm_hostio(desc: Desc, d_blob, h_X, h_Y, stage, ws, bias=None, stream=None) -> None:
    """gqsa_gemm_hostio: host (ideally pinned) X fp16 [B][K] and Y fp32 [B][N]."""
    B = h_X.shape[0]
    _check(lib().gqsa_gemm_hostio(ctypes.byref(desc), d_blob.data_ptr(), h_X.data_ptr(), B,
                                  h_Y.data_ptr(), bias.data_ptr() if bias is not None else None,
                                  stage.data_ptr(), stage.numel(), ws.data_ptr(), ws.numel(),
                                  _stream_ptr(stream)), "gqsa_gemm_hostio")


class Grouped:
    """A prepared gqsa_gemm_grouped call (argument arrays built once): the
    independent GEMMs ``items`` = sequence of (desc, d_blob, X fp16 [B][ldx],
    Y [B][ldy] fp32 (or all fp16), bias or None) in ONE launch."""

    def __init__(self, items, ws, partition: int = PARTITION_STREAM_K, x_ready: bool = False):
        import torch
        n = len(items)
        arr = (GemmItem * n)()
        keep = []
        for j, (desc, d_blob, X, Y, bias) in enumerate(items):
            keep.append((desc, d_blob, X, Y, bias))
            arr[j] = GemmItem(ctypes.pointer(desc), d_blob.data_ptr(), X.data_ptr(), X.stride(0),
                              Y.data_ptr(), Y.stride(0), bias.data_ptr() if bias is not None else None)
        out16 = 1 if items[0][3].dtype == torch.float16 else 0
        self._keep = (keep, ws)
        self._opts = Options(int(partition), out16, int(bool(x_ready)), 0)
        self._args = (arr, n, int(items[0][2].shape[0]), ctypes.byref(self._opts), ws.data_ptr(), ws.numel())
        self._fn = lib().gqsa_gemm_grouped

    def __call__(self, stream=None) -> None:
        _check(self._fn(*self._args, _stream_ptr(stream)), "gqsa_gemm_grouped")


def gemm_grouped(items, ws, partition: int = PARTITION_STREAM_K, x_ready: bool = False, stream=None) -> None:
    """gqsa_gemm_grouped (one-shot form of :class:`Grouped`)."""
    Grouped(items, ws, partition, x_ready)(stream)


def _desc_array(descs):
    arr = (ctypes.POINTER(Desc) * len(descs))()
    for j, d in enumerate(descs):
        arr[j] = ctypes.pointer(d)
    return arr


def multi_hostio_stage_size(descs, batch: int = 1) -> int:
    n = ctypes.c_size_t(0)
    _check(lib().gqsa_multi_hostio_stage_size(_desc_array(descs), len(descs), int(batch), ctypes.byref(n)),
           "gqsa_multi_hostio_stage_size")
    return n.value


def gemm_allgather(desc: Desc, d_blob, X, peer_Y, row_offset: int, bias=None, ws=None, stream=None) -> None:
    """gqsa_gemm_allgather: this rank's shard GEMM storing its rows directly into
    every tensor of ``peer_Y`` (each the full [B][ldy] output, same dtype,
    fp32 or fp16) at global rows row_offset + r."""
    import torch
    n = len(peer_Y)
    ptrs = (ctypes.c_void_p * n)(*[t.data_ptr() for t in peer_Y])
    out16 = 1 if peer_Y[0].dtype == torch.float16 else 0
    _check(lib().gqsa_gemm_allgather(ctypes.byref(desc), d_blob.data_ptr(), X.data_ptr(), X.shape[0], X.stride(0),
                                     ptrs, n, peer_Y[0].stride(0), int(row_offset), out16,
                                     bias.data_ptr() if bias is not None else None, ws.data_ptr(), ws.numel(),
                                     _stream_ptr(stream)), "gqsa_gemm_allgather")


def gemm_allgather_multicast(desc: Desc, d_blob, X, mc_ptr: int, ldy: int, row_offset: int, out_f16: bool = False,
                             bias=None, ws=None, stream=None) -> None:
    """gqsa_gemm_allgather_multicast: this rank's shard GEMM storing each output
    element once with multimem.st into the NVLS multicast address ``mc_ptr``
    of the ranks' full [B][ldy] outputs (fp32, or fp16 when out_f16)."""
    _check(lib().gqsa_gemm_allgather_multicast(ctypes.byref(desc), d_blob.data_ptr(), X.data_ptr(), X.shape[0],
                                               X.stride(0), ctypes.c_void_p(int(mc_ptr)), int(ldy), int(row_offset),
                                               int(bool(out_f16)), bias.data_ptr() if bias is not None else None,
                                               ws.data_ptr(), ws.numel(), _stream_ptr(stream)),
           "gqsa_gemm_allgather_multicast")


class MultiHostIO:
    """A prepared gqsa_gemm_multi_hostio call (argument arrays built once):
    n independent layers, host (pinned) fp16 inputs concatenated in h_X, fp32
    outputs concatenated into h_Y; one copy each way per call, the layers as
    grouped launches.  ``ws_list``: one workspace (or a list whose first
    entry is used)."""

    def __init__(self, descs, d_blobs, h_X, h_Y, stage, ws_list, batch: int = 1):
        n = len(descs)
        if not isinstance(ws_list, (list, tuple)):
            ws_list = [ws_list]
        self._keep = (descs, d_blobs, h_X, h_Y, stage, ws_list)
        self._args = (_desc_array(descs), (ctypes.c_void_p * n)(*[b.data_ptr() for b in d_blobs]), n, int(batch),
                      h_X.data_ptr(), h_Y.data_ptr(), stage.data_ptr(), stage.numel(),
                      (ctypes.c_void_p * len(ws_list))(*[w.data_ptr() for w in ws_list]),
                      (ctypes.c_size_t * len(ws_list))(*[w.numel() for w in ws_list]))
        self._fn = lib().gqsa_gemm_multi_hostio

    def __call__(self, stream=None) -> None:
        _check(self._fn(*self._args, _stream_ptr(stream)), "gqsa_gemm_multi_hostio")


def gemm_multi_hostio(descs, d_blobs, h_X, h_Y, stage, ws_list, batch: int = 1, stream=None) -> None:
    """gqsa_gemm_multi_hostio (one-shot form of :class:`MultiHostIO`)."""
    MultiHostIO(descs, d_blobs, h_X, h_Y, stage, ws_list, batch)(stream)


class Layer:
    """A packed GQSA layer resident on a CUDA device, with its own workspace.

    ``Layer(bsr)`` packs on the host (C++), copies the blob to the device once
    (offline, not part of the hot path) and allocates a zeroed workspace.
    """

    def __init__(self, bsr: Optional[dict] = None, blob: Optional[np.ndarray] = None,
                 row_begin: int = 0, row_end: Optional[int] = None, device=None,
                 max_batch: int = 8, layout: int = LAYOUT_STREAM):
        import torch
        if blob is None:
            blob, desc = pack(bsr, row_begin, row_end, layout)
        else:
            desc = read_desc(blob)
        self.desc = desc
        self.host_blob = blob
        dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.device = dev
        self.blob = torch.from_numpy(blob).to(dev)  # caching allocator: >= 512-B aligned
        self.ws = torch.zeros(workspace_size(desc, max_batch), dtype=torch.uint8, device=dev)
        self.rows, self.cols = desc.rows, desc.cols

    def gemv(self, x, y=None, bias=None, stream=None):
        import torch
        if y is None:
            y = torch.empty(self.rows, dtype=torch.float32, device=self.device)
        gemv(self.desc, self.blob, x, y, bias, self.ws, stream)
        return y

    def gemm(self, X, Y=None, bias=None, stream=None, partition: int = PARTITION_STREAM_K,
             out_dtype=None):
        import torch
        if Y is None:
            Y = torch.empty(X.shape[0], self.rows, dtype=out_dtype or torch.float32, device=self.device)
        if partition == PARTITION_STREAM_K and Y.dtype == torch.float32:
            gemm_smallbatch(self.desc, self.blob, X, Y, bias, self.ws, stream)
        else:
            gemm_ex(self.desc, self.blob, X, Y, partition, bias, self.ws, stream)
        return Y
