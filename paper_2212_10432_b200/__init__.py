"""AlphaSparse hot path on B200 (sm_100a): thin Python binding of libalphasparse.

Argument marshalling only — every step of the path (ingest, graph validation, metadata
building, device format, SpMV kernels, search) runs in the native library declared in
include/as.h.  The binding fails loudly if the library is missing; there is no fallback.

    A = Matrix.from_coo(m, n, row, col, val)           # a1 ingest (as_matrix_create)
    g = Graph("COMPRESS; BMT_NNZ_BLOCK(4); THREAD_BITMAP_RED_G; GMEM_ATOM_RED")
    P = Plan(A, g, device=0)                            # a2-a4 (as_plan)
    P.spmv(alpha, x, beta, y)                           # a5-a6 (as_spmv), torch CUDA tensors
    best, text = search(A, device=0, budget_seconds=20)  # a7 (as_search)
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libalphasparse.so")
if os.environ.get("AS_LIB_AB"):  # developer A/B timing of another in-tree build (tools/sweep.py)
    LIB_PATH = os.path.join(_HERE, "..", os.environ["AS_LIB_AB"])
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
_lib = ctypes.CDLL(LIB_PATH)

AS_R32F, AS_R64F = 0, 1
AS_PLAN_KEEP_HOST = 1
AS_PLAN_SPMM = 2
AS_PLAN_GRAPH = 4
AS_PLAN_HOST_BUILD = 8
STATUS = {0: "AS_OK", 1: "AS_ERR_INVALID_ARG", 2: "AS_ERR_MALFORMED", 3: "AS_ERR_INDEX_OUT_OF_RANGE",
          4: "AS_ERR_DUPLICATE", 5: "AS_ERR_GRAPH_PARSE", 6: "AS_ERR_GRAPH_ILLEGAL", 7: "AS_ERR_PLAN_INFEASIBLE",
          8: "AS_ERR_OOM", 9: "AS_ERR_CUDA", 10: "AS_ERR_NO_FEASIBLE", 11: "AS_ERR_DTYPE", 12: "AS_ERR_NOT_FOUND",
          13: "AS_ERR_NCCL"}
AS_DIST_ID_BYTES, AS_DIST_HANDLE_BYTES = 128, 256
EXCHANGE = {"none": 0, "nccl": 1, "peer": 2}

_vp, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
_P = ctypes.POINTER


class AsStats(ctypes.Structure):
    _fields_ = [("m", _i64), ("n", _i64), ("nnz", _i64), ("max_row_len", _i64), ("min_row_len", _i64),
                ("empty_rows", _i64), ("avg_row_len", ctypes.c_double), ("row_len_variance", ctypes.c_double),
                ("irregular", ctypes.c_int)]


class AsPlanInfo(ctypes.Structure):
    _fields_ = [("nnz_real", _i64), ("stored_slots", _i64), ("pads", _i64), ("n_parts", _i64),
                ("n_launches", _i64), ("prepass_rows", _i64), ("bytes_model", ctypes.c_double),
                ("bytes_model_beta", ctypes.c_double), ("bytes_floor", ctypes.c_double),
                ("kernels", ctypes.c_char * 512), ("single_writer", ctypes.c_int),
                ("modeled_arrays", ctypes.c_int), ("device_built", ctypes.c_int)]


class AsSearchCfg(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("max_candidates", ctypes.c_int), ("budget_seconds", ctypes.c_double),
                ("warmup", ctypes.c_int), ("reps", ctypes.c_int), ("flush_l2", ctypes.c_int),
                ("seed_graphs", _P(ctypes.c_char_p)), ("n_seed_graphs", ctypes.c_int), ("log_path", ctypes.c_char_p),
                ("history_graphs", _P(ctypes.c_char_p)), ("history_matrix", _P(ctypes.c_double)),
                ("history_log_t_per_nnz", _P(ctypes.c_double)), ("n_history", ctypes.c_int)]
AS_MATRIX_FEATURES = 8


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_lib.as_last_error.restype = ctypes.c_char_p
_lib.as_version.restype = ctypes.c_char_p
_sig("as_matrix_create", [_i64, _i64, _i64, _vp, _vp, _vp, _i32, _i32, _P(_vp)])
_sig("as_matrix_create_csr", [_i64, _i64, _vp, _vp, _vp, _i32, _P(_vp)])
_sig("as_matrix_create_mtx", [ctypes.c_char_p, _i32, _P(_vp)])
_sig("as_matrix_stats", [_vp, _P(AsStats)])
_sig("as_matrix_row_slice", [_vp, _i64, _i64, _P(_vp)])
_sig("as_matrix_export_csr", [_vp, _vp, _vp, _vp])
_sig("as_matrix_destroy", [_vp], None)
_sig("as_graph_parse", [ctypes.c_char_p, _P(_vp)])
_sig("as_graph_print", [_vp, ctypes.c_char_p, _P(_sz)])
_sig("as_graph_destroy", [_vp], None)
_sig("as_plan", [_vp, _vp, _i32, _vp, _P(_vp)])
_sig("as_plan_ex", [_vp, _vp, _i32, _vp, _i32, _P(_vp)])
_sig("as_plan_info", [_vp, _P(AsPlanInfo)])
_sig("as_plan_export", [_vp, ctypes.c_char_p, _vp, _P(_sz)])
_sig("as_plan_keys", [_vp, ctypes.c_char_p, _P(_sz)])
_sig("as_plan_destroy", [_vp], None)
_sig("as_spmv", [_vp, _vp, _vp, _vp, _vp, _vp])
_sig("as_spmv_host", [_vp, _vp, _vp, _vp, _vp, _vp])
_sig("as_spmm", [_vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp])
_sig("as_plan_profile", [_vp, _vp, _vp, _i32, _vp, _vp, _vp, _P(_sz)])
_sig("as_search", [_vp, _P(AsSearchCfg), _i32, _vp, _P(_vp), ctypes.c_char_p, _P(_sz)])
_sig("as_random_graph", [_vp, ctypes.c_uint64, ctypes.c_char_p, _P(_sz)])
_sig("as_spmv_host_batch", [_vp, _i64, _vp, _vp, _vp, _vp, _vp])
_sig("as_graph_device_buildable", [_vp, _vp, _i32, _P(_i32)])
_sig("as_matrix_features", [_vp, _P(ctypes.c_double)])
_sig("as_graph_features", [_vp, _vp, _P(_sz)])
_sig("as_fit_array_model", [_vp, _sz, _i32, _vp])
_sig("as_surrogate_fit_predict", [_vp, _vp, _sz, _sz, _vp, _sz, _vp])
_sig("as_dist_row_cuts", [_vp, _i32, _vp])
_sig("as_dist_row_cuts_ptr", [_vp, _i64, _i32, _vp])
_sig("as_matrix_col_span", [_vp, _vp, _vp])
_ALLOC_T = ctypes.CFUNCTYPE(_vp, _sz, _vp, _vp)
_FREE_T = ctypes.CFUNCTYPE(None, _vp, _vp, _vp)
_sig("as_set_allocator", [_ALLOC_T, _FREE_T, _vp])
_sig("as_dist_unique_id", [_vp])
_sig("as_dist_init", [_i32, _i32, _vp, _i32, _P(_vp)])
_sig("as_dist_set_cuts", [_vp, _vp])
_sig("as_dist_ipc_handle", [_vp, _vp, _vp])
_sig("as_dist_open_peers", [_vp, _vp, _vp])
_sig("as_dist_set_windows", [_vp, _vp])
_sig("as_spmv_dist", [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp])
_sig("as_dist_check", [_vp])
_sig("as_dist_destroy", [_vp], None)

EXPORTED = ["as_last_error", "as_version", "as_matrix_create", "as_matrix_create_csr", "as_matrix_create_mtx",
            "as_matrix_stats", "as_matrix_row_slice", "as_matrix_export_csr", "as_matrix_destroy", "as_graph_parse",
            "as_graph_print", "as_graph_destroy", "as_plan", "as_plan_ex", "as_plan_info", "as_plan_export",
            "as_plan_keys", "as_plan_destroy", "as_spmv", "as_spmv_host", "as_search", "as_random_graph",
            "as_dist_row_cuts", "as_dist_row_cuts_ptr", "as_matrix_col_span", "as_set_allocator", "as_dist_unique_id", "as_dist_init",
            "as_dist_set_cuts", "as_dist_ipc_handle", "as_dist_open_peers", "as_spmv_dist", "as_dist_check",
            "as_dist_destroy", "as_graph_features", "as_surrogate_fit_predict", "as_dist_set_windows", "as_fit_array_model", "as_spmm", "as_plan_profile",
            "as_graph_device_buildable", "as_spmv_host_batch", "as_matrix_features"]


class AsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = STATUS.get(status, str(status))


def _ck(st):
    if st:
        raise AsError(st, _lib.as_last_error().decode())


def _dt(dtype) -> int:
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return AS_R64F
    if dtype == np.float32:
        return AS_R32F
    raise AsError(11, f"unsupported dtype {dtype}")


def _np_dt(code):
    return np.float64 if code == AS_R64F else np.float32


def _string(fn, *args) -> str:
    n = _sz(0)
    _ck(fn(*args, None, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value)
    _ck(fn(*args, buf, ctypes.byref(n)))
    return buf.value.decode()


class Matrix:
    """a1: host matrix (canonical CSR inside the library)."""

    def __init__(self, handle, dtype):
        self._h = _vp(handle)
        self.dtype = dtype

    @classmethod
    def from_coo(cls, m, n, row, col, val, index_base=0):
        row = np.ascontiguousarray(row, np.int64)
        col = np.ascontiguousarray(col, np.int64)
        val = np.ascontiguousarray(val)
        h = _vp()
        _ck(_lib.as_matrix_create(m, n, row.shape[0], row.ctypes.data, col.ctypes.data, val.ctypes.data,
                                  _dt(val.dtype), index_base, ctypes.byref(h)))
        return cls(h.value, val.dtype)

    @classmethod
    def from_csr(cls, m, n, row_ptr, col, val):
        row_ptr = np.ascontiguousarray(row_ptr, np.int64)
        col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val)
        h = _vp()
        _ck(_lib.as_matrix_create_csr(m, n, row_ptr.ctypes.data, col.ctypes.data, val.ctypes.data,
                                      _dt(val.dtype), ctypes.byref(h)))
        return cls(h.value, val.dtype)

    @classmethod
    def from_mtx(cls, path, dtype=np.float64):
        h = _vp()
        _ck(_lib.as_matrix_create_mtx(str(path).encode(), _dt(dtype), ctypes.byref(h)))
        return cls(h.value, np.dtype(dtype))

    def stats(self) -> dict:
        s = AsStats()
        _ck(_lib.as_matrix_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in AsStats._fields_}

    @property
    def shape(self):
        s = self.stats()
        return s["m"], s["n"]

    @property
    def nnz(self):
        return self.stats()["nnz"]

    def row_slice(self, r0, r1) -> "Matrix":
        h = _vp()
        _ck(_lib.as_matrix_row_slice(self._h, r0, r1, ctypes.byref(h)))
        return Matrix(h.value, self.dtype)

    def export_csr(self):
        s = self.stats()
        rp = np.zeros(s["m"] + 1, np.int64)
        col = np.zeros(s["nnz"], np.int64)
        val = np.zeros(s["nnz"], self.dtype)
        _ck(_lib.as_matrix_export_csr(self._h, rp.ctypes.data, col.ctypes.data, val.ctypes.data))
        return rp, col, val

    def col_span(self):
        lo, hi = ctypes.c_int64(), ctypes.c_int64()
        _ck(_lib.as_matrix_col_span(self._h, ctypes.byref(lo), ctypes.byref(hi)))
        return lo.value, hi.value

    def row_cuts(self, world: int) -> np.ndarray:
        cuts = np.zeros(world + 1, np.int64)
        _ck(_lib.as_dist_row_cuts(self._h, world, cuts.ctypes.data))
        return cuts

    def random_graph(self, seed: int) -> str:
        return _string(_lib.as_random_graph, self._h, ctypes.c_uint64(seed))

    def features(self) -> list:
        """as_matrix_features: the cost model's AS_MATRIX_FEATURES matrix features."""
        out = (ctypes.c_double * AS_MATRIX_FEATURES)()
        _ck(_lib.as_matrix_features(self._h, out))
        return list(out)

    def device_buildable(self, graph, host_build: bool = False) -> bool:
        """Whether as_plan builds `graph` with the on-device Designer (as_graph_device_buildable)."""
        if isinstance(graph, str):
            graph = Graph(graph)
        out = _i32()
        _ck(_lib.as_graph_device_buildable(self._h, graph._h, AS_PLAN_HOST_BUILD if host_build else 0,
                                           ctypes.byref(out)))
        return bool(out.value)

    def __del__(self):
        if getattr(self, "_h", None) and _lib:
            _lib.as_matrix_destroy(self._h)
            self._h = None


class Graph:
    """Operator Graph: parsed + dependency-validated (as_graph_parse)."""

    def __init__(self, text: str):
        h = _vp()
        _ck(_lib.as_graph_parse(text.encode(), ctypes.byref(h)))
        self._h = h

    def __str__(self):
        return _string(_lib.as_graph_print, self._h)

    def features(self) -> np.ndarray:
        """Feature vector of the search's cost model (as_graph_features)."""
        n = _sz(0)
        _ck(_lib.as_graph_features(self._h, None, ctypes.byref(n)))
        out = np.zeros(n.value, np.float64)
        _ck(_lib.as_graph_features(self._h, out.ctypes.data, ctypes.byref(n)))
        return out

    def __del__(self):
        if getattr(self, "_h", None) and _lib:
            _lib.as_graph_destroy(self._h)
            self._h = None


def _stream_handle(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ptr(t):
    return t.data_ptr() if hasattr(t, "data_ptr") else int(t)


class Plan:
    """a2-a4: the graph executed on the Matrix Metadata Set into a device-resident format."""

    def __init__(self, matrix: Matrix, graph, device: int = 0, stream=None, keep_host: bool = False, _handle=None,
                 spmm: bool = False, graph_replay: bool = False, host_build: bool = False):
        self.dtype = np.dtype(matrix.dtype) if matrix is not None else None
        self.device = device
        self.m, self.n = matrix.shape if matrix is not None else (None, None)
        if _handle is not None:
            self._h = _vp(_handle)
            return
        if isinstance(graph, str):
            graph = Graph(graph)
        h = _vp()
        s = 0 if device < 0 else _stream_handle(stream)
        flags = ((AS_PLAN_KEEP_HOST if keep_host else 0) | (AS_PLAN_SPMM if spmm else 0)
                 | (AS_PLAN_GRAPH if graph_replay else 0) | (AS_PLAN_HOST_BUILD if host_build else 0))
        _ck(_lib.as_plan_ex(matrix._h, graph._h, device, s, flags, ctypes.byref(h)))
        self._h = h

    def info(self) -> dict:
        i = AsPlanInfo()
        _ck(_lib.as_plan_info(self._h, ctypes.byref(i)))
        d = {k: getattr(i, k) for k, _ in AsPlanInfo._fields_}
        d["kernels"] = i.kernels.decode()
        return d

    def keys(self):
        return _string(_lib.as_plan_keys, self._h).split(";")

    def device_keys(self):
        """Keys of the device readback ("dev.p<i>.<name>", as_plan_export)."""
        n = _sz(0)
        _ck(_lib.as_plan_export(self._h, b"dev.keys", None, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(max(1, n.value))
        _ck(_lib.as_plan_export(self._h, b"dev.keys", buf, ctypes.byref(n)))
        return [k for k in buf.raw[:n.value].decode().split(";") if k]

    def export(self, key: str) -> np.ndarray:
        n = _sz(0)
        _ck(_lib.as_plan_export(self._h, key.encode(), None, ctypes.byref(n)))
        if key.endswith("val"):
            dt = self.dtype
        elif key.endswith("bitmap"):
            dt = np.uint32
        else:
            dt = np.int64
        out = np.zeros(n.value // np.dtype(dt).itemsize, dt)
        _ck(_lib.as_plan_export(self._h, key.encode(), out.ctypes.data if out.size else None, ctypes.byref(n)))
        return out

    def _check_dev(self, t, shape, name):
        """Argument checks before the C-ABI call (A33): a torch tensor of the plan dtype, the
        given shape, contiguous (vectors) or unit column stride (SpMM), on the plan's device.
        A plain int is taken as a raw device pointer the caller vouches for."""
        if isinstance(t, int):
            return
        if not hasattr(t, "data_ptr") or not hasattr(t, "is_cuda"):
            raise AsError(1, f"{name}: expected a torch CUDA tensor or a raw device pointer")
        import torch
        want = torch.float64 if self.dtype == np.float64 else torch.float32
        if t.dtype != want:
            raise AsError(1, f"{name}: dtype {t.dtype} does not match the plan's {want}")
        if not t.is_cuda or (self.device >= 0 and t.device.index != self.device):
            raise AsError(1, f"{name}: tensor on {t.device}, plan on cuda:{self.device}")
        if self.m is not None and tuple(t.shape) != tuple(shape):
            raise AsError(1, f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
        if len(shape) == 1 and not t.is_contiguous():
            raise AsError(1, f"{name}: must be contiguous")

    def _check_host(self, a, length, name, writable=False):
        if not isinstance(a, np.ndarray) or a.dtype != self.dtype or a.ndim != 1 or not a.flags.c_contiguous:
            raise AsError(1, f"{name}: expected a contiguous 1-D numpy array of {self.dtype}")
        if self.m is not None and a.shape[0] != length:
            raise AsError(1, f"{name}: length {a.shape[0]}, expected {length}")
        if writable and not a.flags.writeable:
            raise AsError(1, f"{name}: read-only array")

    def _scalars(self, alpha, beta):
        if self.dtype == np.float64:
            return ctypes.c_double(alpha), ctypes.c_double(beta)
        return ctypes.c_float(alpha), ctypes.c_float(beta)

    def spmv(self, alpha, x, beta, y, stream=None):
        """y = alpha*A*x + beta*y on device tensors (asynchronous on `stream`)."""
        self._check_dev(x, (self.n,), "x")
        self._check_dev(y, (self.m,), "y")
        a, b = self._scalars(alpha, beta)
        _ck(_lib.as_spmv(self._h, ctypes.byref(a), _ptr(x), ctypes.byref(b), _ptr(y), _stream_handle(stream)))

    def profile(self, x, y, reps: int = 10, stream=None):
        """Per-launch mean device time (ms) and algorithmic bytes (as_plan_profile):
        list of (kernel name, ms, bytes) in as_plan_info.kernels order."""
        n = _sz(0)
        _ck(_lib.as_plan_profile(self._h, _ptr(x), _ptr(y), reps, _stream_handle(stream), None, None,
                                 ctypes.byref(n)))
        ms = np.zeros(n.value)
        by = np.zeros(n.value)
        _ck(_lib.as_plan_profile(self._h, _ptr(x), _ptr(y), reps, _stream_handle(stream), ms.ctypes.data,
                                 by.ctypes.data, ctypes.byref(n)))
        names = self.info()["kernels"].split(";")
        return [(names[i] if i < len(names) else f"launch{i}", float(ms[i]), float(by[i])) for i in range(n.value)]

    def spmm(self, alpha, X, beta, Y, stream=None):
        """a5 with k right-hand sides (as_spmm): X (n x k), Y (m x k) row-major device tensors
        with unit column stride; plan built with spmm=True."""
        if X.dim() != 2 or Y.dim() != 2 or X.stride(1) != 1 or Y.stride(1) != 1 or X.shape[1] != Y.shape[1]:
            raise AsError(1, "X (n x k) and Y (m x k) must be 2-D row-major with matching k")
        self._check_dev(X, (self.n, X.shape[1]), "X")
        self._check_dev(Y, (self.m, X.shape[1]), "Y")
        a, b = self._scalars(alpha, beta)
        _ck(_lib.as_spmm(self._h, X.shape[1], ctypes.byref(a), _ptr(X), X.stride(0), ctypes.byref(b), _ptr(Y),
                         Y.stride(0), _stream_handle(stream)))

    def spmv_host(self, alpha, x: np.ndarray, beta, y: np.ndarray, stream=None):
        """Same with host arrays (copies inside; synchronous)."""
        self._check_host(x, self.n, "x")
        self._check_host(y, self.m, "y", writable=True)
        a, b = self._scalars(alpha, beta)
        _ck(_lib.as_spmv_host(self._h, ctypes.byref(a), x.ctypes.data, ctypes.byref(b), y.ctypes.data,
                              _stream_handle(stream)))

    def spmv_host_batch(self, alpha, xs, beta, ys, stream=None):
        """as_spmv_host_batch: y_i = alpha*A*x_i + beta*y_i for host arrays xs[i], ys[i], the
        copies of consecutive SpMVs overlapped with the kernels (blocking)."""
        if len(xs) != len(ys):
            raise AsError(1, "xs and ys differ in length")
        for x in xs:
            self._check_host(x, self.n, "x")
        for y in ys:
            self._check_host(y, self.m, "y", writable=True)
        a, b = self._scalars(alpha, beta)
        k = len(xs)
        xp = (ctypes.c_void_p * max(k, 1))(*[x.ctypes.data for x in xs])
        yp = (ctypes.c_void_p * max(k, 1))(*[y.ctypes.data for y in ys])
        _ck(_lib.as_spmv_host_batch(self._h, k, ctypes.byref(a), xp, ctypes.byref(b), yp, _stream_handle(stream)))

    def __del__(self):
        if getattr(self, "_h", None) and _lib:
            _lib.as_plan_destroy(self._h)
            self._h = None


def row_cuts_from_ptr(row_ptr, world: int) -> np.ndarray:
    """as_dist_row_cuts_ptr: nnz-balanced ROW_DIV cuts (reading A35) from a row_ptr alone."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cuts = np.zeros(world + 1, np.int64)
    _ck(_lib.as_dist_row_cuts_ptr(rp.ctypes.data, rp.shape[0] - 1, world, cuts.ctypes.data))
    return cuts


def search(matrix: Matrix, device: int = 0, stream=None, seed: int = 1, max_candidates: int = 32,
           budget_seconds: float = 30.0, warmup: int = 3, reps: int = 10, flush_l2: bool = True,
           seed_graphs=(), log_path: str | None = None, history=()):
    """a7: time random legal graphs on the device, keep the fastest -> (Plan, canonical graph).
    history: (graph text, matrix features, median ms, nnz) records of earlier searches for the
    cost model (as_search_cfg_t.history_*)."""
    arr = (ctypes.c_char_p * max(1, len(seed_graphs)))(*[g.encode() for g in seed_graphs])
    nh = len(history)
    hg = (ctypes.c_char_p * max(1, nh))(*[h[0].encode() for h in history])
    hm = (ctypes.c_double * max(1, nh * AS_MATRIX_FEATURES))(*[v for h in history for v in h[1]])
    hy = (ctypes.c_double * max(1, nh))(*[float(np.log(h[2] / h[3])) for h in history])
    cfg = AsSearchCfg(seed, max_candidates, budget_seconds, warmup, reps, int(flush_l2), arr, len(seed_graphs),
                      log_path.encode() if log_path else None, hg, hm, hy, nh)
    h = _vp()
    n = _sz(4096)
    buf = ctypes.create_string_buffer(4096)
    _ck(_lib.as_search(matrix._h, ctypes.byref(cfg), device, _stream_handle(stream), ctypes.byref(h), buf,
                       ctypes.byref(n)))
    if n.value > 4096:
        text = None
    else:
        text = buf.value.decode()
    p = Plan(matrix, None, device, _handle=h.value)
    return p, text


def fit_array_model(a, budget: int = 8):
    """Model-Driven Format Compression fit (as_fit_array_model): (kind, b, k1, k2, w,
    [(index, value), ...]) or None."""
    a = np.ascontiguousarray(a, np.int64)
    out = np.zeros(6 + 2 * 8, np.int64)
    st = _lib.as_fit_array_model(a.ctypes.data, a.shape[0], budget, out.ctypes.data)
    if STATUS.get(st) == "AS_ERR_NOT_FOUND":
        return None
    _ck(st)
    k, np_ = int(out[0]), int(out[5])
    return (k, int(out[1]), int(out[2]), int(out[3]), int(out[4]),
            [(int(out[6 + 2 * j]), int(out[7 + 2 * j])) for j in range(np_)])


def surrogate_fit_predict(X, y, Xq) -> np.ndarray:
    """The search's gradient-boosted tree cost model: fit on (X, y), predict Xq."""
    X = np.ascontiguousarray(X, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    Xq = np.ascontiguousarray(Xq, np.float64)
    out = np.zeros(Xq.shape[0], np.float64)
    _ck(_lib.as_surrogate_fit_predict(X.ctypes.data, y.ctypes.data, X.shape[0], X.shape[1], Xq.ctypes.data,
                                      Xq.shape[0], out.ctypes.data))
    return out


def version() -> str:
    return _lib.as_version().decode()


_hooks = None  # keeps the ctypes callbacks alive while installed


_hooks_ever = []  # every installed callback pair stays alive (the library frees with the allocating hooks)


def set_allocator(alloc=None, release=None):
    """as_set_allocator with Python callables alloc(nbytes, stream) -> int pointer (0 = out of
    memory) and release(ptr, stream); no arguments restores cudaMalloc/cudaFree."""
    global _hooks
    if alloc is None and release is None:
        _ck(_lib.as_set_allocator(_ALLOC_T(), _FREE_T(), None))
        _hooks = None
        return

    def _a(nbytes, stream, ctx):
        try:
            return alloc(nbytes, stream or 0) or None
        except Exception:
            return None

    def _r(ptr, stream, ctx):
        release(ptr, stream or 0)

    hooks = (_ALLOC_T(_a), _FREE_T(_r))
    _ck(_lib.as_set_allocator(hooks[0], hooks[1], None))
    _hooks = hooks
    _hooks_ever.append(hooks)  # memory made through these hooks is released through them later


def use_torch_allocator():
    """Route the library's device allocations through torch's caching allocator."""
    import torch
    set_allocator(lambda n, s: torch.cuda.caching_allocator_alloc(n, torch.cuda.current_device(), s),
                  lambda p, s: torch.cuda.caching_allocator_delete(p))


class Dist:
    """e: ROW_DIV multi-GPU SpMV of one rank (as_dist_*): band plan -> y_full, then the
    exchange ("none" | "nccl" AllGatherV | "peer" push over peer memory)."""

    def __init__(self, rank: int, world: int, device: int, nccl_id: bytes | None = None):
        h = _vp()
        idb = ctypes.create_string_buffer(nccl_id, AS_DIST_ID_BYTES) if nccl_id is not None else None
        _ck(_lib.as_dist_init(rank, world, idb, device, ctypes.byref(h)))
        self._h = h
        self.rank, self.world, self.device = rank, world, device

    @staticmethod
    def unique_id() -> bytes:
        b = ctypes.create_string_buffer(AS_DIST_ID_BYTES)
        _ck(_lib.as_dist_unique_id(b))
        return b.raw

    def set_cuts(self, cuts):
        c = np.ascontiguousarray(cuts, np.int64)
        if c.shape[0] != self.world + 1:
            raise AsError(1, "cuts must have world+1 entries")
        _ck(_lib.as_dist_set_cuts(self._h, c.ctypes.data))

    def ipc_handle(self, y_full) -> bytes:
        b = ctypes.create_string_buffer(AS_DIST_HANDLE_BYTES)
        _ck(_lib.as_dist_ipc_handle(self._h, _ptr(y_full), b))
        return b.raw

    def open_peers(self, y_full, handles):
        blob = b"".join(handles)
        if len(blob) != AS_DIST_HANDLE_BYTES * self.world:
            raise AsError(1, "one handle per rank expected")
        buf = ctypes.create_string_buffer(blob, len(blob))
        _ck(_lib.as_dist_open_peers(self._h, _ptr(y_full), buf))

    def set_windows(self, spans):
        """Halo windows: spans[q] = (first, last) row of y_full rank q reads (None: full bands)."""
        if spans is None:
            _ck(_lib.as_dist_set_windows(self._h, None))
            return
        w = np.ascontiguousarray(np.asarray(spans, np.int64).reshape(self.world, 2))
        _ck(_lib.as_dist_set_windows(self._h, w.ctypes.data))

    def spmv(self, plan: Plan, alpha, x_full, beta, y_full, exchange: str = "none", stream=None):
        a, b = plan._scalars(alpha, beta)
        _ck(_lib.as_spmv_dist(self._h, plan._h, ctypes.byref(a), _ptr(x_full), ctypes.byref(b), _ptr(y_full),
                              EXCHANGE[exchange], _stream_handle(stream)))

    def check(self):
        _ck(_lib.as_dist_check(self._h))

    def close(self):
        if getattr(self, "_h", None) and _lib:
            _lib.as_dist_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
