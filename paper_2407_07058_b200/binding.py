"""Thin ctypes binding of libappd (include/appd.h).  Argument marshalling only:
every step of the computation runs in libappd's CUDA kernels.  There is no CPU
fallback -- if the shared library is missing or no sm_100 device is present,
calls raise.

The C names are exposed one to one (appd_create, appd_solve_weights,
appd_solve_points, appd_destroy, ...); :class:`Context` wraps them for torch
tensors (torch supplies device memory and streams only).
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libappd.so")

APPD_OK = 0
STATUS = {
    0: "APPD_OK",
    1: "APPD_ERR_INVALID_ARGUMENT",
    2: "APPD_ERR_NONFINITE",
    3: "APPD_ERR_NOT_SYMMETRIC",
    4: "APPD_ERR_BAD_DIAGONAL",
    5: "APPD_ERR_UNSUPPORTED",
    6: "APPD_ERR_OUT_OF_MEMORY",
    7: "APPD_ERR_CUDA",
    8: "APPD_ERR_NCCL",
    9: "APPD_ERR_POISONED",
}
VARIANT_AUTO, VARIANT_PRIM, VARIANT_BORUVKA = 0, 1, 2
REDUCE_MIN, REDUCE_MAX = 0, 1
# appd_options.host_allreduce: int32 (*)(void* user, uint64_t* words, int64_t count, int32 op)
HOST_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.POINTER(ctypes.c_uint64),
                                     ctypes.c_int64, ctypes.c_int32)
# cudaStreamLegacy: the legacy default stream (torch's default stream has handle 0, which
# appd_set_stream would read as "library-owned stream")
CUDA_STREAM_LEGACY = 0x1
# appd_solve_points_sink: int32 (*)(void* user, int64 row0, int64 rows, const float* block)
BLOCK_SINK_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.POINTER(ctypes.c_float))


class appd_options(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("device", ctypes.c_int32),
        ("cuda_stream", ctypes.c_void_p),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("nccl_unique_id", ctypes.c_void_p),
        ("variant", ctypes.c_int32),
        ("validate", ctypes.c_int32),
        ("sense", ctypes.c_int32),
        ("timing", ctypes.c_int32),
        ("dendrogram", ctypes.c_int32),
        ("points_engine", ctypes.c_int32),
        ("topk", ctypes.c_int32),
        ("finish_k", ctypes.c_int32),
        ("metric", ctypes.c_int32),
        ("host_allreduce", HOST_ALLREDUCE_FN),
        ("host_allreduce_user", ctypes.c_void_p),
        ("timeout_ms", ctypes.c_int32),
        ("list_cap", ctypes.c_int32),
        ("wide_keys", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 3),
    ]


class appd_stats(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_uint32),
        ("variant", ctypes.c_int32),
        ("rounds", ctypes.c_int32),
        ("dendrogram", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("d", ctypes.c_int64),
        ("row0", ctypes.c_int64),
        ("rows", ctypes.c_int64),
        ("ms_validate", ctypes.c_double),
        ("ms_mst", ctypes.c_double),
        ("ms_sort", ctypes.c_double),
        ("ms_dendrogram", ctypes.c_double),
        ("ms_prep", ctypes.c_double),
        ("ms_fill", ctypes.c_double),
        ("ms_total", ctypes.c_double),
        ("kernel_launches", ctypes.c_int64),
        ("fill_launches", ctypes.c_int64),
        ("fill_bytes", ctypes.c_int64),
        ("tc_candidates", ctypes.c_int64),
        ("points_engine", ctypes.c_int32),
        ("exact_rounds", ctypes.c_int32),
        ("ms_scan", ctypes.c_double),
        ("scan_launches", ctypes.c_int64),
        ("tc_fallback_rows", ctypes.c_int64),
        ("ms_tcscan", ctypes.c_double),
        ("tcscan_launches", ctypes.c_int64),
        ("tcscan_flops", ctypes.c_double),
        ("topk", ctypes.c_int32),
        ("rescan_rounds", ctypes.c_int32),
        ("cache_invalid_rows", ctypes.c_int64),
        ("rescan_rows", ctypes.c_int64),
        ("rescan_blocks", ctypes.c_int64),
        ("cm_k", ctypes.c_int32),
        ("cm_retries", ctypes.c_int32),
        ("collectives", ctypes.c_int64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "struct_size"}


EXPORTS = [
    "appd_options_init", "appd_create", "appd_set_stream", "appd_solve_weights", "appd_solve_points",
    "appd_solve_points_host", "appd_solve_weights_host", "appd_floyd_weights", "appd_solve_points_stream", "appd_solve_points_sink", "appd_solve_weights_f64", "appd_destroy", "appd_row_range", "appd_row_range_of",
    "appd_points_weights", "appd_get_nccl_unique_id", "appd_get_stats", "appd_last_dendrogram",
    "appd_error_index", "appd_last_error", "appd_status_string", "appd_version",
]

_lib = None


def load(path: str | None = None):
    """Load libappd.so (raises OSError if it has not been built).  APPD_LIB names another
    build of the same ABI (the development library, tools/ only)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("APPD_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise OSError(f"{path} not built: run `python -m paper_2407_07058_b200.build`")
    L = ctypes.CDLL(path)
    P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
    L.appd_options_init.restype = None
    L.appd_options_init.argtypes = [ctypes.POINTER(appd_options)]
    L.appd_create.argtypes = [ctypes.POINTER(P), ctypes.POINTER(appd_options)]
    L.appd_set_stream.argtypes = [P, P]
    L.appd_solve_weights.argtypes = [P, P, I64, P]
    L.appd_solve_points.argtypes = [P, P, I64, I64, P]
    L.appd_solve_points_host.argtypes = [P, P, I64, I64, P]
    L.appd_solve_weights_host.argtypes = [P, P, I64, P]
    L.appd_floyd_weights.argtypes = [P, P, I64, P]
    L.appd_solve_weights_f64.argtypes = [P, P, I64, P]
    L.appd_solve_points_stream.argtypes = [P, P, I64, I64, P, I64]
    L.appd_solve_points_sink.argtypes = [P, P, I64, I64, I64, BLOCK_SINK_FN, P]
    L.appd_destroy.restype = None
    L.appd_destroy.argtypes = [P]
    L.appd_row_range.argtypes = [P, I64, ctypes.POINTER(I64), ctypes.POINTER(I64)]
    L.appd_row_range_of.argtypes = [I64, I32, I32, ctypes.POINTER(I64), ctypes.POINTER(I64)]
    L.appd_points_weights.argtypes = [P, P, I64, I64, I64, I64, P]
    L.appd_get_nccl_unique_id.argtypes = [P]
    L.appd_get_stats.argtypes = [P, ctypes.POINTER(appd_stats)]
    L.appd_last_dendrogram.argtypes = [P, P, P, I64]
    L.appd_error_index.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
    L.appd_last_error.restype = ctypes.c_char_p
    L.appd_last_error.argtypes = [P]
    L.appd_status_string.restype = ctypes.c_char_p
    L.appd_status_string.argtypes = [ctypes.c_int]
    L.appd_version.restype = ctypes.c_char_p
    L.appd_version.argtypes = []
    for name in EXPORTS:
        getattr(L, name)
    _lib = L
    return L


class AppdError(RuntimeError):
    def __init__(self, status: int, message: str, index=None):
        self.status = status
        self.name = STATUS.get(status, str(status))
        self.index = index
        super().__init__(f"{self.name}: {message}")


def _ptr(t) -> int:
    return int(t.data_ptr())


def _check_tensor(t, name, dtype_name="float32"):
    import torch

    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor")
    want = getattr(torch, dtype_name)
    if t.dtype != want:
        raise TypeError(f"{name} must be {dtype_name} (got {t.dtype})")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


# ---- one-to-one C names ----------------------------------------------------
def appd_row_range_of(n: int, rank: int, world: int):
    L = load()
    r0, rows = ctypes.c_int64(), ctypes.c_int64()
    s = L.appd_row_range_of(n, rank, world, ctypes.byref(r0), ctypes.byref(rows))
    if s != APPD_OK:
        raise AppdError(s, "appd_row_range_of")
    return r0.value, rows.value


def appd_get_nccl_unique_id() -> bytes:
    L = load()
    buf = (ctypes.c_uint8 * 128)()
    s = L.appd_get_nccl_unique_id(buf)
    if s != APPD_OK:
        raise AppdError(s, "appd_get_nccl_unique_id")
    return bytes(buf)


def appd_version() -> str:
    return load().appd_version().decode()


class Context:
    """A libappd context (appd_create / appd_destroy) bound to one CUDA device."""

    def __init__(self, device: int = 0, stream=None, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 variant: int = VARIANT_AUTO, validate: bool = True, sense: int = 1, timing: bool = False,
                 dendrogram: int = 0, points_engine: int = 0, topk: int = 0,
                 finish_k: int = 0, metric: int = 0, host_allreduce=None, timeout_ms: int = 0,
                 list_cap: int = 0, wide_keys: int = 0):
        """stream: a cudaStream_t handle (int) every call runs on; None (default) follows
        torch.cuda.current_stream(device) at each call, so the library's work is ordered
        with the torch kernels that produced its inputs and that read its outputs.
        host_allreduce: world > 1 exchange through host memory instead of NCCL, a Python
        callable (words: numpy uint64 array, op: REDUCE_MIN / REDUCE_MAX) -> None that
        all-reduces `words` in place over the ranks (e.g. torch.distributed with gloo)."""
        L = load()
        o = appd_options()
        L.appd_options_init(ctypes.byref(o))
        o.device = device
        self._follow_torch_stream = stream is None
        o.cuda_stream = stream if stream is not None else self._torch_stream(device)
        o.rank, o.world = rank, world
        o.timeout_ms = timeout_ms
        o.list_cap = list_cap
        o.wide_keys = wide_keys
        self._xchg = None
        if host_allreduce is not None:
            import numpy as np

            def _cb(user, words, count, op, _f=host_allreduce):
                try:
                    arr = np.ctypeslib.as_array(words, shape=(count,))
                    _f(arr, int(op))
                    return 0
                except Exception:  # noqa: BLE001 -- reported to the library as a failed exchange
                    import traceback

                    traceback.print_exc()
                    return 1

            self._xchg = HOST_ALLREDUCE_FN(_cb)  # kept alive with the context
            o.host_allreduce = self._xchg
        self._id = None
        if nccl_id is not None:
            self._id = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
            o.nccl_unique_id = ctypes.cast(self._id, ctypes.c_void_p)
        o.variant = variant
        o.validate = 1 if validate else 0
        o.sense = sense
        o.timing = 1 if timing else 0
        o.dendrogram = dendrogram
        o.points_engine = points_engine
        o.topk = topk
        o.finish_k = finish_k
        o.metric = metric
        h = ctypes.c_void_p()
        s = L.appd_create(ctypes.byref(h), ctypes.byref(o))
        if s != APPD_OK:
            raise AppdError(s, "appd_create")
        self._h = h
        self._L = L
        self._stream_h = o.cuda_stream
        self.device = device
        self.rank, self.world = rank, world

    # -- helpers --
    @staticmethod
    def _torch_stream(device):
        try:
            import torch

            if not torch.cuda.is_available():
                return None
            h = torch.cuda.current_stream(device).cuda_stream
            return h if h else CUDA_STREAM_LEGACY
        except Exception:  # noqa: BLE001
            return None

    def _sync_stream(self):
        """Follow torch's current stream (inputs made by pending torch kernels)."""
        if self._follow_torch_stream:
            h = self._torch_stream(self.device)
            if h is not None and h != self._stream_h:
                s = self._L.appd_set_stream(self._h, h)
                if s != APPD_OK:
                    self._raise(s, "appd_set_stream")
                self._stream_h = h

    def _raise(self, s, what):
        i, j = ctypes.c_int64(-1), ctypes.c_int64(-1)
        self._L.appd_error_index(self._h, ctypes.byref(i), ctypes.byref(j))
        msg = self._L.appd_last_error(self._h).decode()
        idx = (i.value, j.value) if i.value >= 0 else None
        raise AppdError(s, f"{what}: {msg}", idx)

    def set_stream(self, stream):
        self._follow_torch_stream = False
        self._stream_h = stream
        s = self._L.appd_set_stream(self._h, stream)
        if s != APPD_OK:
            self._raise(s, "appd_set_stream")

    def row_range(self, n: int):
        r0, rows = ctypes.c_int64(), ctypes.c_int64()
        s = self._L.appd_row_range(self._h, n, ctypes.byref(r0), ctypes.byref(rows))
        if s != APPD_OK:
            self._raise(s, "appd_row_range")
        return r0.value, rows.value

    def _out(self, n, M):
        import torch

        _, rows = self.row_range(n)
        if M is None:
            M = torch.empty((rows, n), dtype=torch.float32, device=f"cuda:{self.device}")
        _check_tensor(M, "M")
        if M.numel() != rows * n:
            raise ValueError(f"M must hold {rows} x {n} floats")
        return M

    # -- the four calls of the north star --
    def solve_weights(self, W, M=None):
        """appd_solve_weights: W is this rank's rows x n block (n x n for world 1)."""
        _check_tensor(W, "W")
        n = W.shape[-1]
        _, rows = self.row_range(n)
        if tuple(W.shape) != (rows, n):
            raise ValueError(f"W must be this rank's {rows} x {n} row block (got {tuple(W.shape)})")
        M = self._out(n, M)
        self._sync_stream()
        s = self._L.appd_solve_weights(self._h, _ptr(W), n, _ptr(M))
        if s != APPD_OK:
            self._raise(s, "appd_solve_weights")
        return M

    def floyd_weights(self, W, M=None):
        """appd_floyd_weights (NEXT-2): the minimax Floyd–Warshall closure of the n x n W
        on the GPU (one rank); M must not alias W."""
        _check_tensor(W, "W")
        n = W.shape[-1]
        if tuple(W.shape) != (n, n):
            raise ValueError(f"W must be n x n (got {tuple(W.shape)})")
        M = self._out(n, M)
        self._sync_stream()
        s = self._L.appd_floyd_weights(self._h, _ptr(W), n, _ptr(M))
        if s != APPD_OK:
            self._raise(s, "appd_floyd_weights")
        return M

    def solve_weights_f64(self, W, M=None):
        """appd_solve_weights_f64 (NEXT-3): W and M are n x n float64 CUDA tensors (one rank)."""
        import torch

        _check_tensor(W, "W", "float64")
        n = W.shape[-1]
        if tuple(W.shape) != (n, n):
            raise ValueError(f"W must be n x n (got {tuple(W.shape)})")
        if M is None:
            M = torch.empty((n, n), dtype=torch.float64, device=f"cuda:{self.device}")
        _check_tensor(M, "M", "float64")
        if M.numel() != n * n:
            raise ValueError(f"M must hold {n} x {n} doubles")
        self._sync_stream()
        s = self._L.appd_solve_weights_f64(self._h, _ptr(W), n, _ptr(M))
        if s != APPD_OK:
            self._raise(s, "appd_solve_weights_f64")
        return M

    def solve_points_stream(self, X, M, block_rows=0):
        """appd_solve_points_stream (NEXT-4): X and M are HOST (CPU) float32 tensors, M n x n
        (pinned for overlap); M is written in blocks of block_rows rows (0 = auto)."""
        _check_tensor(X, "X")
        _check_tensor(M, "M")
        n, d = X.shape
        if X.is_cuda or M.is_cuda:
            raise ValueError("solve_points_stream takes host tensors")
        if M.numel() != n * n:
            raise ValueError(f"M must hold {n} x {n} floats")
        self._sync_stream()
        s = self._L.appd_solve_points_stream(self._h, _ptr(X), n, d, _ptr(M), int(block_rows))
        if s != APPD_OK:
            self._raise(s, "appd_solve_points_stream")
        return M

    def solve_points_sink(self, X, sink, block_rows=0):
        """appd_solve_points_sink (NEXT-4): X is a HOST float32 tensor; sink(row0, block) is
        called in row order with each block as a numpy (rows x n) float32 view that is only
        valid during the call (copy it to keep it).  Returns nothing; M is never held."""
        import numpy as np

        _check_tensor(X, "X")
        if X.is_cuda:
            raise ValueError("solve_points_sink takes a host X")
        n, d = X.shape
        err = []

        def _cb(user, row0, rows, block, _n=n):
            try:
                sink(int(row0), np.ctypeslib.as_array(block, shape=(int(rows), _n)))
                return 0
            except Exception as e:  # noqa: BLE001 -- the library stops the solve
                err.append(e)
                return 1

        cb = BLOCK_SINK_FN(_cb)
        self._sync_stream()
        s = self._L.appd_solve_points_sink(self._h, _ptr(X), n, d, int(block_rows), cb, None)
        if err:
            raise err[0]
        if s != APPD_OK:
            self._raise(s, "appd_solve_points_sink")

    def solve_points(self, X, M=None):
        """appd_solve_points: X is n x d (replicated on every rank)."""
        _check_tensor(X, "X")
        n, d = X.shape
        M = self._out(n, M)
        self._sync_stream()
        s = self._L.appd_solve_points(self._h, _ptr(X), n, d, _ptr(M))
        if s != APPD_OK:
            self._raise(s, "appd_solve_points")
        return M

    def solve_points_host(self, X, M):
        """appd_solve_points_host: X (n x d) and M (rows x n) are CPU tensors (pinned for speed)."""
        _check_tensor(X, "X")
        _check_tensor(M, "M")
        n, d = X.shape
        _, rows = self.row_range(n)
        if M.numel() != rows * n:
            raise ValueError(f"M must hold {rows} x {n} floats")
        self._sync_stream()
        s = self._L.appd_solve_points_host(self._h, _ptr(X), n, d, _ptr(M))
        if s != APPD_OK:
            self._raise(s, "appd_solve_points_host")
        return M

    def solve_weights_host(self, W, M):
        _check_tensor(W, "W")
        _check_tensor(M, "M")
        n = W.shape[-1]
        _, rows = self.row_range(n)
        if tuple(W.shape) != (rows, n) or M.numel() != rows * n:
            raise ValueError(f"W and M must be this rank's {rows} x {n} row blocks")
        self._sync_stream()
        s = self._L.appd_solve_weights_host(self._h, _ptr(W), n, _ptr(M))
        if s != APPD_OK:
            self._raise(s, "appd_solve_weights_host")
        return M

    def points_weights(self, X, row0: int = 0, rows: int | None = None, out=None):
        """appd_points_weights: R1 weights of rows [row0, row0+rows) (K11 test hook)."""
        import torch

        _check_tensor(X, "X")
        n, d = X.shape
        rows = n - row0 if rows is None else rows
        if out is None:
            out = torch.empty((rows, n), dtype=torch.float32, device=X.device)
        self._sync_stream()
        s = self._L.appd_points_weights(self._h, _ptr(X), n, d, row0, rows, _ptr(out))
        if s != APPD_OK:
            self._raise(s, "appd_points_weights")
        return out

    def stats(self) -> dict:
        st = appd_stats()
        st.struct_size = ctypes.sizeof(appd_stats)
        s = self._L.appd_get_stats(self._h, ctypes.byref(st))
        if s != APPD_OK:
            self._raise(s, "appd_get_stats")
        return st.as_dict()

    def last_dendrogram(self, n: int):
        import numpy as np

        pi = np.empty(n, np.int32)
        h = np.empty(max(n - 1, 1), np.float32)
        s = self._L.appd_last_dendrogram(self._h, pi.ctypes.data, h.ctypes.data, n)
        if s != APPD_OK:
            self._raise(s, "appd_last_dendrogram")
        return pi, h[: n - 1]

    def close(self):
        if getattr(self, "_h", None):
            self._L.appd_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def appd_create(**kw) -> Context:
    return Context(**kw)


def appd_solve_weights(ctx: Context, W, M=None):
    return ctx.solve_weights(W, M)


def appd_solve_points(ctx: Context, X, M=None):
    return ctx.solve_points(X, M)


def appd_destroy(ctx: Context) -> None:
    ctx.close()
