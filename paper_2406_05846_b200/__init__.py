"""Python binding of libstrom (the B200-native sGS-ADMM hot path).

Argument marshalling only: every step of Algorithm 1 runs in
the sm_100a kernels of `libstrom.so` behind the C-ABI declared in
`include/strom.h`. Function and method names mirror the C entry points. There is
no CPU fallback: importing works without a GPU (for build/symbol checks), but
`strom_admm_setup` fails loudly when no CUDA device or no library is present.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# STROM_LIB overrides the in-tree library (A/B timing of two builds)
LIB_PATH = os.environ.get("STROM_LIB") or os.path.join(_HERE, "libstrom.so")

STATUS = {0: "STROM_OK", 1: "STROM_MAXITER", -1: "STROM_EINVAL", -2: "STROM_ENOMEM",
          -3: "STROM_EFACTOR", -4: "STROM_EEIG", -5: "STROM_EDIVERGED", -6: "STROM_ECUDA",
          -7: "STROM_ENCCL", -8: "STROM_ENOTIMPL"}
STROM_OK, STROM_MAXITER = 0, 1

# Every symbol include/strom.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "strom_sdp_create", "strom_sdp_destroy", "strom_sdp_dims", "strom_admm_default_config",
    "strom_admm_setup", "strom_admm_destroy", "strom_admm_set_start",
    "strom_admm_set_start_device", "strom_admm_iterate", "strom_admm_solve", "strom_admm_get",
    "strom_admm_get_device", "strom_admm_lower_bound", "strom_admm_extract", "strom_admm_launches_per_iter",
    "strom_admm_factor_info", "strom_admm_kernel_times", "strom_admm_kernel_work", "strom_nccl_get_unique_id", "strom_last_error", "strom_version",
    "strom_debug_project_psd", "strom_debug_spmv", "strom_debug_solve", "strom_debug_host_solve",
    "strom_debug_eps", "strom_debug_link_virtual", "strom_debug_iterate_virtual",
    "strom_debug_host_part", "strom_debug_setup_virtual",
    "strom_batch_create", "strom_batch_destroy", "strom_batch_iterate", "strom_batch_solve",
    "strom_admm_reconfigure", "strom_admm_setup_times",
]


class StromError(RuntimeError):
    def __init__(self, status: int, where: str, msg: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")
        self.status = status


class strom_block(C.Structure):
    _fields_ = [("n", C.c_int32), ("stage", C.c_int32), ("nrows", C.c_int32),
                ("rows", C.POINTER(C.c_int32)), ("rowptr", C.POINTER(C.c_int64)),
                ("col", C.POINTER(C.c_int32)), ("val", C.POINTER(C.c_double)),
                ("C_svec", C.POINTER(C.c_double))]


class strom_admm_config(C.Structure):
    _fields_ = [("sigma", C.c_double), ("tau", C.c_double), ("eps_rel", C.c_double),
                ("eps", C.c_double), ("sigma_period", C.c_int32), ("sigma_ratio", C.c_double),
                ("sigma_factor", C.c_double), ("sigma_min", C.c_double), ("sigma_max", C.c_double),
                ("check_every", C.c_int32), ("eig_max_sweeps", C.c_int32), ("eig_tol", C.c_double),
                ("eig_warm", C.c_int32), ("eig_cold_every", C.c_int32)]


class strom_residuals(C.Structure):
    _fields_ = [("iter", C.c_int64), ("eta_p", C.c_double), ("eta_d", C.c_double),
                ("eta_g", C.c_double), ("pobj", C.c_double), ("dobj", C.c_double),
                ("sigma", C.c_double), ("eta_x", C.c_double), ("eig_sweeps", C.c_int64),
                ("iter_eta", C.c_int64 * 3)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["iter_eta"] = {"1e-4": self.iter_eta[0] or None, "1e-5": self.iter_eta[1] or None,
                         "1e-6": self.iter_eta[2] or None}
        return d


_lib: Optional[C.CDLL] = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load libstrom.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libstrom.so not built at {path}; run paper_2406_05846_b200/build.py")
    # torch first: libstrom resolves libnccl.so.2 to the NCCL torch already loaded (the
    # system libnccl loaded first would leave torch's CUDA library with unresolved
    # NCCL symbols when torch is imported afterwards)
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    lib = C.CDLL(path)
    P, VP, D, I32, I64 = C.POINTER, C.c_void_p, C.c_double, C.c_int32, C.c_int64
    sig = {
        "strom_sdp_create": (I32, [P(VP), I32, P(strom_block), I32, P(D)]),
        "strom_sdp_destroy": (None, [VP]),
        "strom_sdp_dims": (I32, [VP, P(I64), P(I32), P(I32)]),
        "strom_admm_default_config": (None, [P(strom_admm_config)]),
        "strom_admm_setup": (I32, [P(VP), VP, P(strom_admm_config), C.c_int, VP, VP, C.c_int, C.c_int]),
        "strom_admm_destroy": (None, [VP]),
        "strom_admm_set_start": (I32, [VP, P(D), P(D), P(D)]),
        "strom_admm_reconfigure": (I32, [VP, P(strom_admm_config)]),
        "strom_admm_setup_times": (I32, [VP, P(D)]),
        "strom_admm_set_start_device": (I32, [VP, VP, VP, VP]),
        "strom_admm_iterate": (I32, [VP, I64]),
        "strom_admm_solve": (I32, [VP, D, I64, P(I64)]),
        "strom_admm_get": (I32, [VP, P(D), P(D), P(D), P(strom_residuals)]),
        "strom_admm_get_device": (I32, [VP, VP, VP, VP]),
        "strom_admm_lower_bound": (I32, [VP, P(D), P(D), P(D)]),
        "strom_admm_extract": (I32, [VP, P(D), P(D)]),
        "strom_admm_launches_per_iter": (I32, [VP]),
        "strom_admm_factor_info": (I32, [VP, P(I64), P(I32), P(I32), P(I32)]),
        "strom_admm_kernel_times": (I32, [VP, P(D), P(C.c_char_p), I32]),
        "strom_admm_kernel_work": (I32, [VP, C.c_char_p, P(D), P(D)]),
        "strom_nccl_get_unique_id": (I32, [VP]),
        "strom_last_error": (C.c_char_p, []),
        "strom_version": (C.c_char_p, []),
        "strom_debug_project_psd": (I32, [VP, P(D), D, P(D), P(D)]),
        "strom_debug_spmv": (I32, [VP, P(D), P(D), P(D), P(D)]),
        "strom_debug_solve": (I32, [VP, P(D), P(D)]),
        "strom_debug_host_solve": (I32, [VP, P(strom_admm_config), P(D), P(D)]),
        "strom_debug_eps": (D, [VP]),
        "strom_batch_create": (I32, [P(VP), P(VP), I32, I32, VP]),
        "strom_batch_destroy": (None, [VP]),
        "strom_batch_iterate": (I32, [VP, I64]),
        "strom_batch_solve": (I32, [VP, D, I64, P(I64), P(I32)]),
        "strom_debug_host_part": (I32, [VP, P(strom_admm_config), I32, I32, P(D), P(D), P(D), P(D), P(I32)]),
        "strom_debug_link_virtual": (I32, [P(VP), I32, VP]),
        "strom_debug_setup_virtual": (I32, [P(VP), VP, P(strom_admm_config), C.c_int, VP, C.c_int, C.c_int]),
        "strom_debug_iterate_virtual": (I32, [P(VP), I32, I64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(st: int, where: str):
    if st not in (STROM_OK, STROM_MAXITER):
        raise StromError(st, where, load().strom_last_error().decode())
    return st


def _dptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def strom_admm_default_config(**over) -> strom_admm_config:
    cfg = strom_admm_config()
    load().strom_admm_default_config(C.byref(cfg))
    for k, v in over.items():
        setattr(cfg, k, v)
    return cfg


class StromSdp:
    """strom_sdp_create from a BlockSdp-like object (block_n, block_stage,
    block_offset, A_indptr/A_indices/A_data global CSR, b, C): splits A into the
    per-block CSR the C-ABI takes."""

    def __init__(self, sdp):
        lib = load()
        bn = np.asarray(sdp.block_n, dtype=np.int32)
        bst = np.asarray(sdp.block_stage, dtype=np.int32)
        bo = np.asarray(sdp.block_offset, dtype=np.int64)
        ip = np.asarray(sdp.A_indptr, dtype=np.int64)
        ind = np.asarray(sdp.A_indices, dtype=np.int64)
        dat = np.asarray(sdp.A_data, dtype=np.float64)
        m = int(np.asarray(sdp.b).shape[0])
        rows_of = np.repeat(np.arange(m, dtype=np.int64), np.diff(ip))
        blk = np.searchsorted(bo, ind, side="right") - 1
        order = np.argsort(blk, kind="stable")
        self._keep = []
        blocks = (strom_block * len(bn))()
        starts = np.searchsorted(blk[order], np.arange(len(bn) + 1))
        Cv = np.ascontiguousarray(np.asarray(sdp.C, dtype=np.float64))
        for beta in range(len(bn)):
            sel = order[starts[beta]:starts[beta + 1]]
            r = rows_of[sel]
            urows, first, counts = np.unique(r, return_index=True, return_counts=True)
            rp = np.zeros(len(urows) + 1, dtype=np.int64)
            rp[1:] = np.cumsum(counts)
            col = np.ascontiguousarray((ind[sel] - bo[beta]).astype(np.int32))
            val = np.ascontiguousarray(dat[sel])
            urows = np.ascontiguousarray(urows.astype(np.int32))
            cb = np.ascontiguousarray(Cv[bo[beta]:bo[beta + 1]])
            self._keep += [urows, rp, col, val, cb]
            blocks[beta] = strom_block(
                int(bn[beta]), int(bst[beta]), len(urows),
                urows.ctypes.data_as(C.POINTER(C.c_int32)), rp.ctypes.data_as(C.POINTER(C.c_int64)),
                col.ctypes.data_as(C.POINTER(C.c_int32)), val.ctypes.data_as(C.POINTER(C.c_double)),
                cb.ctypes.data_as(C.POINTER(C.c_double)))
        b = np.ascontiguousarray(np.asarray(sdp.b, dtype=np.float64))
        h = C.c_void_p()
        _check(lib.strom_sdp_create(C.byref(h), len(bn), blocks, m, _dptr(b)), "strom_sdp_create")
        self._keep = None
        self.handle = h
        self.m = m
        self.n = int(bo[-1])
        self.nblocks = len(bn)
        self.block_n = bn.copy()

    def dims(self):
        n, m, nb = C.c_int64(), C.c_int32(), C.c_int32()
        _check(load().strom_sdp_dims(self.handle, C.byref(n), C.byref(m), C.byref(nb)), "strom_sdp_dims")
        return n.value, m.value, nb.value

    def host_solve(self, r: np.ndarray, cfg: Optional[strom_admm_config] = None) -> np.ndarray:
        """strom_debug_host_solve (test hook: host execution of the setup factor)."""
        cfg = cfg or strom_admm_default_config()
        r = np.ascontiguousarray(r, dtype=np.float64)
        y = np.zeros(self.m)
        _check(load().strom_debug_host_solve(self.handle, C.byref(cfg), _dptr(r), _dptr(y)),
               "strom_debug_host_solve")
        return y

    def host_part(self, nranks: int, rank: int, r: np.ndarray, recv: Optional[np.ndarray] = None,
                  cfg: Optional[strom_admm_config] = None):
        """strom_debug_host_part (test hook): without `recv`, the rank's partial boundary
        right-hand side (nB doubles); with `recv` (the summed partials), the rank's rows of y."""
        cfg = cfg or strom_admm_default_config()
        r = np.ascontiguousarray(r, dtype=np.float64)
        nB = C.c_int32()
        lib = load()
        _check(lib.strom_debug_host_part(self.handle, C.byref(cfg), nranks, rank, _dptr(r), None, None, None,
                                         C.byref(nB)), "strom_debug_host_part")
        if recv is None:
            send = np.zeros(nB.value)
            _check(lib.strom_debug_host_part(self.handle, C.byref(cfg), nranks, rank, _dptr(r), _dptr(send),
                                             None, None, None), "strom_debug_host_part")
            return send
        recv = np.ascontiguousarray(recv, dtype=np.float64)
        y = np.zeros(self.m)
        _check(lib.strom_debug_host_part(self.handle, C.byref(cfg), nranks, rank, _dptr(r), None, _dptr(recv),
                                         _dptr(y), None), "strom_debug_host_part")
        return y

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.strom_sdp_destroy(self.handle)
            self.handle = None


def _torch_stream_ptr(stream):
    """cudaStream_t of a torch stream. torch's legacy default stream has handle 0,
    which the C-ABI would read as "create your own stream"; refuse it so that
    events recorded by the caller always see the solver's work."""
    if stream is None:
        return None
    ptr = int(stream.cuda_stream)
    if ptr == 0:
        raise ValueError("pass a non-default torch.cuda.Stream() (the legacy default stream is 0)")
    return C.c_void_p(ptr)


class StromAdmm:
    """strom_admm_setup and friends on one device / stream."""

    def __init__(self, sdp: StromSdp, cfg: Optional[strom_admm_config] = None, device: int = 0,
                 stream=None, rank: int = 0, nranks: int = 1, nccl_id: Optional[bytes] = None,
                 virtual: bool = False):
        """nranks > 1: one process per GPU, the same SDP and the same `nccl_id`
        (strom_nccl_get_unique_id() on rank 0, broadcast by the caller) on every rank;
        the chain is partitioned along the horizon.
        virtual=True (tests): rank `rank` of `nranks` in-process ranks on one device
        (strom_debug_setup_virtual; link them with strom_debug_link_virtual)."""
        lib = load()
        self.sdp = sdp
        self.cfg = cfg or strom_admm_default_config()
        h = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        if virtual:
            _check(lib.strom_debug_setup_virtual(C.byref(h), sdp.handle, C.byref(self.cfg), device,
                                                 _torch_stream_ptr(stream), rank, nranks), "strom_debug_setup_virtual")
        else:
            _check(lib.strom_admm_setup(C.byref(h), sdp.handle, C.byref(self.cfg), device,
                                        _torch_stream_ptr(stream), idbuf, rank, nranks), "strom_admm_setup")
        self.handle = h
        self.n, self.m = sdp.n, sdp.m
        self.device, self.stream = device, stream

    def _device_arg(self, t, count: int, what: str):
        """A torch CUDA tensor handed to the C-ABI as a raw device pointer: float64,
        contiguous, exactly `count` elements, on the handle's device (the library reads
        or writes count doubles through it)."""
        if t is None:
            return None
        import torch
        if not (t.is_cuda and t.device.index == self.device):
            raise ValueError(f"{what}: tensor must live on cuda:{self.device}")
        if t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != count:
            raise ValueError(f"{what}: need a contiguous float64 tensor of {count} elements, got "
                             f"{t.dtype} {tuple(t.shape)} contiguous={t.is_contiguous()}")
        return C.c_void_p(int(t.data_ptr()))

    def _order_before(self):
        """The library copies on the handle's stream: make it wait for the caller's
        current stream (which produced the tensors)."""
        import torch
        cur = torch.cuda.current_stream(self.device)
        if self.stream is not None:
            self.stream.wait_stream(cur)
        else:
            cur.synchronize()

    def _order_after(self):
        """... and make the caller's current stream wait for the handle's copies."""
        import torch
        cur = torch.cuda.current_stream(self.device)
        if self.stream is not None:
            cur.wait_stream(self.stream)
        else:
            torch.cuda.synchronize(self.device)

    def reconfigure(self, **over):
        """strom_admm_reconfigure: new sigma / tau / sigma policy / eigensolver settings,
        effective at the next set_start."""
        for k, v in over.items():
            setattr(self.cfg, k, v)
        return _check(load().strom_admm_reconfigure(self.handle, C.byref(self.cfg)), "strom_admm_reconfigure")

    def set_start(self, X=None, y=None, S=None):
        f = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64)
        X, y, S = f(X), f(y), f(S)
        return _check(load().strom_admm_set_start(self.handle, _dptr(X), _dptr(y), _dptr(S)),
                      "strom_admm_set_start")

    def set_start_device(self, X=None, y=None, S=None):
        args = (self._device_arg(X, self.n, "X"), self._device_arg(y, self.m, "y"),
                self._device_arg(S, self.n, "S"))
        self._order_before()
        return _check(load().strom_admm_set_start_device(self.handle, *args), "strom_admm_set_start_device")

    def iterate(self, iters: int):
        return _check(load().strom_admm_iterate(self.handle, int(iters)), "strom_admm_iterate")

    def solve(self, tol: float, maxiter: int):
        done = C.c_int64()
        st = _check(load().strom_admm_solve(self.handle, float(tol), int(maxiter), C.byref(done)),
                    "strom_admm_solve")
        return st == STROM_OK, done.value

    def get(self, X=True, y=True, S=True):
        Xa = np.zeros(self.n) if X else None
        ya = np.zeros(self.m) if y else None
        Sa = np.zeros(self.n) if S else None
        res = strom_residuals()
        _check(load().strom_admm_get(self.handle, _dptr(Xa), _dptr(ya), _dptr(Sa), C.byref(res)),
               "strom_admm_get")
        return Xa, ya, Sa, res.as_dict()

    def get_device(self, X=None, y=None, S=None):
        args = (self._device_arg(X, self.n, "X"), self._device_arg(y, self.m, "y"),
                self._device_arg(S, self.n, "S"))
        self._order_before()          # the caller may still be reading the buffers
        st = _check(load().strom_admm_get_device(self.handle, *args), "strom_admm_get_device")
        self._order_after()
        return st

    def residuals(self):
        return self.get(False, False, False)[3]

    def lower_bound(self, R_beta: np.ndarray):
        R = np.ascontiguousarray(R_beta, dtype=np.float64)
        lb = C.c_double()
        lam = np.zeros(self.sdp.nblocks)
        _check(load().strom_admm_lower_bound(self.handle, _dptr(R), C.byref(lb), _dptr(lam)),
               "strom_admm_lower_bound")
        return lb.value, lam

    def extract(self):
        """(lam12 [nblocks, 2], [top unit eigenvector of each block]) of the current X,
        computed on the device (strom_admm_extract)."""
        nb = self.sdp.nblocks
        bn = np.asarray(self.sdp.block_n, dtype=np.int64)
        lam12 = np.zeros(2 * nb)
        vtop = np.zeros(int(bn.sum()))
        _check(load().strom_admm_extract(self.handle, _dptr(lam12), _dptr(vtop)), "strom_admm_extract")
        offs = np.concatenate([[0], np.cumsum(bn)])
        return lam12.reshape(nb, 2), [vtop[offs[k]:offs[k + 1]] for k in range(nb)]

    def kernel_times(self):
        """[(kernel name, ms)] of the instrumented iteration of the last graph launch."""
        cap = 256
        ms = np.zeros(cap)
        names = (C.c_char_p * cap)()
        cnt = load().strom_admm_kernel_times(self.handle, _dptr(ms), names, cap)
        if cnt < 0:
            _check(cnt, "strom_admm_kernel_times")
        return [(names[i].decode(), float(ms[i])) for i in range(min(cnt, cap))]

    def kernel_work(self, name: str):
        """(algorithmic bytes, flops) of one launch of the marked kernel `name`
        (strom_admm_kernel_work); None for a name without a table entry (K-EIG classes)."""
        b, f = C.c_double(), C.c_double()
        if load().strom_admm_kernel_work(self.handle, name.encode(), C.byref(b), C.byref(f)) != 0:
            return None
        return b.value, f.value

    def setup_times(self):
        """Setup phases in ms (strom_admm_setup_times)."""
        ms = np.zeros(5)
        _check(load().strom_admm_setup_times(self.handle, _dptr(ms)), "strom_admm_setup_times")
        return dict(zip(("host_factor", "uploads", "device_factor", "eig_state", "graph_capture"), ms.tolist()))

    def launches_per_iter(self) -> int:
        return int(load().strom_admm_launches_per_iter(self.handle))

    def factor_info(self):
        b, nl, ns, nu = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        _check(load().strom_admm_factor_info(self.handle, C.byref(b), C.byref(nl), C.byref(ns), C.byref(nu)),
               "strom_admm_factor_info")
        return {"device_bytes": b.value, "leaf_rows": nl.value, "sep_rows": ns.value, "unique_dense": nu.value}

    def eps(self) -> float:
        return float(load().strom_debug_eps(self.handle))

    # ---- test hooks ----
    def debug_project_psd(self, Xb: np.ndarray, sigma: float):
        Xb = np.ascontiguousarray(Xb, dtype=np.float64)
        S = np.zeros(self.n); Pi = np.zeros(self.n)
        _check(load().strom_debug_project_psd(self.handle, _dptr(Xb), float(sigma), _dptr(S), _dptr(Pi)),
               "strom_debug_project_psd")
        return S, Pi

    def debug_spmv(self, X: Optional[np.ndarray] = None, y: Optional[np.ndarray] = None):
        X = None if X is None else np.ascontiguousarray(X, dtype=np.float64)
        y = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
        AX = np.zeros(self.m) if X is not None else None
        Aty = np.zeros(self.n) if y is not None else None
        _check(load().strom_debug_spmv(self.handle, _dptr(X), _dptr(AX), _dptr(y), _dptr(Aty)),
               "strom_debug_spmv")
        return AX, Aty

    def debug_solve(self, r: np.ndarray) -> np.ndarray:
        r = np.ascontiguousarray(r, dtype=np.float64)
        y = np.zeros(self.m)
        _check(load().strom_debug_solve(self.handle, _dptr(r), _dptr(y)), "strom_debug_solve")
        return y

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.strom_admm_destroy(self.handle)
            self.handle = None


class StromBatch:
    """strom_batch_create: several StromAdmm handles (one device, own streams) iterated by
    one CUDA graph with a concurrent branch per instance (NEXT-2)."""

    def __init__(self, admms, iters_per_launch: int = 50, stream=None):
        lib = load()
        self.admms = list(admms)            # the handles must outlive the batch
        arr = (C.c_void_p * len(self.admms))(*[a.handle.value for a in self.admms])
        h = C.c_void_p()
        _check(lib.strom_batch_create(C.byref(h), arr, len(self.admms), int(iters_per_launch),
                                      _torch_stream_ptr(stream)), "strom_batch_create")
        self.handle, self.K = h, int(iters_per_launch)

    def iterate(self, iters: int):
        return _check(load().strom_batch_iterate(self.handle, int(iters)), "strom_batch_iterate")

    def solve(self, tol: float, maxiter: int):
        """-> (all converged, iterations per instance, converged flags per instance)"""
        B = len(self.admms)
        done = np.zeros(B, dtype=np.int64)
        conv = np.zeros(B, dtype=np.int32)
        st = _check(load().strom_batch_solve(self.handle, float(tol), int(maxiter),
                                             done.ctypes.data_as(C.POINTER(C.c_int64)),
                                             conv.ctypes.data_as(C.POINTER(C.c_int32))), "strom_batch_solve")
        return st == STROM_OK, done, conv.astype(bool)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.strom_batch_destroy(self.handle)
            self.handle = None


def strom_nccl_get_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(load().strom_nccl_get_unique_id(buf), "strom_nccl_get_unique_id")
    return buf.raw


def strom_debug_link_virtual(admms, sdp: StromSdp):
    """Test harness: len(admms) handles of the same SDP on one device act as the ranks of
    the multi-GPU mode (exchange by device copies instead of NCCL)."""
    arr = (C.c_void_p * len(admms))(*[a.handle.value for a in admms])
    _check(load().strom_debug_link_virtual(arr, len(admms), sdp.handle), "strom_debug_link_virtual")


def strom_debug_iterate_virtual(admms, iters: int):
    arr = (C.c_void_p * len(admms))(*[a.handle.value for a in admms])
    _check(load().strom_debug_iterate_virtual(arr, len(admms), int(iters)), "strom_debug_iterate_virtual")


def strom_version() -> str:
    return load().strom_version().decode()
