"""ctypes binding of the bkfac C ABI (include/bkfac.h).  Argument marshalling only:
every step of the hot path runs in the CUDA kernels of ``libbkfac.so``.

Tensor conventions (PyTorch, all fp32, CUDA):
  U: shape (r, n)   == col-major n x r          M: shape (c, n) == col-major n x c
  D: shape (r,)                                  K_dense: shape (n, n) (symmetric)
  J, S: shape (d_G, d_A)  == row-major d_G x d_A (weight.grad layout)
U, M, J, S (and G, A of Algorithm 8) need unit stride along their last dimension only: a
view t[:, :n] of a padded (b, ld) buffer is passed with its row stride as the operand's
leading dimension (bkfac.h "Leading dimensions"; ld a multiple of 32 takes the 16-byte
load path).  D, K_dense and index arrays must be contiguous.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbkfac.so")

BKFAC_FACTOR_DENSE_EA = 1
BKFAC_FACTOR_FULL_RANK = 2
BKFAC_BRAND_NO_REORTH = 1
BKFAC_BRAND_NO_REFRESH = 2
BKFAC_PRECOND_CONTINUATION = 1
BKFAC_PRECOND_LAMBDA_RELATIVE = 2
BKFAC_GEMM_TCGEN05 = 0
BKFAC_GEMM_SIMT = 1
BKFAC_GEMM_TCGEN05_PAIR = 2
BKFAC_OPT_TWO_STAGE = 1
BKFAC_OPT_GT_CLUSTER = 2
BKFAC_OPT_GEMM_PAIR = 3
BKFAC_OPT_GEMM_SIMT = 4
BKFAC_OPT_EA_MODE = 5
BKFAC_OPT_EA_CAP = 6
BKFAC_OPT_SYT_CLUSTER = 7
BKFAC_OPT_BT_SIMT = 8
BKFAC_OPT_CHOL_BLOCKED = 9
BKFAC_OPT_NVTX = 10
BKFAC_OPT_SBR_X = 11
BKFAC_OPT_GEMM_CAP = 12
BKFAC_OPT_PREC_BLOCK = 13

STATUS = {0: "BKFAC_OK", 1: "BKFAC_ERR_INVALID_ARG", 2: "BKFAC_ERR_DIM", 3: "BKFAC_ERR_RANK",
          4: "BKFAC_ERR_ALIAS", 5: "BKFAC_ERR_WORKSPACE", 6: "BKFAC_ERR_CUDA",
          7: "BKFAC_ERR_NUMERIC", 8: "BKFAC_ERR_UNSUPPORTED"}

EXPORTED = ["bkfac_init", "bkfac_set_option", "bkfac_workspace_bytes", "bkfac_set_workspace", "bkfac_destroy",
            "bkfac_brand_update", "bkfac_brand_ea_update", "bkfac_ea_accumulate", "bkfac_ea_accumulate_batch",
            "bkfac_rsvd_overwrite", "bkfac_rsvd_overwrite_batch",
            "bkfac_precondition", "bkfac_precondition_factored", "bkfac_light_correction", "bkfac_gaussian_sketch", "bkfac_check", "bkfac_launch_count",
            "bkfac_profile_enable", "bkfac_profile_read", "bkfac_profile_count", "bkfac_profile_read_range", "bkfac_status_string",
            "bkfac_build_info", "bkfac_gemm"]


class BkfacError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {STATUS.get(code, code)}")
        self.code = code


class FactorDesc(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int), ("r", ctypes.c_int), ("c_max", ctypes.c_int),
                ("flags", ctypes.c_int)]


class LayerDesc(ctypes.Structure):
    _fields_ = [("d_G", ctypes.c_int), ("d_A", ctypes.c_int), ("r_G", ctypes.c_int),
                ("r_A", ctypes.c_int), ("n_max", ctypes.c_int)]


class BrandArgs(ctypes.Structure):
    _fields_ = [("factor", ctypes.c_int), ("U_in", ctypes.c_void_p), ("D_in", ctypes.c_void_p),
                ("M", ctypes.c_void_p), ("c", ctypes.c_int), ("U_out", ctypes.c_void_p),
                ("D_out", ctypes.c_void_p), ("alpha", ctypes.c_float), ("beta", ctypes.c_float),
                ("flags", ctypes.c_int), ("ld_U", ctypes.c_int), ("ld_M", ctypes.c_int)]


class EaArgs(ctypes.Structure):
    _fields_ = [("factor", ctypes.c_int), ("K_dense", ctypes.c_void_p), ("M", ctypes.c_void_p),
                ("c", ctypes.c_int), ("rho", ctypes.c_float), ("ld_M", ctypes.c_int)]


class RsvdArgs(ctypes.Structure):
    _fields_ = [("factor", ctypes.c_int), ("K_dense", ctypes.c_void_p), ("oversample", ctypes.c_int),
                ("power_iters", ctypes.c_int), ("seed", ctypes.c_uint64), ("counter", ctypes.c_uint64),
                ("U_out", ctypes.c_void_p), ("D_out", ctypes.c_void_p), ("ld_U", ctypes.c_int)]


class StageStat(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("calls", ctypes.c_longlong),
                ("launches", ctypes.c_longlong), ("ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


class CorrectArgs(ctypes.Structure):
    _fields_ = [("factor", ctypes.c_int), ("K_dense", ctypes.c_void_p), ("U", ctypes.c_void_p),
                ("D", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("n_crc", ctypes.c_int),
                ("ld_U", ctypes.c_int)]


class PrecondFactoredArgs(ctypes.Structure):
    _fields_ = [("layer", ctypes.c_int), ("U_G", ctypes.c_void_p), ("D_G", ctypes.c_void_p),
                ("lambda_G", ctypes.c_float), ("U_A", ctypes.c_void_p), ("D_A", ctypes.c_void_p),
                ("lambda_A", ctypes.c_float), ("G", ctypes.c_void_p), ("A", ctypes.c_void_p),
                ("n", ctypes.c_int), ("S", ctypes.c_void_p), ("flags", ctypes.c_int),
                ("ld_UG", ctypes.c_int), ("ld_UA", ctypes.c_int), ("ld_G", ctypes.c_int),
                ("ld_A", ctypes.c_int), ("ld_S", ctypes.c_int)]


class PrecondArgs(ctypes.Structure):
    _fields_ = [("layer", ctypes.c_int), ("U_G", ctypes.c_void_p), ("D_G", ctypes.c_void_p),
                ("lambda_G", ctypes.c_float), ("U_A", ctypes.c_void_p), ("D_A", ctypes.c_void_p),
                ("lambda_A", ctypes.c_float), ("J", ctypes.c_void_p), ("S", ctypes.c_void_p),
                ("flags", ctypes.c_int), ("ld_UG", ctypes.c_int), ("ld_UA", ctypes.c_int),
                ("ld_J", ctypes.c_int), ("ld_S", ctypes.c_int)]


_lib = None


def load(path: str = None) -> ctypes.CDLL:
    """Load libbkfac.so.  Raises loudly if it is missing: there is no fallback path.
    ``BKFAC_LIB`` may point at another in-tree build of the same library (tuning runs)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("BKFAC_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise RuntimeError(f"bkfac CUDA library not built: {path} is missing "
                           "(run `python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = ctypes.CDLL(path)
    vp, ci, cf, sz, u64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_float, ctypes.c_size_t, ctypes.c_uint64
    lib.bkfac_init.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(FactorDesc), ci,
                               ctypes.POINTER(LayerDesc), ci, ci]
    lib.bkfac_init.restype = ci
    lib.bkfac_workspace_bytes.argtypes = [vp]
    lib.bkfac_workspace_bytes.restype = sz
    lib.bkfac_set_workspace.argtypes = [vp, vp, sz]
    lib.bkfac_set_workspace.restype = ci
    lib.bkfac_destroy.argtypes = [vp]
    lib.bkfac_destroy.restype = ci
    lib.bkfac_brand_update.argtypes = [vp, ctypes.POINTER(BrandArgs), ci, vp]
    lib.bkfac_brand_update.restype = ci
    lib.bkfac_brand_ea_update.argtypes = [vp, ctypes.POINTER(BrandArgs), ci, ctypes.POINTER(EaArgs), ci, vp]
    lib.bkfac_brand_ea_update.restype = ci
    lib.bkfac_ea_accumulate.argtypes = [vp, ci, vp, vp, ci, cf, vp]
    lib.bkfac_ea_accumulate.restype = ci
    lib.bkfac_ea_accumulate_batch.argtypes = [vp, ctypes.POINTER(EaArgs), ci, vp]
    lib.bkfac_ea_accumulate_batch.restype = ci
    lib.bkfac_rsvd_overwrite.argtypes = [vp, ci, vp, ci, ci, u64, u64, vp, vp, vp]
    lib.bkfac_rsvd_overwrite.restype = ci
    lib.bkfac_rsvd_overwrite_batch.argtypes = [vp, ctypes.POINTER(RsvdArgs), ci, vp]
    lib.bkfac_rsvd_overwrite_batch.restype = ci
    lib.bkfac_gaussian_sketch.argtypes = [vp, ci, ci, u64, u64, vp]
    lib.bkfac_gaussian_sketch.restype = ci
    lib.bkfac_precondition.argtypes = [vp, ctypes.POINTER(PrecondArgs), ci, vp]
    lib.bkfac_precondition.restype = ci
    lib.bkfac_precondition_factored.argtypes = [vp, ctypes.POINTER(PrecondFactoredArgs), ci, vp]
    lib.bkfac_precondition_factored.restype = ci
    lib.bkfac_light_correction.argtypes = [vp, ctypes.POINTER(CorrectArgs), ci, vp]
    lib.bkfac_light_correction.restype = ci
    lib.bkfac_check.argtypes = [vp, vp, ctypes.POINTER(ci), ctypes.POINTER(ci)]
    lib.bkfac_check.restype = ci
    lib.bkfac_set_option.argtypes = [vp, ci, ci]
    lib.bkfac_set_option.restype = ci
    lib.bkfac_launch_count.argtypes = [vp]
    lib.bkfac_launch_count.restype = u64
    lib.bkfac_profile_enable.argtypes = [vp, ci]
    lib.bkfac_profile_enable.restype = ci
    lib.bkfac_profile_read.argtypes = [vp, ctypes.POINTER(StageStat), ci]
    lib.bkfac_profile_read.restype = ci
    lib.bkfac_profile_count.argtypes = [vp]
    lib.bkfac_profile_count.restype = ci
    lib.bkfac_profile_read_range.argtypes = [vp, ci, ci, ctypes.POINTER(StageStat), ci]
    lib.bkfac_profile_read_range.restype = ci
    lib.bkfac_status_string.argtypes = [ci]
    lib.bkfac_status_string.restype = ctypes.c_char_p
    lib.bkfac_build_info.argtypes = []
    lib.bkfac_build_info.restype = ctypes.c_char_p
    lib.bkfac_gemm.argtypes = [ci, ci, ci, ci, ci, cf, vp, ci, vp, ci, cf, vp, ci, vp, sz, ci, vp]
    lib.bkfac_gemm.restype = ci
    _lib = lib
    return lib


def _check(code: int, where: str) -> None:
    if code != 0:
        raise BkfacError(code, where)


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError("bkfac expects contiguous float32 CUDA tensors")
    return t.data_ptr()


def _mat(t):
    """(device pointer, leading dimension) of a 2-D float32 CUDA tensor whose rows are the
    col-major columns of the operand: unit stride along dim 1, any row stride >= the row
    length (a view t[:, :n] of a padded (b, ld) buffer passes ld; bkfac.h "Leading
    dimensions")."""
    import torch
    if t is None:
        return None, 0
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if t.dtype != torch.float32 or not t.is_cuda or t.dim() != 2:
        raise ValueError("bkfac expects 2-D float32 CUDA tensors")
    rows, cols = t.shape
    if cols > 1 and t.stride(1) != 1:
        raise ValueError("bkfac expects unit stride along the last dimension")
    ld = t.stride(0) if rows > 1 else max(t.stride(0), cols)
    if rows > 1 and ld < cols:
        raise ValueError("bkfac expects row stride >= row length")
    return t.data_ptr(), int(ld)


def _iptr(t) -> Optional[int]:
    """Device pointer of a contiguous int32 CUDA tensor (index arrays)."""
    import torch
    if not isinstance(t, torch.Tensor) or t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
        raise ValueError("bkfac expects a contiguous int32 CUDA tensor of indices")
    return t.data_ptr()


def _stream_ptr(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _brand_args(u) -> BrandArgs:
    (ui, ldu), (uo, ldo), (m, ldm) = _mat(u["U_in"]), _mat(u["U_out"]), _mat(u["M"])
    if ldu != ldo:
        raise ValueError("U_in and U_out must share one leading dimension")
    return BrandArgs(u["factor"], ui, _ptr(u["D_in"]), m, int(u["M"].shape[0]), uo,
                     _ptr(u["D_out"]), float(u["alpha"]), float(u["beta"]),
                     int(u.get("flags", 0)), ldu, ldm)


class Context:
    """Owns a bkfac_ctx and its device workspace (a torch uint8 tensor)."""

    def __init__(self, factors: Sequence[tuple], layers: Sequence[tuple] = (), device: int = 0):
        import torch
        self.lib = load()
        self.device = device
        fd = (FactorDesc * max(1, len(factors)))(*[FactorDesc(*f) for f in factors])
        # (d_G, d_A, r_G, r_A[, n_max]); n_max > 0 enables bkfac_precondition_factored
        ld = (LayerDesc * max(1, len(layers)))(*[LayerDesc(*(tuple(l) + (0,) * (5 - len(l))))
                                                 for l in layers])
        h = ctypes.c_void_p()
        _check(self.lib.bkfac_init(ctypes.byref(h), fd, len(factors), ld, len(layers), device),
               "bkfac_init")
        self.h = h
        self.factors = [tuple(f) for f in factors]
        self.layers = [tuple(l) for l in layers]
        nbytes = int(self.lib.bkfac_workspace_bytes(h))
        self.workspace = torch.empty(max(nbytes, 256), dtype=torch.uint8,
                                     device=f"cuda:{device}")
        _check(self.lib.bkfac_set_workspace(h, self.workspace.data_ptr(), self.workspace.numel()),
               "bkfac_set_workspace")

    def close(self) -> None:
        if getattr(self, "h", None) is not None and self.h.value:
            self.lib.bkfac_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- calls with the C names --------------------------------------------------------
    def bkfac_brand_update(self, updates: List[dict], stream=None) -> None:
        arr = (BrandArgs * len(updates))()
        for i, u in enumerate(updates):
            arr[i] = _brand_args(u)
        _check(self.lib.bkfac_brand_update(self.h, arr, len(updates), _stream_ptr(stream)),
               "bkfac_brand_update")

    def bkfac_brand_ea_update(self, updates: List[dict], ea_items: List[dict], stream=None) -> None:
        """bkfac_brand_ea_update: bkfac_brand_update(updates) + bkfac_ea_accumulate_batch(ea_items)
        of one step, the EA GEMM overlapped with the eigensolver inside the library."""
        arr = (BrandArgs * max(len(updates), 1))()
        for i, u in enumerate(updates):
            arr[i] = _brand_args(u)
        ea = (EaArgs * max(len(ea_items), 1))()
        for i, a in enumerate(ea_items):
            m, ldm = _mat(a["M"])
            ea[i] = EaArgs(a["factor"], _ptr(a["K"]), m, int(a["M"].shape[0]), float(a["rho"]), ldm)
        _check(self.lib.bkfac_brand_ea_update(self.h, arr, len(updates), ea, len(ea_items),
                                              _stream_ptr(stream)),
               "bkfac_brand_ea_update")

    def bkfac_ea_accumulate(self, factor: int, K, M, rho: float, stream=None) -> None:
        _check(self.lib.bkfac_ea_accumulate(self.h, factor, _ptr(K), _ptr(M), int(M.shape[0]),
                                            float(rho), _stream_ptr(stream)),
               "bkfac_ea_accumulate")

    def bkfac_ea_batch(self, items: List[dict], stream=None) -> None:
        """bkfac_ea_accumulate_batch: items of dict(factor, K, M, rho)."""
        arr = (EaArgs * len(items))()
        for i, a in enumerate(items):
            m, ldm = _mat(a["M"])
            arr[i] = EaArgs(a["factor"], _ptr(a["K"]), m, int(a["M"].shape[0]), float(a["rho"]), ldm)
        _check(self.lib.bkfac_ea_accumulate_batch(self.h, arr, len(items), _stream_ptr(stream)),
               "bkfac_ea_accumulate_batch")

    def bkfac_rsvd_overwrite(self, factor: int, K, oversample: int, power_iters: int,
                             seed: int, counter: int, U_out, D_out, stream=None) -> None:
        _check(self.lib.bkfac_rsvd_overwrite(self.h, factor, _ptr(K), oversample, power_iters,
                                             seed, counter, _ptr(U_out), _ptr(D_out),
                                             _stream_ptr(stream)),
               "bkfac_rsvd_overwrite")

    def bkfac_rsvd_batch(self, items: List[dict], stream=None) -> None:
        """bkfac_rsvd_overwrite_batch: dict(factor, K, oversample, power_iters, seed, counter,
        U_out, D_out)."""
        arr = (RsvdArgs * len(items))()
        for i, a in enumerate(items):
            uo, ldu = _mat(a["U_out"])
            arr[i] = RsvdArgs(a["factor"], _ptr(a["K"]), int(a["oversample"]), int(a["power_iters"]),
                              int(a["seed"]), int(a["counter"]), uo, _ptr(a["D_out"]), ldu)
        _check(self.lib.bkfac_rsvd_overwrite_batch(self.h, arr, len(items), _stream_ptr(stream)),
               "bkfac_rsvd_overwrite_batch")

    def bkfac_precondition(self, items: List[dict], stream=None) -> None:
        arr = (PrecondArgs * len(items))()
        for i, a in enumerate(items):
            (ug, ldg), (ua, lda) = _mat(a["U_G"]), _mat(a["U_A"])
            (j, ldj), (sp, lds) = _mat(a["J"]), _mat(a["S"])
            arr[i] = PrecondArgs(a["layer"], ug, _ptr(a["D_G"]), float(a["lambda_G"]),
                                 ua, _ptr(a["D_A"]), float(a["lambda_A"]),
                                 j, sp, int(a.get("flags", 0)), ldg, lda, ldj, lds)
        _check(self.lib.bkfac_precondition(self.h, arr, len(items), _stream_ptr(stream)),
               "bkfac_precondition")

    def bkfac_precondition_factored(self, items: List[dict], stream=None) -> None:
        """Algorithm 8: dict(layer, U_G, D_G, lambda_G, U_A, D_A, lambda_A, G, A, S, flags);
        G, A are (n, d) tensors (= col-major d x n), n = G.shape[0]."""
        arr = (PrecondFactoredArgs * len(items))()
        for i, a in enumerate(items):
            (ug, ldug), (ua, ldua) = _mat(a["U_G"]), _mat(a["U_A"])
            (g, ldg), (am, lda), (sp, lds) = _mat(a["G"]), _mat(a["A"]), _mat(a["S"])
            arr[i] = PrecondFactoredArgs(a["layer"], ug, _ptr(a["D_G"]), float(a["lambda_G"]),
                                         ua, _ptr(a["D_A"]), float(a["lambda_A"]),
                                         g, am, int(a["G"].shape[0]), sp, int(a.get("flags", 0)),
                                         ldug, ldua, ldg, lda, lds)
        _check(self.lib.bkfac_precondition_factored(self.h, arr, len(items), _stream_ptr(stream)),
               "bkfac_precondition_factored")

    def bkfac_light_correction(self, items: List[dict], stream=None) -> None:
        """Algorithm 6: dict(factor, K, U, D, col_idx (int32 device tensor of n_crc indices))."""
        arr = (CorrectArgs * len(items))()
        for i, a in enumerate(items):
            u, ldu = _mat(a["U"])
            arr[i] = CorrectArgs(a["factor"], _ptr(a["K"]), u, _ptr(a["D"]),
                                 _iptr(a["col_idx"]), int(a["col_idx"].numel()), ldu)
        _check(self.lib.bkfac_light_correction(self.h, arr, len(items), _stream_ptr(stream)),
               "bkfac_light_correction")

    def bkfac_check(self, stream=None):
        bad = ctypes.c_int(-1)
        info = ctypes.c_int(0)
        code = self.lib.bkfac_check(self.h, _stream_ptr(stream), ctypes.byref(bad),
                                    ctypes.byref(info))
        return code, bad.value, info.value

    def bkfac_set_option(self, option: int, value: int) -> None:
        _check(self.lib.bkfac_set_option(self.h, int(option), int(value)), "bkfac_set_option")

    def bkfac_launch_count(self) -> int:
        return int(self.lib.bkfac_launch_count(self.h))

    def bkfac_profile_enable(self, on: bool = True) -> None:
        _check(self.lib.bkfac_profile_enable(self.h, 1 if on else 0), "bkfac_profile_enable")

    def bkfac_profile_count(self) -> int:
        return int(self.lib.bkfac_profile_count(self.h))

    def bkfac_profile_read(self, rng=None) -> List[dict]:
        """Per-stage event times.  rng=(begin, end): only those records, kept in place
        (bkfac_profile_read_range; events captured into a CUDA graph are re-recorded by every
        replay); else all records, cleared (bkfac_profile_read)."""
        arr = (StageStat * 128)()
        if rng is None:
            n = self.lib.bkfac_profile_read(self.h, arr, 128)
        else:
            n = self.lib.bkfac_profile_read_range(self.h, int(rng[0]), int(rng[1]), arr, 128)
        if n < 0:
            raise BkfacError(6, "bkfac_profile_read")
        return [dict(name=arr[i].name.decode(), calls=arr[i].calls, launches=arr[i].launches,
                     ms=arr[i].ms, flops=arr[i].flops, bytes=arr[i].bytes) for i in range(min(n, 128))]


def bkfac_gaussian_sketch(Omega, seed: int, counter: int, stream=None) -> None:
    """Omega: tensor of shape (l, n) (col-major n x l) filled with the RSVD sketch."""
    l, n = Omega.shape
    _check(load().bkfac_gaussian_sketch(_ptr(Omega), n, l, seed, counter, _stream_ptr(stream)),
           "bkfac_gaussian_sketch")


def bkfac_gemm(transA: bool, transB: bool, alpha: float, A, B, beta: float, C, ws=None,
               path: int = BKFAC_GEMM_TCGEN05, stream=None) -> None:
    """C = alpha op(A) op(B) + beta C in BLAS col-major terms.  Tensors are PyTorch
    row-major, so a (cols, rows) tensor is a col-major rows x cols matrix:
    C has shape (N, M); A has shape (K, M) (or (M, K) if transA); B has shape (N, K)
    (or (K, N) if transB)."""
    N, M = C.shape
    K = A.shape[1] if transA else A.shape[0]
    lda, ldb, ldc = A.shape[1], B.shape[1], C.shape[1]
    wsb = 0 if ws is None else ws.numel() * ws.element_size()
    _check(load().bkfac_gemm(int(transA), int(transB), M, N, K, alpha, _ptr(A), lda, _ptr(B), ldb,
                             beta, _ptr(C), ldc, _ptr(ws), wsb, path, _stream_ptr(stream)),
           "bkfac_gemm")


def bkfac_status_string(code: int) -> str:
    return load().bkfac_status_string(code).decode()
