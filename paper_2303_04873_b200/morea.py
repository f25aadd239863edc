"""Thin Python binding of libmorea.so (include/morea.h).

Argument marshalling only: every step of an evaluation runs in the sm_100a
kernels behind the C-ABI.  Arrays may be torch tensors (CUDA or CPU) or numpy
arrays; their data pointers are handed to the library, which detects host vs
device memory itself.  There is no CPU fallback: if libmorea.so is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOREA_LIB") or os.path.join(_HERE, "libmorea.so")

MOREA_OK = 0
ERRORS = {-1: "EINVAL", -2: "ESTATE", -3: "EDOMAIN", -4: "ECUDA", -5: "ENOMEM"}
F_DOMAIN = 1
F_EMPTY = 2
F_COVERAGE = 4
SPOKE_FACE_CENTROID = 0
SPOKE_TET_CENTROID = 1

ACC_DTYPE = np.dtype([("h_sum", "<f8"), ("g_sum", "<f8"), ("m_sum", "<f8"), ("severity", "<f8"),
                      ("n_samples", "<i8"), ("folds", "<i4"), ("flags", "<i4")])
assert ACC_DTYPE.itemsize == 48

EXPORTS = ["morea_create", "morea_destroy", "morea_last_error", "morea_stream", "morea_load_images",
           "morea_set_mesh", "morea_eval_full", "morea_eval_partial", "morea_partial_deps",
           "morea_check_folds", "morea_owner_map", "morea_distance_map", "morea_prof_enable",
           "morea_prof_read", "morea_kernel_launches", "morea_set_sampler", "morea_repair", "morea_label_counts", "morea_elasticity", "morea_dvf",
           "morea_mix_class", "morea_prepare_partial", "morea_partial_groups", "morea_sample_map"]
SAMPLER_VOXEL = 0
SAMPLER_SOBOL = 1


class MoreaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"morea error {code} ({ERRORS.get(code, '?')}): {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    L.morea_create.argtypes = [i32, vp, ctypes.POINTER(vp)]
    L.morea_destroy.argtypes = [vp]
    L.morea_destroy.restype = None
    L.morea_last_error.argtypes = [vp]
    L.morea_last_error.restype = ctypes.c_char_p
    L.morea_stream.argtypes = [vp]
    L.morea_stream.restype = vp
    L.morea_load_images.argtypes = [vp, i32, i32, i32, vp, vp, vp, i32, vp, vp, vp, vp, f64]
    L.morea_set_mesh.argtypes = [vp, i32, vp, i32, vp, vp, i32]
    L.morea_eval_full.argtypes = [vp, i32, vp, vp, vp, vp]
    L.morea_eval_partial.argtypes = [vp, i32, vp, vp, i32, vp, vp, vp, vp, vp, vp, vp]
    L.morea_partial_deps.argtypes = [vp, i32, vp, i32, vp]
    L.morea_partial_groups.argtypes = [vp]
    L.morea_prepare_partial.argtypes = [vp, i32, vp, vp]
    L.morea_check_folds.argtypes = [vp, i32, vp, vp, vp, vp]
    L.morea_owner_map.argtypes = [vp, vp, i32, vp]
    L.morea_sample_map.argtypes = [vp, vp, i32, vp, vp]
    L.morea_distance_map.argtypes = [vp, i32, i32, vp]
    L.morea_prof_enable.argtypes = [vp, i32]
    L.morea_set_sampler.argtypes = [vp, i32, f64]
    L.morea_repair.argtypes = [vp, i32, vp, vp, ctypes.c_uint64, i64, vp, vp]
    L.morea_label_counts.argtypes = [vp, vp, i32, vp, i32, vp]
    L.morea_elasticity.argtypes = [vp, vp, i32, vp, vp]
    L.morea_dvf.argtypes = [vp, vp, i32, vp, vp]
    L.morea_mix_class.argtypes = [vp, i32, vp, vp, vp, vp, i32, vp, vp, vp, i32, vp, vp, vp, i32, vp, f64,
                                  ctypes.c_uint64, i64, i64, vp]
    L.morea_kernel_launches.argtypes = [vp]
    L.morea_kernel_launches.restype = i64
    L.morea_prof_read.argtypes = [vp] + [ctypes.POINTER(i64), ctypes.POINTER(f64)] + \
        [ctypes.POINTER(i64)] * 4
    return L


_lib = _load()


def lib():
    return _lib


def _ptr(a):
    """Data pointer of a torch tensor / numpy array (None -> NULL).  Must be contiguous."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported array type {type(a)}")


def _np(a, dtype):
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def _is_torch(a):
    return hasattr(a, "data_ptr") and not isinstance(a, np.ndarray)


_DT = {"f4": ("float32",), "f8": ("float64",), "i8": ("int64",), "i4": ("int32",), "u1": ("uint8",)}


def _check(a, name, kind, shape):
    """Marshalling guard: dtype and shape of an array handed to the C-ABI (the library
    reads raw pointers, so a wrong dtype would be silently misread)."""
    if a is None:
        return
    if not _is_torch(a) and kind == "i8" and a.dtype == ACC_DTYPE:
        dt = "int64"  # structured accumulator records: 48 bytes = 6 x int64
        a = a.view(np.uint8)
        if a.size < 48 * (shape[0] if shape else 1):
            raise ValueError(f"{name}: {a.size} bytes, at least {48 * shape[0]} needed")
        return
    dt = str(a.dtype).replace("torch.", "")
    if dt not in _DT[kind]:
        raise TypeError(f"{name}: dtype {dt}, expected {_DT[kind][0]}")
    n = 1
    for d in shape:
        n *= d
    got = int(a.numel()) if _is_torch(a) else int(a.size)
    if got < n:
        raise ValueError(f"{name}: {got} elements, at least {n} {tuple(shape)} needed")


class Context:
    """One evaluator instance bound to one CUDA device (include/morea.h)."""

    def __init__(self, device: int = 0, stream=None):
        h = ctypes.c_void_p()
        s = None if stream is None else (stream if isinstance(stream, int) else stream.cuda_stream)
        rc = _lib.morea_create(int(device), s, ctypes.byref(h))
        if rc != MOREA_OK:
            raise MoreaError(rc, "morea_create failed (no usable CUDA device?)")
        self.h = h
        self.device = device
        self.N = self.T = self.V = self.K = 0
        self.dims = None

    def close(self):
        if getattr(self, "h", None):
            if _lib is not None:  # the module may already be torn down at interpreter exit
                _lib.morea_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _check(self, rc):
        if rc != MOREA_OK:
            raise MoreaError(rc, _lib.morea_last_error(self.h).decode())

    @property
    def stream_handle(self):
        return _lib.morea_stream(self.h)

    # ------------------------------------------------------------------ setup
    def load_images(self, dims, spacing, I_s, I_t, cs_off, cs_xyz, ct_off, ct_xyz, r_mm=0.0):
        nx, ny, nz = (int(d) for d in dims)
        sp = _np(spacing, np.float64)
        Is = I_s if _is_torch(I_s) else _np(I_s, np.float32)
        It = I_t if _is_torch(I_t) else _np(I_t, np.float32)
        cso, cto = _np(cs_off, np.int64), _np(ct_off, np.int64)
        csx = cs_xyz if _is_torch(cs_xyz) else _np(cs_xyz, np.float32)
        ctx_ = ct_xyz if _is_torch(ct_xyz) else _np(ct_xyz, np.float32)
        K = len(cso) - 1
        self._check(_lib.morea_load_images(self.h, nx, ny, nz, _ptr(sp), _ptr(Is), _ptr(It), K,
                                           _ptr(cso), _ptr(csx), _ptr(cto), _ptr(ctx_),
                                           float(r_mm)))
        self.dims = (nx, ny, nz)
        self.V = nx * ny * nz
        self.K = K

    def set_mesh(self, base, tets, c_delta=None, spoke_mode=SPOKE_FACE_CENTROID):
        b = base if _is_torch(base) else _np(base, np.float32)
        t = tets if _is_torch(tets) else _np(tets, np.int32)
        c = None if c_delta is None else (c_delta if _is_torch(c_delta) else _np(c_delta, np.float32))
        N = int(b.shape[0])
        T = int(t.shape[0])
        self._check(_lib.morea_set_mesh(self.h, N, _ptr(b), T, _ptr(t), _ptr(c), int(spoke_mode)))
        self.N, self.T = N, T

    @classmethod
    def from_workload(cls, w, device=0, stream=None):
        ctx = cls(device, stream)
        ctx.load_images(w.dims, w.spacing, w.I_s, w.I_t, w.cs_off, w.cs_xyz, w.ct_off, w.ct_xyz,
                        w.r_mm)
        ctx.set_mesh(w.base, w.tets, w.c_delta)
        return ctx

    # ------------------------------------------------------------------ evaluation
    def eval_full(self, offsets, obj=None, acc=None, tet_cache=None):
        """offsets: (P, N, 6) float32 (device or host).  Outputs are written into
        the given arrays (device or host); returns (obj, acc, tet_cache)."""
        P = int(offsets.shape[0])
        _check(offsets, "offsets", "f4", (P, self.N, 6))
        _check(obj, "obj", "f8", (P, 3))
        _check(acc, "acc", "i8", (P, 6))
        _check(tet_cache, "tet_cache", "f8", (P, self.T, 4))
        self._check(_lib.morea_eval_full(self.h, P, _ptr(offsets), _ptr(obj), _ptr(acc),
                                         _ptr(tet_cache)))
        return obj, acc, tet_cache

    def eval_partial(self, base_offsets, base_acc, grp_off, changed, new_vals, tet_cache=None,
                     obj=None, acc=None, dep_cache_out=None):
        P = int(base_offsets.shape[0])
        go = _np(grp_off, np.int32)
        ch = _np(changed, np.int32)
        G = len(go) - 1
        S = int(go[-1]) if G >= 0 else 0
        _check(base_offsets, "base_offsets", "f4", (P, self.N, 6))
        _check(base_acc, "base_acc", "i8", (P, 6))
        _check(new_vals, "new_vals", "f4", (P, S, 6))
        _check(tet_cache, "tet_cache", "f8", (P, self.T, 4))
        _check(obj, "obj", "f8", (P * G, 3))
        _check(acc, "acc", "i8", (P * G, 6))
        self._check(_lib.morea_eval_partial(self.h, P, _ptr(base_offsets), _ptr(base_acc), G,
                                            _ptr(go), _ptr(ch), _ptr(new_vals), _ptr(tet_cache),
                                            _ptr(obj), _ptr(acc), _ptr(dep_cache_out)))
        return obj, acc, dep_cache_out

    def prepare_partial(self, grp_off, changed):
        """Build (or find) the cached dependent-tet plan of a partial request ahead of time."""
        go = _np(grp_off, np.int32)
        ch = _np(changed, np.int32)
        self._check(_lib.morea_prepare_partial(self.h, len(go) - 1, _ptr(go), _ptr(ch)))

    def partial_deps(self):
        """Dependent tets (group order) and their group offsets of the last plan used."""
        n = _lib.morea_partial_deps(self.h, 0, None, 0, None)
        if n < 0:
            self._check(n)
        G = _lib.morea_partial_groups(self.h)
        if G < 0:
            self._check(G)
        tets = np.zeros(max(n, 1), np.int32)
        off = np.zeros(G + 1, np.int32)
        _lib.morea_partial_deps(self.h, n, _ptr(tets), G + 1, _ptr(off))
        return tets[:n], off

    def check_folds(self, offsets, fold_count=None, severity=None, tet_flags=None):
        P = int(offsets.shape[0])
        self._check(_lib.morea_check_folds(self.h, P, _ptr(offsets), _ptr(fold_count),
                                           _ptr(severity), _ptr(tet_flags)))
        return fold_count, severity, tet_flags

    def owner_map(self, offsets_one, side, owner=None):
        if owner is None:
            owner = np.empty(self.V, np.int32)
        o = offsets_one if _is_torch(offsets_one) else _np(offsets_one, np.float32)
        self._check(_lib.morea_owner_map(self.h, _ptr(o), int(side), _ptr(owner)))
        return owner

    def sample_map(self, offsets_one, side):
        """Test hook: per-voxel h (fp32, NaN = not sampled) and exact fg (255 = not sampled)."""
        h = np.empty(self.V, np.float32)
        fg = np.empty(self.V, np.uint8)
        o = offsets_one if _is_torch(offsets_one) else _np(offsets_one, np.float32)
        self._check(_lib.morea_sample_map(self.h, _ptr(o), int(side), _ptr(h), _ptr(fg)))
        return h, fg

    def distance_map(self, side, pair, out=None):
        if out is None:
            out = np.empty(self.V, np.float32)
        self._check(_lib.morea_distance_map(self.h, int(side), int(pair), _ptr(out)))
        return out

    def repair(self, offsets, seed, fixed=None, sol_base=0, moved=None, aborted=None):
        """Fold repair (§4.3.1) of `offsets` (P x N x 6, torch CUDA or numpy,
        updated in place); fixed: None or N x 3 axes that must not move."""
        P = int(offsets.shape[0])
        fx = None if fixed is None else (fixed if _is_torch(fixed) else _np(fixed, np.uint8))
        if not _is_torch(offsets):
            assert offsets.dtype == np.float32 and offsets.flags["C_CONTIGUOUS"]
        self._check(_lib.morea_repair(self.h, P, _ptr(offsets), _ptr(fx), ctypes.c_uint64(int(seed) % 2 ** 64),
                                      int(sol_base), _ptr(moved), _ptr(aborted)))
        return offsets

    def label_counts(self, offsets_one, side, masks, M, counts=None):
        """Owned voxel counts per tet and object label (T x (M+1) int64)."""
        if counts is None:
            counts = np.zeros((self.T, M + 1), np.int64)
        o = None if offsets_one is None else (offsets_one if _is_torch(offsets_one) else _np(offsets_one, np.float32))
        m = masks if _is_torch(masks) else _np(masks, np.uint8)
        self._check(_lib.morea_label_counts(self.h, _ptr(o), int(side), _ptr(m), int(M), _ptr(counts)))
        return counts

    def elasticity(self, masks, factors):
        """c_delta per tet from object masks (bit m = object m) and their factors."""
        f = _np(factors, np.float32)
        m = masks if _is_torch(masks) else _np(masks, np.uint8)
        out = np.zeros(self.T, np.float32)
        self._check(_lib.morea_elasticity(self.h, _ptr(m), len(f), _ptr(f), _ptr(out)))
        return out

    def dvf(self, offsets_one, side, dvf=None, coverage=None):
        """T(q) - q (mm) at the voxel centres owned on `side` (V x 3) and coverage (V)."""
        if dvf is None:
            dvf = np.zeros((self.V, 3), np.float32)
        if coverage is None:
            coverage = np.zeros(self.V, np.uint8)
        o = offsets_one if _is_torch(offsets_one) else _np(offsets_one, np.float32)
        self._check(_lib.morea_dvf(self.h, _ptr(o), int(side), _ptr(dvf), _ptr(coverage)))
        return dvf, coverage

    def mix_class(self, offsets, acc, obj, tet_cache, grp_off, changed, cluster, mu, L, fixed=None,
                  archive=None, steer_max=0.0, seed=0, gen=0, sol_base=0, accepted=None):
        """Optimal mixing of one FOS colour class (§3); the population state
        (offsets, acc, obj, tet_cache) is updated in place."""
        P = int(offsets.shape[0])
        go = _np(grp_off, np.int32)
        ch = _np(changed, np.int32)
        cl = cluster if _is_torch(cluster) else _np(cluster, np.int32)
        mu_ = mu if _is_torch(mu) else _np(mu, np.float64)
        L_ = L if _is_torch(L) else _np(L, np.float64)
        fx = None if fixed is None else (fixed if _is_torch(fixed) else _np(fixed, np.uint8))
        ar = np.zeros((0, 3)) if archive is None else archive
        ar = ar if _is_torch(ar) else _np(ar, np.float64)
        n_clusters = max(1, int(mu_.numel() if _is_torch(mu_) else mu_.size) // max(1, 6 * len(ch)))
        self._check(_lib.morea_mix_class(self.h, P, _ptr(offsets), _ptr(acc), _ptr(obj), _ptr(tet_cache),
                                         len(go) - 1, _ptr(go), _ptr(ch), _ptr(cl), n_clusters, _ptr(mu_),
                                         _ptr(L_), _ptr(fx), int(ar.shape[0]), _ptr(ar), float(steer_max),
                                         ctypes.c_uint64(int(seed) % 2 ** 64), int(gen), int(sol_base),
                                         _ptr(accepted)))

    def set_sampler(self, mode, rate=1.0):
        """SAMPLER_VOXEL (exactly-once voxel centres) or SAMPLER_SOBOL (App. A.2
        Sobol points per tet, `rate` samples per voxel of tet volume)."""
        self._check(_lib.morea_set_sampler(self.h, int(mode), float(rate)))

    # ------------------------------------------------------------------ profiling
    def kernel_launches(self):
        return int(_lib.morea_kernel_launches(self.h))

    def prof_enable(self, on=True):
        self._check(_lib.morea_prof_enable(self.h, 1 if on else 0))

    def prof_read(self):
        la, sa, ba, it, stp = (ctypes.c_int64() for _ in range(5))
        ms = ctypes.c_double()
        self._check(_lib.morea_prof_read(self.h, ctypes.byref(la), ctypes.byref(ms),
                                         ctypes.byref(sa), ctypes.byref(ba), ctypes.byref(it),
                                         ctypes.byref(stp)))
        return dict(launches=la.value, ms=ms.value, samples=sa.value, band_entries=ba.value,
                    items=it.value, skipped=stp.value)


# ---------------------------------------------------------------------------- helpers
def acc_to_numpy(acc):
    """Decode an accumulator buffer (torch (P,6) int64 / uint8 bytes / numpy) to ACC_DTYPE."""
    if _is_torch(acc):
        acc = acc.detach().cpu().contiguous().numpy()
    return np.ascontiguousarray(acc).view(np.uint8).reshape(-1).view(ACC_DTYPE)


def empty_outputs(P, T=None, G=1, device="cuda", cache=False, torch=None):
    """Device output buffers (torch) for P solutions x G groups."""
    if torch is None:
        import torch
    obj = torch.empty((P * G, 3), dtype=torch.float64, device=device)
    acc = torch.empty((P * G, 6), dtype=torch.int64, device=device)
    tc = torch.empty((P, T, 4), dtype=torch.float64, device=device) if cache else None
    return obj, acc, tc
