"""ctypes wrapper of the C oracle (oracle/morea_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` leg -- never by the product
package paper_2303_04873_b200/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "morea_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")

F_DOMAIN = 1
F_EMPTY = 2
F_COVERAGE = 4
PT = dict(h=0, g=1, ns=2, nt=3, m=4, fold_s=5, fold_t=6, sev=7, domain=8)
PT_N = 10


class Acc(ctypes.Structure):
    _fields_ = [("h_sum", ctypes.c_double), ("g_sum", ctypes.c_double),
                ("m_sum", ctypes.c_double), ("severity", ctypes.c_double),
                ("n_samples", ctypes.c_int64), ("folds", ctypes.c_int32),
                ("flags", ctypes.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def build(force=False):
    """Compile the oracle: plain -O2, no fast-math, no FP contraction, 1 thread."""
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-Wall", "-Wno-unused-function", SRC, "-o", LIB + ".tmp", "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB)
        vp = ctypes.c_void_p
        L.orc_create.restype = vp
        L.orc_create.argtypes = [ctypes.c_int] * 3 + [vp, vp, vp, ctypes.c_int, vp, vp, vp, vp,
                                                      ctypes.c_double, ctypes.c_int, vp,
                                                      ctypes.c_int, vp, vp, ctypes.c_int, vp]
        L.orc_destroy.argtypes = [vp]
        L.orc_eval_tets.argtypes = [vp, vp, ctypes.c_int, vp, vp]
        L.orc_eval.argtypes = [vp, vp, vp, vp]
        L.orc_eval_partial.argtypes = [vp, vp, vp, ctypes.c_int, vp, vp, vp, vp]
        L.orc_check_folds.argtypes = [vp, vp, vp, vp, vp]
        L.orc_owner_map.argtypes = [vp, vp, ctypes.c_int, vp]
        L.orc_distance_map.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp]
        L.orc_sample_map.argtypes = [vp, vp, ctypes.c_int, vp, vp]
        L.orc_distance_at.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp, vp]
        L.orc_sample_debug.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.orc_h.restype = ctypes.c_double
        L.orc_h.argtypes = [ctypes.c_double, ctypes.c_double, ctypes.c_int]
        L.orc_trilinear_raw.restype = ctypes.c_double
        L.orc_trilinear_raw.argtypes = [ctypes.c_int] * 3 + [vp] + [ctypes.c_double] * 3
        L.orc_signed_det.argtypes = [vp, vp, vp]
        L.orc_canon.restype = ctypes.c_int64
        L.orc_canon.argtypes = [ctypes.c_float, ctypes.c_float]
        L.orc_ref_sign.argtypes = [vp, ctypes.c_int]
        L.orc_r.restype = ctypes.c_double
        L.orc_r.argtypes = [vp]
        L.orc_set_sampler.argtypes = [vp, ctypes.c_int, ctypes.c_double]
        L.orc_sobol_point.argtypes = [ctypes.c_uint64, vp]
        L.orc_neg_log.restype = ctypes.c_double
        L.orc_neg_log.argtypes = [ctypes.c_uint32]
        L.orc_fnv1a64.restype = ctypes.c_uint64
        L.orc_fnv1a64.argtypes = [ctypes.c_char_p, ctypes.c_int64]
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_tet_seed.restype = ctypes.c_uint64
        L.orc_tet_seed.argtypes = [vp, vp]
        L.orc_sobol_debug.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp]
        L.orc_label_counts.argtypes = [vp, vp, ctypes.c_int, vp, ctypes.c_int, vp]
        L.orc_elasticity.argtypes = [vp, vp, ctypes.c_int, vp, vp]
        L.orc_dvf.argtypes = [vp, vp, ctypes.c_int, vp, vp]
        L.orc_mix.argtypes = [vp, vp, vp, vp, ctypes.c_int, vp, vp, vp, vp, vp, ctypes.c_int, vp,
                              ctypes.c_double, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, vp]
        L.orc_mix_sample.argtypes = [vp, vp, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int, vp]
        L.orc_det_ln.restype = ctypes.c_double
        L.orc_det_ln.argtypes = [ctypes.c_double]
        L.orc_gauss.argtypes = [ctypes.c_uint64, ctypes.c_int, vp]
        L.orc_repair.argtypes = [vp, vp, vp, ctypes.c_uint64, ctypes.c_int64, vp, vp]
        L.orc_repair_sigma.restype = ctypes.c_double
        L.orc_repair_sigma.argtypes = [vp, vp, ctypes.c_int, ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


class Oracle:
    """One problem instance (volumes, contours, mesh) of the oracle."""

    def __init__(self, dims, spacing, I_s, I_t, cs_off, cs_xyz, ct_off, ct_xyz, r_mm, base, tets,
                 c_delta=None, spoke_mode=0):
        L = lib()
        self._keep = []

        def arr(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a

        nx, ny, nz = dims
        self.dims = tuple(int(d) for d in dims)
        self.V = nx * ny * nz
        sp = arr(spacing, np.float64)
        Is = arr(np.asarray(I_s).reshape(-1), np.float32)
        It = arr(np.asarray(I_t).reshape(-1), np.float32)
        cso = arr(cs_off, np.int64)
        cto = arr(ct_off, np.int64)
        csx = arr(np.asarray(cs_xyz).reshape(-1, 3), np.float32)
        ctx = arr(np.asarray(ct_xyz).reshape(-1, 3), np.float32)
        b = arr(np.asarray(base).reshape(-1, 3), np.float32)
        t = arr(np.asarray(tets).reshape(-1, 4), np.int32)
        cd = arr(c_delta, np.float32) if c_delta is not None else None
        self.K = len(cso) - 1
        self.N = b.shape[0]
        self.T = t.shape[0]
        st = ctypes.c_int(0)
        self.h = L.orc_create(nx, ny, nz, _p(sp), _p(Is), _p(It), self.K, _p(cso), _p(csx), _p(cto),
                              _p(ctx), float(r_mm), self.N, _p(b), self.T, _p(t), _p(cd),
                              int(spoke_mode), ctypes.byref(st))
        self.status = st.value
        if not self.h:
            raise ValueError(f"oracle create failed: status {st.value}")
        self.r = L.orc_r(self.h)

    @classmethod
    def from_workload(cls, w, **kw):
        return cls(w.dims, w.spacing, w.I_s, w.I_t, w.cs_off, w.cs_xyz, w.ct_off, w.ct_xyz, w.r_mm,
                   w.base, w.tets, w.c_delta, **kw)

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_destroy(self.h)
            self.h = None

    @staticmethod
    def _off(o):
        return np.ascontiguousarray(np.asarray(o, dtype=np.float32).reshape(-1, 6))

    def eval(self, offsets_one):
        o = self._off(offsets_one)
        obj = np.zeros(3)
        acc = Acc()
        lib().orc_eval(self.h, _p(o), _p(obj), ctypes.byref(acc))
        return obj, acc

    def eval_tets(self, offsets_one, subset=None):
        o = self._off(offsets_one)
        sub = None if subset is None else np.ascontiguousarray(subset, dtype=np.int32)
        n = self.T if sub is None else len(sub)
        out = np.zeros((n, PT_N))
        lib().orc_eval_tets(self.h, _p(o), n, _p(sub), _p(out))
        return out

    def eval_partial(self, base_offsets_one, base_acc, changed, new_vals):
        o = self._off(base_offsets_one)
        ch = np.ascontiguousarray(changed, dtype=np.int32)
        nv = np.ascontiguousarray(np.asarray(new_vals, dtype=np.float32).reshape(-1, 6))
        obj = np.zeros(3)
        acc = Acc()
        rc = lib().orc_eval_partial(self.h, _p(o), ctypes.byref(base_acc), len(ch), _p(ch), _p(nv),
                                    _p(obj), ctypes.byref(acc))
        if rc != 0:
            raise ValueError("bad changed point id")
        return obj, acc

    def check_folds(self, offsets_one):
        o = self._off(offsets_one)
        cnt = ctypes.c_int32(0)
        sev = ctypes.c_double(0)
        flags = np.zeros(2 * self.T, dtype=np.uint8)
        lib().orc_check_folds(self.h, _p(o), ctypes.byref(cnt), ctypes.byref(sev), _p(flags))
        return cnt.value, sev.value, flags.reshape(2, self.T)

    def owner_map(self, offsets_one, side):
        o = self._off(offsets_one)
        out = np.empty(self.V, dtype=np.int32)
        lib().orc_owner_map(self.h, _p(o), int(side), _p(out))
        return out

    def distance_map(self, side, pair):
        out = np.empty(self.V, dtype=np.float32)
        lib().orc_distance_map(self.h, int(side), int(pair), _p(out))
        return out

    def sample_map(self, offsets_one, side):
        """Per-voxel h (NaN = not sampled) and fg (255 = not sampled) of one side."""
        o = self._off(offsets_one)
        h = np.empty(self.V, dtype=np.float64)
        fg = np.empty(self.V, dtype=np.uint8)
        lib().orc_sample_map(self.h, _p(o), int(side), _p(h), _p(fg))
        return h, fg

    def distance_at(self, side, pair, q):
        """D_pair^side at voxel centres q (n x 3 integer voxel indices)."""
        qq = np.ascontiguousarray(q, dtype=np.int64)
        out = np.empty(len(qq), dtype=np.float32)
        lib().orc_distance_at(self.h, int(side), int(pair), len(qq), _p(qq), _p(out))
        return out

    def sample_debug(self, offsets_one, tet, side, q):
        o = self._off(offsets_one)
        qq = np.ascontiguousarray(q, dtype=np.int64)
        out = np.zeros(8)
        sets = np.zeros(9, dtype=np.int64)
        rc = lib().orc_sample_debug(self.h, _p(o), int(tet), int(side), _p(qq), _p(out), _p(sets))
        if rc != 0:
            raise ValueError(rc)
        return dict(owned=bool(out[0]), x=out[1:4].copy(), a=out[4], b=out[5], fg=bool(out[6]),
                    h=out[7], sets=sets.reshape(3, 3))

    def ref_sign(self, t):
        return lib().orc_ref_sign(self.h, int(t))

    def label_counts(self, offsets_one, side, masks, M):
        """NEXT-4 (E1): per tet, owned voxel counts per label (T x (M+1))."""
        o = None if offsets_one is None else self._off(offsets_one)
        m = np.ascontiguousarray(masks, dtype=np.uint8).reshape(-1)
        out = np.zeros((self.T, M + 1), dtype=np.int64)
        if lib().orc_label_counts(self.h, _p(o), int(side), _p(m), int(M), _p(out)) != 0:
            raise ValueError("bad M")
        return out

    def elasticity(self, masks, factors):
        """NEXT-4 (E2): c_delta per tet from object masks (bit m = object m) and factors."""
        f = np.ascontiguousarray(factors, dtype=np.float32)
        m = np.ascontiguousarray(masks, dtype=np.uint8).reshape(-1)
        out = np.zeros(self.T, dtype=np.float32)
        if lib().orc_elasticity(self.h, _p(m), len(f), _p(f), _p(out)) != 0:
            raise ValueError("bad M")
        return out

    def dvf(self, offsets_one, side):
        """NEXT-4 (E3): displacement field (V x 3, mm) and coverage (V) of one side."""
        o = self._off(offsets_one)
        d = np.zeros((self.V, 3), dtype=np.float32)
        c = np.zeros(self.V, dtype=np.uint8)
        lib().orc_dvf(self.h, _p(o), int(side), _p(d), _p(c))
        return d, c

    def mix(self, offsets_one, acc, obj, grp_off, changed, mu, Lc, fixed, archive, steer_max, seed, gen, k):
        """NEXT-3 optimal mixing (M1-M7) of one solution over one colour class; returns
        (offsets, acc, obj, accepted flags)."""
        o = np.array(self._off(offsets_one), copy=True)
        a = Acc()
        ctypes.memmove(ctypes.byref(a), ctypes.byref(acc), ctypes.sizeof(Acc))
        ob = np.array(obj, dtype=np.float64, copy=True)
        go = np.ascontiguousarray(grp_off, dtype=np.int32)
        ch = np.ascontiguousarray(changed, dtype=np.int32)
        m = np.ascontiguousarray(mu, dtype=np.float64)
        l = np.ascontiguousarray(Lc, dtype=np.float64)
        fx = None if fixed is None else np.ascontiguousarray(fixed, dtype=np.uint8)
        ar = np.ascontiguousarray(archive, dtype=np.float64).reshape(-1, 3)
        G = len(go) - 1
        accd = np.zeros(G, dtype=np.uint8)
        lib().orc_mix(self.h, _p(o), ctypes.byref(a), _p(ob), G, _p(go), _p(ch), _p(m), _p(l), _p(fx),
                      len(ar), _p(ar), float(steer_max), ctypes.c_uint64(seed % 2 ** 64), int(gen), int(k),
                      _p(accd))
        return o, a, ob, accd

    def repair(self, offsets_one, seed, k, fixed=None):
        """NEXT-2 fold repair (P1-P8) of one solution (generator index k); fixed: None or
        N x 3 bools of axes that must not move.  Returns (offsets, moved, aborted)."""
        o = np.array(self._off(offsets_one), copy=True)
        fx = None if fixed is None else np.ascontiguousarray(fixed, dtype=np.uint8).reshape(-1, 3)
        mv, ab = ctypes.c_int32(0), ctypes.c_int32(0)
        lib().orc_repair(self.h, _p(o), _p(fx), ctypes.c_uint64(seed % 2 ** 64), int(k),
                         ctypes.byref(mv), ctypes.byref(ab))
        return o, mv.value, ab.value

    def repair_sigma(self, offsets_one, side, j):
        o = self._off(offsets_one)
        return lib().orc_repair_sigma(self.h, _p(o), int(side), int(j))

    def set_sampler(self, mode, rate=1.0):
        """0: exactly-once voxel centres (O3); 1: Sobol points per tet (NEXT-1, S1-S9)."""
        if lib().orc_set_sampler(self.h, int(mode), float(rate)) != 0:
            raise ValueError("bad sampler")

    def sobol_debug(self, offsets_one, tet, side, k):
        o = self._off(offsets_one)
        out = np.zeros(16)
        rc = lib().orc_sobol_debug(self.h, _p(o), int(tet), int(side), int(k), _p(out))
        if rc != 0:
            raise ValueError(rc)
        return dict(lam=out[0:4].copy(), p=out[4:7].copy(), tp=out[7:10].copy(), a=out[10],
                    b=out[11], fa=bool(out[12]), fb=bool(out[13]), h=out[14], N=int(out[15]))


def h(a, b, fg):
    return lib().orc_h(float(a), float(b), int(fg))


def trilinear(vol, x):
    vol = np.ascontiguousarray(vol, dtype=np.float32)
    nz, ny, nx = vol.shape
    return lib().orc_trilinear_raw(nx, ny, nz, _p(vol), float(x[0]), float(x[1]), float(x[2]))


def signed_det(Q):
    Q = np.ascontiguousarray(np.asarray(Q, dtype=np.int64).reshape(4, 3))
    hi = ctypes.c_int64(0)
    lo = ctypes.c_uint64(0)
    s = lib().orc_signed_det(_p(Q), ctypes.byref(hi), ctypes.byref(lo))
    return s, (hi.value << 64) + lo.value


def canon(b, o):
    return lib().orc_canon(float(b), float(o))


def sobol_points(n):
    """The first n points (uint32 x 4) of the unscrambled sequence, Gray-code order."""
    out = np.zeros((n, 4), dtype=np.uint32)
    for k in range(n):
        lib().orc_sobol_point(k, _p(out[k]))
    return out


def neg_log(x):
    return lib().orc_neg_log(int(x))


def det_ln(r):
    return lib().orc_det_ln(float(r))


def gauss(key, n):
    out = np.zeros(n)
    lib().orc_gauss(ctypes.c_uint64(key % 2 ** 64), int(n), _p(out))
    return out


def mix_sample(mu, Lc, seed, gen, k, g):
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    Lc = np.ascontiguousarray(Lc, dtype=np.float64)
    x = np.zeros(len(mu))
    lib().orc_mix_sample(_p(mu), _p(Lc), len(mu), ctypes.c_uint64(seed % 2 ** 64), int(gen), int(k), int(g), _p(x))
    return x


def fnv1a64(b: bytes):
    return lib().orc_fnv1a64(b, len(b))


def splitmix64(z):
    return lib().orc_splitmix64(int(z))


def tet_seed(Q12):
    Q = np.ascontiguousarray(np.asarray(Q12, dtype=np.int64).reshape(12))
    m = np.zeros(4, dtype=np.uint32)
    seed = lib().orc_tet_seed(_p(Q), _p(m))
    return seed, m
