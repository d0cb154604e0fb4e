"""ctypes access to the parity checkers (TEST INFRASTRUCTURE ONLY).

  oracle/liboracle.so    CPU restatement of the reference evaluation path (oracle/dp_oracle.cpp)
  oracle/_ref/libdpref.so  the unmodified reference library + C shim (oracle/ref_shim.cpp);
                           present only where it was built from /root/reference
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

import paper_2201_01446_b200 as dp
from paper_2201_01446_b200 import _MDConfig, _MDResult, _Thermo, _dp, _ip, _u8

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libdpref.so"

_or = None
_ref = None


def build_oracle() -> None:
    src = ROOT / "oracle" / "dp_oracle.cpp"
    if not ORACLE_SO.exists() or ORACLE_SO.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), str(ORACLE_SO)], check=True)


def oracle():
    global _or
    if _or is None:
        build_oracle()
        L = C.CDLL(str(ORACLE_SO))
        D, I64, I32P, U8P = C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_uint8)
        L.or_last_error.restype = C.c_char_p
        L.or_neighbor_list.argtypes = [I64, D, D, U8P, C.c_double, C.c_int, C.POINTER(I64)]
        L.or_neighbor_list_get.argtypes = [C.POINTER(I64), I32P, I32P]
        L.or_compute.argtypes = [C.POINTER(dp._ModelDesc), C.POINTER(dp._TableDesc), I64, D, I32P, D,
                                 U8P, C.c_double, D, D, D, D, C.POINTER(C.c_uint64)]
        L.or_run_md.argtypes = [C.POINTER(dp._ModelDesc), C.POINTER(dp._TableDesc), I64, D, D, I32P,
                                D, U8P, C.POINTER(_MDConfig), C.POINTER(_Thermo), I64,
                                C.POINTER(I64), C.POINTER(_MDResult)]
        _or = L
    return _or


def have_ref() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(str(REF_SO))
        D, I64, I32P, U8P, U64 = (C.POINTER(C.c_double), C.c_int64, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_uint8), C.c_uint64)
        P = C.POINTER(dp._Preset)
        L.ref_last_error.restype = C.c_char_p
        L.ref_gen_model.argtypes = [C.c_char_p, U64, D]
        L.ref_gen_test_model.argtypes = [P, U64, C.c_double, D]
        L.ref_build_tables.argtypes = [P, D, C.c_double, C.POINTER(U64), D]
        L.ref_gen_config.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_double, U64, D, I32P, D]
        L.ref_random_config.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double, U64, D, I32P]
        L.ref_init_velocities.argtypes = [P, I64, D, I32P, D, C.c_double, U64, D]
        L.ref_neighbor_list.argtypes = [I64, D, I32P, D, U8P, C.c_double, C.c_int, C.POINTER(I64)]
        L.ref_neighbor_list_get.argtypes = [C.POINTER(I64), I32P, I32P]
        L.ref_compute_tabulated.argtypes = [P, D, U64, C.c_double, D, I64, D, I32P, D, U8P,
                                            C.c_double, C.c_int, C.c_int, D, D, D, D,
                                            C.POINTER(U64), D]
        L.ref_compute_exact.argtypes = [P, D, I64, D, I32P, D, U8P, D, D, D, D]
        L.ref_run_md.argtypes = [P, D, U64, C.c_double, D, I64, D, D, I32P, D, U8P,
                                 C.POINTER(_MDConfig), C.c_int, C.POINTER(_Thermo), I64,
                                 C.POINTER(I64), C.POINTER(_MDResult)]
        L.ref_partition_domain.argtypes = [I64, D, D, U8P, C.c_int, C.c_double, C.POINTER(C.c_int),
                                           I32P, U8P]
        _ref = L
    return _ref


def _chk(rc, lib, fn="or_last_error"):
    if rc:
        msg = getattr(lib, fn)().decode()
        if rc == 2:
            raise dp.InputError(msg)
        if rc == 1:
            raise dp.NumericalError(msg)
        raise RuntimeError(msg)


# ---------------------------------------------------------------- oracle entry points
def or_neighbor_list(cfg: dp.AtomicConfig, cutoff: float, brute: bool = False) -> dp.NeighborList:
    L = oracle()
    tot = C.c_int64()
    _chk(L.or_neighbor_list(cfg.n_atoms, _dp(cfg.pos), _dp(cfg.h), _u8(cfg.periodic), cutoff,
                            int(brute), C.byref(tot)), L)
    off = np.empty(cfg.n_atoms + 1, dtype=np.int64)
    j = np.empty(max(tot.value, 1), dtype=np.int32)
    s = np.empty((max(tot.value, 1), 3), dtype=np.int32)
    L.or_neighbor_list_get(off.ctypes.data_as(C.POINTER(C.c_int64)), _ip(j), _ip(s))
    return dp.NeighborList(cutoff, off, j[: tot.value], s[: tot.value])


def or_compute(cfg: dp.AtomicConfig, model: dp.DPModel, tabs: dp.Tables, list_cutoff: float = 0.0):
    L = oracle()
    md, k1 = model.desc()
    td, k2 = tabs.desc()
    n = cfg.n_atoms
    e = C.c_double()
    f = np.empty((n, 3))
    v = np.empty(9)
    ae = np.empty(n)
    cnt = (C.c_uint64 * 3)()
    _chk(L.or_compute(C.byref(md), C.byref(td), n, _dp(cfg.pos), _ip(cfg.type), _dp(cfg.h),
                      _u8(cfg.periodic), list_cutoff, C.byref(e), _dp(f), _dp(v), _dp(ae), cnt), L)
    return dp.EvalResult(e.value, ae, f, v), dp.FusedCounters(cnt[0], cnt[1], cnt[2])


def or_run_md(cfg: dp.AtomicConfig, vel: np.ndarray, model: dp.DPModel, tabs: dp.Tables,
              mc: dp.MDConfig) -> dp.MDResult:
    L = oracle()
    md, k1 = model.desc()
    td, k2 = tabs.desc()
    c = _MDConfig(mc.n_steps, mc.dt, mc.buffer, mc.rebuild_every, mc.thermo_every)
    cap = mc.n_steps // mc.thermo_every + 2
    th = (_Thermo * cap)()
    nth = C.c_int64()
    res = _MDResult()
    _chk(L.or_run_md(C.byref(md), C.byref(td), cfg.n_atoms, _dp(cfg.pos), _dp(vel), _ip(cfg.type),
                     _dp(cfg.h), _u8(cfg.periodic), C.byref(c), th, cap, C.byref(nth),
                     C.byref(res)), L)
    return dp._md_result(th, nth.value, res)


# ---------------------------------------------------------------- reference entry points
def ref_gen_model(name: str, seed: int) -> dp.DPModel:
    p = dp.get_preset(name)
    blob = np.empty(dp._blob_size(p))
    _chk(ref().ref_gen_model(name.encode(), seed, _dp(blob)), ref(), "ref_last_error")
    return dp.DPModel(p, blob)


def ref_make_test_model(model_like: dp.DPModel, seed: int, fit_scale: float = 0.2) -> np.ndarray:
    blob = np.empty_like(model_like.blob)
    _chk(ref().ref_gen_test_model(C.byref(model_like.shape._c()), seed, fit_scale, _dp(blob)), ref(),
         "ref_last_error")
    return blob


def ref_build_tables(model: dp.DPModel, h: float) -> dp.Tables:
    n = C.c_uint64()
    shp = model.shape._c()
    _chk(ref().ref_build_tables(C.byref(shp), _dp(model.blob), h, C.byref(n), None), ref(),
         "ref_last_error")
    m = 4 * model.shape.d1
    stride = ((m + 15) // 16) * 96
    co = np.empty((model.shape.n_types, n.value * stride))
    _chk(ref().ref_build_tables(C.byref(shp), _dp(model.blob), h, C.byref(n), _dp(co)), ref(),
         "ref_last_error")
    return dp.Tables(0.0, h, n.value, m, 16, co)


def ref_gen_config(name, nx, ny, nz, jitter, seed) -> dp.AtomicConfig:
    n = 4 * nx * ny * nz
    pos = np.empty((n, 3))
    ty = np.empty(n, dtype=np.int32)
    h = np.empty(9)
    _chk(ref().ref_gen_config(name.encode(), nx, ny, nz, jitter, seed, _dp(pos), _ip(ty), _dp(h)),
         ref(), "ref_last_error")
    return dp.AtomicConfig(pos, ty, h)


def ref_random_config(n, n_types, box, min_sep, seed) -> dp.AtomicConfig:
    pos = np.empty((n, 3))
    ty = np.empty(n, dtype=np.int32)
    _chk(ref().ref_random_config(n, n_types, box, min_sep, seed, _dp(pos), _ip(ty)), ref(),
         "ref_last_error")
    return dp.AtomicConfig(pos, ty, np.array([box, 0, 0, 0, box, 0, 0, 0, box], dtype=np.float64))


def ref_neighbor_list(cfg: dp.AtomicConfig, cutoff: float, brute: bool = False) -> dp.NeighborList:
    L = ref()
    tot = C.c_int64()
    _chk(L.ref_neighbor_list(cfg.n_atoms, _dp(cfg.pos), _ip(cfg.type), _dp(cfg.h),
                             _u8(cfg.periodic), cutoff, int(brute), C.byref(tot)), L, "ref_last_error")
    off = np.empty(cfg.n_atoms + 1, dtype=np.int64)
    j = np.empty(max(tot.value, 1), dtype=np.int32)
    s = np.empty((max(tot.value, 1), 3), dtype=np.int32)
    L.ref_neighbor_list_get(off.ctypes.data_as(C.POINTER(C.c_int64)), _ip(j), _ip(s))
    return dp.NeighborList(cutoff, off, j[: tot.value], s[: tot.value])


def ref_compute(cfg, model, tabs, list_cutoff=0.0, n_workers=1, repeats=1):
    L = ref()
    n = cfg.n_atoms
    e = C.c_double()
    f = np.empty((n, 3))
    v = np.empty(9)
    ae = np.empty(n)
    cnt = (C.c_uint64 * 3)()
    secs = np.zeros(2)
    shp = model.shape._c()
    _chk(L.ref_compute_tabulated(C.byref(shp), _dp(model.blob), tabs.n, tabs.h, _dp(tabs.coeffs), n,
                                 _dp(cfg.pos), _ip(cfg.type), _dp(cfg.h), _u8(cfg.periodic),
                                 list_cutoff, n_workers, repeats, C.byref(e), _dp(f), _dp(v),
                                 _dp(ae), cnt, _dp(secs)), L, "ref_last_error")
    return dp.EvalResult(e.value, ae, f, v), dp.FusedCounters(cnt[0], cnt[1], cnt[2]), secs


def ref_run_md(cfg, vel, model, tabs, mc: dp.MDConfig, n_workers=1) -> dp.MDResult:
    L = ref()
    c = _MDConfig(mc.n_steps, mc.dt, mc.buffer, mc.rebuild_every, mc.thermo_every)
    cap = mc.n_steps // mc.thermo_every + 2
    th = (_Thermo * cap)()
    nth = C.c_int64()
    res = _MDResult()
    shp = model.shape._c()
    _chk(L.ref_run_md(C.byref(shp), _dp(model.blob), tabs.n, tabs.h, _dp(tabs.coeffs), cfg.n_atoms,
                      _dp(cfg.pos), _dp(vel), _ip(cfg.type), _dp(cfg.h), _u8(cfg.periodic),
                      C.byref(c), n_workers, th, cap, C.byref(nth), C.byref(res)), L,
         "ref_last_error")
    return dp._md_result(th, nth.value, res)


def lists_equal(a: dp.NeighborList, b: dp.NeighborList) -> bool:
    return (np.array_equal(a.offsets, b.offsets) and np.array_equal(a.j, b.j)
            and np.array_equal(a.shift, b.shift))


def normwise(a: np.ndarray, b: np.ndarray) -> float:
    """max|a-b| / max|b| (SURVEY.md §8d parity metric)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale


def ref_compute_exact(cfg: dp.AtomicConfig, model: dp.DPModel) -> dp.EvalResult:
    """compute_energy_forces_virial (exact.cpp:155-173) of the compiled reference."""
    n = cfg.n_atoms
    e = C.c_double()
    f = np.empty((n, 3))
    v = np.empty(9)
    ae = np.empty(n)
    _chk(ref().ref_compute_exact(C.byref(model.shape._c()), _dp(model.blob), n, _dp(cfg.pos), _ip(cfg.type),
                                 _dp(cfg.h), _u8(cfg.periodic), C.byref(e), _dp(f), _dp(v), _dp(ae)),
         ref(), "ref_last_error")
    return dp.EvalResult(e.value, ae, f, v)


def ref_rmse_sweep(model: dp.DPModel, h_list, configs):
    """rmse_sweep + loglog_slope (rmse.cpp:63-116) of the compiled reference."""
    L = ref()
    D, I64 = C.POINTER(C.c_double), C.c_int64
    L.ref_rmse_sweep.argtypes = [C.POINTER(dp._Preset), D, C.c_int, C.POINTER(I64), D, C.POINTER(C.c_int32), D,
                                 C.POINTER(C.c_uint8), C.c_int, D, D, D, D]
    na = np.array([c.n_atoms for c in configs], dtype=np.int64)
    pos = np.ascontiguousarray(np.concatenate([c.pos.reshape(-1) for c in configs]))
    typ = np.ascontiguousarray(np.concatenate([c.type for c in configs]).astype(np.int32))
    box = np.ascontiguousarray(np.concatenate([c.h.reshape(-1) for c in configs]))
    pbc = np.ascontiguousarray(np.concatenate([c.periodic for c in configs]).astype(np.uint8))
    hl = np.ascontiguousarray(h_list, dtype=np.float64)
    re, rf, sl = np.empty(len(hl)), np.empty(len(hl)), np.empty(1)
    _chk(L.ref_rmse_sweep(C.byref(model.shape._c()), _dp(model.blob), len(configs),
                          na.ctypes.data_as(C.POINTER(I64)), _dp(pos), _ip(typ), _dp(box), _u8(pbc), len(hl),
                          _dp(hl), _dp(re), _dp(rf), _dp(sl)), L, "ref_last_error")
    return re, rf, float(sl[0])


def ref_write_model(path: str, model: dp.DPModel, preset: str, seed: int) -> None:
    L = ref()
    L.ref_write_model.argtypes = [C.c_char_p, C.POINTER(dp._Preset), C.POINTER(C.c_double), C.c_char_p,
                                  C.c_uint64]
    _chk(L.ref_write_model(path.encode(), C.byref(model.shape._c()), _dp(model.blob), preset.encode(), seed),
         L, "ref_last_error")


def ref_read_model(path: str, model_like: dp.DPModel):
    L = ref()
    L.ref_read_model.argtypes = [C.c_char_p, C.POINTER(dp._Preset), C.POINTER(C.c_double),
                                 C.POINTER(C.c_uint64)]
    blob = np.empty_like(model_like.blob)
    seed = C.c_uint64()
    _chk(L.ref_read_model(path.encode(), C.byref(model_like.shape._c()), _dp(blob), C.byref(seed)), L,
         "ref_last_error")
    return blob, seed.value


def ref_init_velocities(cfg: dp.AtomicConfig, model: dp.DPModel, t_init: float, seed: int) -> np.ndarray:
    """init_velocities (md.cpp:14-55) of the unmodified reference."""
    v = np.empty((cfg.n_atoms, 3))
    _chk(ref().ref_init_velocities(C.byref(model.shape._c()), cfg.n_atoms, _dp(cfg.pos), _ip(cfg.type),
                                   _dp(cfg.h), t_init, seed, _dp(v)), ref(), "ref_last_error")
    return v
