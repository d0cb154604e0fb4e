"""B200-native Deep Potential force evaluation (arXiv 2201.01446 hot path).

Host-side mirror of the reference C++ API (/root/reference/proj/include/dpmd/*.hpp) over the
C-ABI library lib/libdpb200.so (include/dp_b200.h). Names, argument meaning and error classes
follow the reference so its tests read the same here:

    reference (dpmd::)                          here
    gen_model / get_preset  model_io.hpp:39-47  gen_model / get_preset
    gen_config              model_io.hpp:44-47  gen_config
    build_tables            table.hpp:46-50     build_tables
    build_neighbor_list     neighbor.hpp:31-36  build_neighbor_list            (GPU)
    compute_energy_forces_virial_tabulated
                            fused.hpp:70-73     compute_energy_forces_virial_tabulated (GPU)
    run_md / MDConfig       md.hpp:14-60        run_md / MDConfig              (GPU)
    init_velocities         md.hpp:41-44        init_velocities
    InputError / NumericalError error.hpp:9-17  InputError / NumericalError

The compute path has no CPU fallback: if the CUDA library cannot be loaded or no GPU is
present, the GPU entry points raise instead of computing anything on the host.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "InputError", "NumericalError", "DPRuntimeError", "Preset", "get_preset", "preset_names",
    "DPModel", "gen_model", "make_test_model", "Tables", "build_tables", "read_tables",
    "write_tables", "AtomicConfig", "gen_config", "make_random_config", "init_velocities",
    "mix_seed", "EvalResult", "FusedCounters", "NeighborList", "MDConfig", "ThermoRecord",
    "MDResult", "DeepPot", "build_neighbor_list", "compute_energy_forces_virial_tabulated",
    "run_md", "library_path", "tanh_table", "partition_domain",
]

_PKG = Path(__file__).resolve().parent
_LIBPATH = _PKG / "lib" / "libdpb200.so"


class InputError(ValueError):
    """Bad user input (reference dpmd::InputError, error.hpp:9-12)."""


class NumericalError(RuntimeError):
    """Violated numerical contract (reference dpmd::NumericalError, error.hpp:15-17)."""


class DPRuntimeError(RuntimeError):
    """CUDA / runtime failure inside the library."""


# ---------------------------------------------------------------- ctypes mirror of dp_b200.h
class _Fitting(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("widths", C.POINTER(C.c_int)),
                ("w", C.POINTER(C.POINTER(C.c_double))), ("b", C.POINTER(C.POINTER(C.c_double))),
                ("w_out", C.POINTER(C.c_double)), ("b_out", C.c_double)]


class _ModelDesc(C.Structure):
    _fields_ = [("n_types", C.c_int), ("r_cut", C.c_double), ("r_smooth", C.c_double),
                ("d1", C.c_int), ("m_lt", C.c_int), ("masses", C.POINTER(C.c_double)),
                ("max_nbr", C.POINTER(C.c_int)), ("fitting", C.POINTER(_Fitting))]


class _TableDesc(C.Structure):
    _fields_ = [("n_tables", C.c_int), ("x0", C.c_double), ("h", C.c_double),
                ("n", C.c_uint64), ("m", C.c_int), ("block", C.c_int),
                ("coeffs", C.POINTER(C.POINTER(C.c_double)))]


class _EmbDesc(C.Structure):
    _fields_ = [("d1", C.c_int)] + [(k, C.POINTER(C.c_double)) for k in ("w0", "b0", "w1", "b1", "w2", "b2")]


class _Counters(C.Structure):
    _fields_ = [("rows_forward", C.c_uint64), ("rows_backward", C.c_uint64),
                ("extrapolations", C.c_uint64)]


class _MDConfig(C.Structure):
    _fields_ = [("n_steps", C.c_int64), ("dt", C.c_double), ("buffer", C.c_double),
                ("rebuild_every", C.c_int), ("thermo_every", C.c_int)]


class _Thermo(C.Structure):
    _fields_ = [("step", C.c_int64), ("ke", C.c_double), ("pe", C.c_double),
                ("temperature", C.c_double), ("pressure", C.c_double)]


class _MDResult(C.Structure):
    _fields_ = [("force_evals", C.c_uint64), ("staleness_checks", C.c_uint64),
                ("max_drift_seen", C.c_double), ("counters", _Counters),
                ("final_ke", C.c_double), ("final_pe", C.c_double), ("final_total", C.c_double)]


class _Preset(C.Structure):
    _fields_ = [("n_types", C.c_int), ("r_cut", C.c_double), ("r_smooth", C.c_double),
                ("d1", C.c_int), ("m_lt", C.c_int), ("fit_width", C.c_int),
                ("fit_hidden", C.c_int), ("masses", C.c_double * 8), ("max_nbr", C.c_int * 8),
                ("lattice_a", C.c_double), ("site_pattern", C.c_int * 8), ("n_sites", C.c_int)]


_lib_handle = None


def library_path() -> Path:
    return _LIBPATH


def _lib():
    """Load lib/libdpb200.so (built by __graft_entry__.build / paper_2201_01446_b200.build)."""
    global _lib_handle
    if _lib_handle is not None:
        return _lib_handle
    if not _LIBPATH.exists():
        raise DPRuntimeError(f"{_LIBPATH} is missing: run `python -c 'import __graft_entry__ as g; "
                             "g.build()'` (no CPU fallback exists)")
    L = C.CDLL(str(_LIBPATH))
    P, D, I, I64, U64 = C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_int64, C.c_uint64
    I32P, U8P = C.POINTER(C.c_int32), C.POINTER(C.c_uint8)
    sig = {
        "dp_version": ([], C.c_char_p),
        "dp_create": ([C.POINTER(_ModelDesc), C.POINTER(_TableDesc), I, I, C.POINTER(P)], I),
        "dp_destroy": ([P], I),
        "dp_last_error": ([P], C.c_char_p),
        "dp_set_skin": ([P, C.c_double], I),
        "dp_compute": ([P, I64, D, I32P, D, U8P, D, D, D, D], I),
        "dp_compute_list": ([P, I64, D, I32P, D, U8P, C.POINTER(C.c_int64), I32P, I32P, D, D, D, D], I),
        "dp_counters_get": ([P, C.POINTER(_Counters)], I),
        "dp_neighbor_list_build": ([P, I64, D, I32P, D, U8P, C.c_double, C.POINTER(I64)], I),
        "dp_neighbor_list_get": ([P, C.POINTER(I64), I32P, I32P], I),
        "dp_md_run": ([P, I64, D, D, I32P, D, U8P, C.POINTER(_MDConfig), C.POINTER(_Thermo),
                       I64, C.POINTER(I64), C.POINTER(_MDResult)], I),
        "dp_md_begin": ([P, I64, D, D, I32P, D, U8P, C.POINTER(_MDConfig)], I),
        "dp_md_step": ([P, I64], I),
        "dp_md_end": ([P, D, D, C.POINTER(_Thermo), I64, C.POINTER(I64), C.POINTER(_MDResult)], I),
        "dp_stream": ([P], P),
        "dp_launch_count": ([P], U64),
        "dp_set_timing": ([P, I], I),
        "dp_nccl_unique_id": ([C.c_void_p, I], I),
        "dp_partition_domain": ([I64, D, D, U8P, I, C.c_double, I32P, U8P], I),
        "dp_dist_plan": ([I64, D, D, U8P, I, I, C.c_double, C.POINTER(I64), C.POINTER(I64), U8P,
                          C.POINTER(I64), C.POINTER(I64), C.POINTER(I64), C.POINTER(I64)], I),
        "dp_dist_init": ([P, I, I, C.c_char_p], I),
        "dp_phase_times": ([P, D, C.POINTER(U64)], I),
        "dp_preset_get": ([C.c_char_p, C.POINTER(_Preset)], I),
        "dp_model_blob_size": ([C.POINTER(_Preset)], I64),
        "dp_gen_model": ([C.c_char_p, U64, D], I),
        "dp_gen_test_model": ([C.POINTER(_Preset), U64, C.c_double, D], I),
        "dp_build_tables": ([C.POINTER(_Preset), D, C.c_double, C.POINTER(U64), D, D], I),
        "dp_gen_config": ([C.c_char_p, I, I, I, C.c_double, U64, D, I32P, D], I),
        "dp_gen_random_config": ([I, I, C.c_double, C.c_double, U64, D, I32P], I),
        "dp_init_velocities": ([I64, I32P, D, C.c_double, U64, D], I),
        "dp_mix_seed": ([U64, U64], U64),
        "dp_write_tables": ([C.c_char_p, C.POINTER(_TableDesc)], I),
        "dp_read_tables_header": ([C.c_char_p, C.POINTER(I), C.POINTER(I), C.POINTER(I),
                                   C.POINTER(U64), D, D], I),
        "dp_read_tables": ([C.c_char_p, D], I),
        "dp_tanh_table": ([D], I),
        "dp_set_embedding": ([P, C.POINTER(_EmbDesc)], I),
        "dp_set_pipeline": ([P, I], I),
        "dp_set_chunk_size": ([P, I64], I),
        "dp_write_model_json": ([C.c_char_p, C.POINTER(_Preset), D, C.c_char_p, C.c_char_p, U64], I),
        "dp_read_model_json": ([C.c_char_p, C.POINTER(_Preset), D, I64, C.c_char_p, I, C.c_char_p, I,
                                C.POINTER(U64)], I),
        "dp_compute_exact": ([P, I64, D, I32P, D, U8P, D, D, D, D], I),
        "dp_build_tables_gpu": ([P, C.c_double, C.POINTER(U64), D, D, I], I),
        "dp_rmse_sweep": ([P, I, C.POINTER(I64), D, I32P, D, U8P, I, D, D, D], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib_handle = L
    return L


def _check(rc: int, handle=None) -> None:
    if rc == 0:
        return
    msg = _lib().dp_last_error(handle)
    msg = msg.decode() if msg else ""
    if rc == 2:
        raise InputError(msg)
    if rc == 1:
        raise NumericalError(msg)
    raise DPRuntimeError(msg or f"dp_b200 error {rc}")


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _u8(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def mix_seed(seed: int, k: int) -> int:
    """splitmix64 stream seed (rng.hpp:44-49)."""
    return int(_lib().dp_mix_seed(seed, k))


# ---------------------------------------------------------------- model / presets
@dataclass
class Preset:
    """Shape of a model family (model_io.hpp:14-31)."""
    name: str
    n_types: int
    masses: List[float]
    max_nbr: List[int]
    r_cut: float
    r_smooth: float
    d1: int
    m_lt: int
    fit_width: int
    fit_hidden: int
    lattice_a: float = 0.0
    site_pattern: List[int] = field(default_factory=lambda: [0])

    def _c(self) -> _Preset:
        p = _Preset()
        p.n_types, p.r_cut, p.r_smooth = self.n_types, self.r_cut, self.r_smooth
        p.d1, p.m_lt, p.fit_width, p.fit_hidden = self.d1, self.m_lt, self.fit_width, self.fit_hidden
        for t in range(self.n_types):
            p.masses[t] = self.masses[t]
            p.max_nbr[t] = self.max_nbr[t]
        p.lattice_a = self.lattice_a
        for k, s in enumerate(self.site_pattern[:8]):
            p.site_pattern[k] = s
        p.n_sites = len(self.site_pattern)
        return p


def preset_names() -> List[str]:
    return ["copper-like", "water-like"]


def get_preset(name: str) -> Preset:
    p = _Preset()
    _check(_lib().dp_preset_get(name.encode(), C.byref(p)))
    return Preset(name, p.n_types, list(p.masses[: p.n_types]), list(p.max_nbr[: p.n_types]),
                  p.r_cut, p.r_smooth, p.d1, p.m_lt, p.fit_width, p.fit_hidden, p.lattice_a,
                  list(p.site_pattern[: p.n_sites]))


class DPModel:
    """DPModel (model.hpp:38-58) backed by one flat float64 blob (dp_b200.h layout)."""

    def __init__(self, shape: Preset, blob: np.ndarray):
        self.shape = shape
        self.blob = np.ascontiguousarray(blob, dtype=np.float64)
        s = shape
        d1 = s.d1
        at = 0
        self.embedding = []
        for _ in range(s.n_types):
            e = {}
            for key, n in (("w0", d1), ("b0", d1), ("w1", 2 * d1 * d1), ("b1", 2 * d1),
                           ("w2", 8 * d1 * d1), ("b2", 4 * d1)):
                e[key] = self.blob[at: at + n]
                at += n
            self.embedding.append(e)
        self.fitting = []
        din = s.m_lt * 4 * d1
        for _ in range(s.n_types):
            layers = []
            cur = din
            for _k in range(s.fit_hidden):
                w = self.blob[at: at + cur * s.fit_width].reshape(cur, s.fit_width)
                at += cur * s.fit_width
                b = self.blob[at: at + s.fit_width]
                at += s.fit_width
                layers.append((w, b))
                cur = s.fit_width
            w_out = self.blob[at: at + cur]
            at += cur
            b_out = self.blob[at: at + 1]
            at += 1
            self.fitting.append({"hidden": layers, "w_out": w_out, "b_out": b_out})
        if at != self.blob.size:
            raise InputError("model blob size does not match its shape")

    r_cut = property(lambda self: self.shape.r_cut)
    r_smooth = property(lambda self: self.shape.r_smooth)
    masses = property(lambda self: list(self.shape.masses))
    max_nbr = property(lambda self: list(self.shape.max_nbr))
    m_lt = property(lambda self: self.shape.m_lt)

    def n_types(self) -> int:
        return self.shape.n_types

    def feature_width(self) -> int:
        return 4 * self.shape.d1

    def descriptor_size(self) -> int:
        return self.shape.m_lt * self.feature_width()

    def copy(self) -> "DPModel":
        s = self.shape
        shape = Preset(s.name, s.n_types, list(s.masses), list(s.max_nbr), s.r_cut, s.r_smooth,
                       s.d1, s.m_lt, s.fit_width, s.fit_hidden, s.lattice_a, list(s.site_pattern))
        return DPModel(shape, self.blob.copy())

    def embedding_desc(self):
        """ctypes dp_embedding_desc[n_types] (model.hpp:14-20) plus the arrays it points into."""
        arr = (_EmbDesc * self.shape.n_types)()
        for t, e in enumerate(self.embedding):
            arr[t] = _EmbDesc(self.shape.d1, *[_dp(e[k]) for k in ("w0", "b0", "w1", "b1", "w2", "b2")])
        return arr, [self.blob]

    def desc(self):
        """ctypes dp_model_desc (plus the objects that keep its pointers alive)."""
        s = self.shape
        keep = []
        L = s.fit_hidden
        widths = (C.c_int * (L + 1))(*([s.m_lt * 4 * s.d1] + [s.fit_width] * L))
        keep.append(widths)
        fits = (_Fitting * s.n_types)()
        for t in range(s.n_types):
            f = self.fitting[t]
            ws = (C.POINTER(C.c_double) * L)(*[_dp(w) for w, _ in f["hidden"]])
            bs = (C.POINTER(C.c_double) * L)(*[_dp(b) for _, b in f["hidden"]])
            keep += [ws, bs]
            fits[t].n_layers = L
            fits[t].widths = widths
            fits[t].w = ws
            fits[t].b = bs
            fits[t].w_out = _dp(f["w_out"])
            fits[t].b_out = float(f["b_out"][0])
        masses = np.asarray(s.masses, dtype=np.float64)
        cap = np.asarray(s.max_nbr, dtype=np.int32)
        keep += [fits, masses, cap, self.blob]
        d = _ModelDesc(s.n_types, s.r_cut, s.r_smooth, s.d1, s.m_lt, _dp(masses),
                       cap.ctypes.data_as(C.POINTER(C.c_int)), fits)
        return d, keep


def _blob_size(shape: Preset) -> int:
    n = int(_lib().dp_model_blob_size(C.byref(shape._c())))
    if n < 0:
        raise InputError("inconsistent model shape")
    return n


def gen_model(preset, seed: int) -> DPModel:
    """gen_model(get_preset(name), seed) (model_io.cpp:129-188), bit-identical."""
    p = get_preset(preset) if isinstance(preset, str) else preset
    blob = np.empty(_blob_size(p), dtype=np.float64)
    _check(_lib().dp_gen_model(p.name.encode(), seed, _dp(blob)))
    return DPModel(p, blob)


def make_test_model(n_types: int, d1: int, m_lt: int, fit_width: int, n_hidden: int,
                    max_nbr: Sequence[int], r_cut: float, r_smooth: float, seed: int,
                    fit_scale: float = 0.2) -> DPModel:
    """testutil::make_test_model (tests/helpers.hpp:21-72), bit-identical."""
    p = Preset("test", n_types, [10.0 + t for t in range(n_types)], list(max_nbr), r_cut, r_smooth,
               d1, m_lt, fit_width, n_hidden)
    blob = np.empty(_blob_size(p), dtype=np.float64)
    _check(_lib().dp_gen_test_model(C.byref(p._c()), seed, fit_scale, _dp(blob)))
    return DPModel(p, blob)


@dataclass
class ModelFile:
    """ModelFile (model_io.hpp:52-56)."""
    model: "DPModel"
    preset: str = ""
    seed: int = 0
    species: List[str] = field(default_factory=list)


def write_model(path: str, model: DPModel, preset: str = "", seed: int = 0,
                species: Optional[Sequence[str]] = None) -> None:
    """write_model (model_io.cpp:226-250): JSON, shortest round-trip doubles."""
    csv = ",".join(species) if species else None
    _check(_lib().dp_write_model_json(path.encode(), C.byref(model.shape._c()), _dp(model.blob),
                                      csv.encode() if csv else None, preset.encode(), seed))


def read_model(path: str) -> ModelFile:
    """read_model (model_io.cpp:252-283): InputError on unreadable / malformed / inconsistent files."""
    shp = _Preset()
    sp = C.create_string_buffer(512)
    pr = C.create_string_buffer(256)
    sd = C.c_uint64()
    _check(_lib().dp_read_model_json(path.encode(), C.byref(shp), None, 0, sp, 512, pr, 256, C.byref(sd)))
    p = Preset(pr.value.decode(), shp.n_types, [shp.masses[t] for t in range(shp.n_types)],
               [shp.max_nbr[t] for t in range(shp.n_types)], shp.r_cut, shp.r_smooth, shp.d1, shp.m_lt,
               shp.fit_width, shp.fit_hidden)
    blob = np.empty(_blob_size(p), dtype=np.float64)
    _check(_lib().dp_read_model_json(path.encode(), C.byref(shp), _dp(blob), blob.size, sp, 512, pr, 256,
                                     C.byref(sd)))
    return ModelFile(DPModel(p, blob), pr.value.decode(), int(sd.value), sp.value.decode().split(","))


# ---------------------------------------------------------------- tables
class Tables:
    """One CompressionTable per neighbour type (table.hpp:20-35), DPTB header fields."""

    def __init__(self, x0: float, h: float, n: int, m: int, block: int, coeffs: np.ndarray):
        self.x0, self.h, self.n, self.m, self.block = float(x0), float(h), int(n), int(m), int(block)
        self.coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)  # [n_tables, n*stride]
        if self.coeffs.ndim != 2 or self.coeffs.shape[1] != self.n * self.interval_stride():
            raise InputError("table coefficient array has the wrong shape")

    def n_blocks(self) -> int:
        return (self.m + self.block - 1) // self.block

    def interval_stride(self) -> int:
        return self.n_blocks() * 6 * self.block

    def x_end(self) -> float:
        return self.x0 + self.h * float(self.n)

    def __len__(self) -> int:
        return self.coeffs.shape[0]

    def desc(self):
        ptrs = (C.POINTER(C.c_double) * len(self))(*[_dp(self.coeffs[t]) for t in range(len(self))])
        d = _TableDesc(len(self), self.x0, self.h, self.n, self.m, self.block, ptrs)
        return d, [ptrs, self.coeffs]


def build_tables(model: DPModel, h: float) -> Tables:
    """build_tables(model, h) (table.cpp:77-162): quintic Hermite per interval, node-verified."""
    shp = model.shape._c()
    n = C.c_uint64()
    xe = C.c_double()
    _check(_lib().dp_build_tables(C.byref(shp), _dp(model.blob), h, C.byref(n), C.byref(xe), None))
    m = 4 * model.shape.d1
    stride = ((m + 15) // 16) * 6 * 16
    coeffs = np.empty((model.shape.n_types, n.value * stride), dtype=np.float64)
    _check(_lib().dp_build_tables(C.byref(shp), _dp(model.blob), h, C.byref(n), C.byref(xe),
                                  _dp(coeffs)))
    return Tables(0.0, h, n.value, m, 16, coeffs)


def write_tables(path: str, tabs: Tables) -> None:
    d, keep = tabs.desc()
    _check(_lib().dp_write_tables(str(path).encode(), C.byref(d)))


def read_tables(path: str) -> Tables:
    nt, m, blk = C.c_int(), C.c_int(), C.c_int()
    n = C.c_uint64()
    x0, h = C.c_double(), C.c_double()
    _check(_lib().dp_read_tables_header(str(path).encode(), C.byref(nt), C.byref(m), C.byref(blk),
                                        C.byref(n), C.byref(x0), C.byref(h)))
    stride = ((m.value + blk.value - 1) // blk.value) * 6 * blk.value
    coeffs = np.empty((nt.value, n.value * stride), dtype=np.float64)
    _check(_lib().dp_read_tables(str(path).encode(), _dp(coeffs)))
    return Tables(x0.value, h.value, n.value, m.value, blk.value, coeffs)


def tanh_table() -> np.ndarray:
    """TanhTable coefficients (tanh_table.cpp:5-21), [8193, 3]."""
    c = np.empty(3 * 8193, dtype=np.float64)
    _check(_lib().dp_tanh_table(_dp(c)))
    return c.reshape(8193, 3)


# ---------------------------------------------------------------- configurations
@dataclass
class AtomicConfig:
    """AtomicConfig + Cell (geom.hpp:14-54): rows of h are the cell vectors."""
    pos: np.ndarray            # (n, 3) float64, raw (unwrapped) cartesian
    type: np.ndarray           # (n,) int32
    h: np.ndarray              # (9,) float64
    periodic: np.ndarray = field(default_factory=lambda: np.ones(3, dtype=np.uint8))

    def __post_init__(self):
        self.pos = np.ascontiguousarray(np.asarray(self.pos, dtype=np.float64).reshape(-1, 3))
        self.type = np.ascontiguousarray(np.asarray(self.type, dtype=np.int32).reshape(-1))
        self.h = np.ascontiguousarray(np.asarray(self.h, dtype=np.float64).reshape(9))
        self.periodic = np.ascontiguousarray(np.asarray(self.periodic, dtype=np.uint8).reshape(3))

    @property
    def n_atoms(self) -> int:
        return int(self.pos.shape[0])

    def volume(self) -> float:
        a, b, c = self.h[0:3], self.h[3:6], self.h[6:9]
        return abs(float(np.dot(a, np.cross(b, c))))

    def copy(self) -> "AtomicConfig":
        return AtomicConfig(self.pos.copy(), self.type.copy(), self.h.copy(), self.periodic.copy())


def gen_config(preset, nx: int, ny: int, nz: int, jitter: float, seed: int) -> AtomicConfig:
    """Jittered FCC block (model_io.cpp:190-224), bit-identical."""
    name = preset if isinstance(preset, str) else preset.name
    n = 4 * nx * ny * nz
    pos = np.empty((n, 3), dtype=np.float64)
    ty = np.empty(n, dtype=np.int32)
    h = np.empty(9, dtype=np.float64)
    _check(_lib().dp_gen_config(name.encode(), nx, ny, nz, jitter, seed, _dp(pos), _ip(ty), _dp(h)))
    return AtomicConfig(pos, ty, h)


def make_random_config(n: int, n_types: int, box: float, min_sep: float, seed: int) -> AtomicConfig:
    """testutil::make_random_config (tests/helpers.hpp:75-99), bit-identical."""
    pos = np.empty((n, 3), dtype=np.float64)
    ty = np.empty(n, dtype=np.int32)
    _check(_lib().dp_gen_random_config(n, n_types, box, min_sep, seed, _dp(pos), _ip(ty)))
    return AtomicConfig(pos, ty, np.array([box, 0, 0, 0, box, 0, 0, 0, box], dtype=np.float64))


def init_velocities(cfg: AtomicConfig, model: DPModel, t_init: float, seed: int) -> np.ndarray:
    """Maxwell-Boltzmann draw, momentum removed, rescaled to t_init (md.cpp:14-55)."""
    vel = np.empty((cfg.n_atoms, 3), dtype=np.float64)
    masses = np.asarray(model.masses, dtype=np.float64)
    _check(_lib().dp_init_velocities(cfg.n_atoms, _ip(cfg.type), _dp(masses), t_init, seed, _dp(vel)))
    return vel


# ---------------------------------------------------------------- results
@dataclass
class FusedCounters:
    """FusedCounters (fused.hpp:10-21)."""
    rows_forward: int = 0
    rows_backward: int = 0
    extrapolations: int = 0


@dataclass
class EvalResult:
    """EvalResult (exact.hpp:12-17)."""
    energy: float
    per_atom_energy: np.ndarray
    forces: np.ndarray
    virial: np.ndarray  # (9,), virial[3x+y] = sum d_x g_y


@dataclass
class NeighborList:
    """NeighborList (neighbor.hpp:20-24) in CSR form, canonical order."""
    cutoff: float
    offsets: np.ndarray  # (n+1,) int64
    j: np.ndarray        # (E,) int32
    shift: np.ndarray    # (E, 3) int32

    def row(self, i: int):
        a, b = self.offsets[i], self.offsets[i + 1]
        return self.j[a:b], self.shift[a:b]


@dataclass
class MDConfig:
    """MDConfig (md.hpp:14-21)."""
    n_steps: int = 0
    dt: float = 1.0
    n_workers: int = 1
    buffer: float = 2.0
    rebuild_every: int = 50
    thermo_every: int = 50


@dataclass
class ThermoRecord:
    step: int
    ke: float
    pe: float
    temperature: float
    pressure: float


@dataclass
class MDResult:
    thermo: List[ThermoRecord]
    force_evals: int
    staleness_checks: int
    max_drift_seen: float
    counters: FusedCounters
    final_ke: float
    final_pe: float
    final_total: float


# ---------------------------------------------------------------- the GPU handle
class DeepPot:
    """One dp_handle: model + tables resident on one B200, evaluation on sm_100a kernels."""

    def __init__(self, model: DPModel, tables: Optional[Tables] = None, device: int = 0,
                 precision: str = "fp64"):
        """tables=None: build them on the GPU later with build_tables_gpu(h)."""
        if precision not in ("fp64", "mixed"):
            raise InputError("precision must be 'fp64' or 'mixed'")
        self.model, self.tables = model, tables
        md, self._mkeep = model.desc()
        if tables is not None:
            td, self._tkeep = tables.desc()
            tdp = C.byref(td)
        else:
            tdp = None
        h = C.c_void_p()
        rc = _lib().dp_create(C.byref(md), tdp, device, 0 if precision == "fp64" else 1, C.byref(h))
        _check(rc, None)
        self._h = h
        ed, keep = model.embedding_desc()
        _check(_lib().dp_set_embedding(self._h, ed), self._h)
        self.counters = FusedCounters()

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib().dp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_skin(self, skin: float) -> None:
        _check(_lib().dp_set_skin(self._h, skin), self._h)

    @property
    def stream(self) -> int:
        return int(_lib().dp_stream(self._h) or 0)

    @property
    def launch_count(self) -> int:
        return int(_lib().dp_launch_count(self._h))

    PHASES = ("nlist", "tab_fwd", "fitting", "tab_bwd", "forces", "integrate", "halo")

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(_lib().dp_nccl_unique_id(buf, 128))
        return buf.raw

    def dist_init(self, rank: int, world: int, nccl_id: bytes) -> None:
        """Join a domain-decomposed run (one handle per GPU process)."""
        _check(_lib().dp_dist_init(self._h, rank, world, nccl_id), self._h)
        self._dist = True

    def set_pipeline(self, enable: bool) -> None:
        """Two-stream pipelined evaluation (on by default; FP64 single-type systems)."""
        _check(_lib().dp_set_pipeline(self._h, 1 if enable else 0), self._h)

    def set_chunk_size(self, centres: int) -> None:
        """Largest number of centres per evaluation chunk (0 = default); results are bitwise
        independent of it."""
        _check(_lib().dp_set_chunk_size(self._h, int(centres)), self._h)

    def set_timing(self, enable: bool) -> None:
        _check(_lib().dp_set_timing(self._h, int(enable)), self._h)

    def phase_times(self) -> dict:
        ms = np.zeros(8)
        cnt = (C.c_uint64 * 8)()
        _check(_lib().dp_phase_times(self._h, _dp(ms), cnt), self._h)
        return {name: (float(ms[k]), int(cnt[k])) for k, name in enumerate(self.PHASES)}

    def compute(self, cfg: AtomicConfig, energy_out=None, forces_out=None) -> EvalResult:
        n = cfg.n_atoms
        e = C.c_double()
        f = forces_out if forces_out is not None else np.empty((n, 3), dtype=np.float64)
        v = np.empty(9, dtype=np.float64)
        ae = np.empty(n, dtype=np.float64)
        rc = _lib().dp_compute(self._h, n, _dp(cfg.pos), _ip(cfg.type), _dp(cfg.h),
                               _u8(cfg.periodic), C.byref(e), _dp(f), _dp(v), _dp(ae))
        _check(rc, self._h)
        c = _Counters()
        _lib().dp_counters_get(self._h, C.byref(c))
        self.counters = FusedCounters(c.rows_forward, c.rows_backward, c.extrapolations)
        return EvalResult(e.value, ae, f, v)

    def compute_with_list(self, cfg: AtomicConfig, nlist: "NeighborList") -> EvalResult:
        """compute_energy_forces_virial_tabulated(cfg, model, tables, list) (fused.hpp:70-73) on
        the caller's full, symmetric neighbour list (any cutoff >= r_cut)."""
        n = cfg.n_atoms
        e = C.c_double()
        f = np.empty((n, 3), dtype=np.float64)
        v = np.empty(9, dtype=np.float64)
        ae = np.empty(n, dtype=np.float64)
        off = np.ascontiguousarray(nlist.offsets, dtype=np.int64)
        j = np.ascontiguousarray(nlist.j, dtype=np.int32)
        sh = np.ascontiguousarray(nlist.shift, dtype=np.int32).reshape(-1)
        rc = _lib().dp_compute_list(self._h, n, _dp(cfg.pos), _ip(cfg.type), _dp(cfg.h), _u8(cfg.periodic),
                                    off.ctypes.data_as(C.POINTER(C.c_int64)), _ip(j), _ip(sh), C.byref(e),
                                    _dp(f), _dp(v), _dp(ae))
        _check(rc, self._h)
        c = _Counters()
        _lib().dp_counters_get(self._h, C.byref(c))
        self.counters = FusedCounters(c.rows_forward, c.rows_backward, c.extrapolations)
        return EvalResult(e.value, ae, f, v)

    def compute_exact(self, cfg: AtomicConfig) -> EvalResult:
        """compute_energy_forces_virial (exact.cpp:155-173): full embedding net, on the GPU."""
        n = cfg.n_atoms
        e = C.c_double()
        f = np.empty((n, 3), dtype=np.float64)
        v = np.empty(9, dtype=np.float64)
        ae = np.empty(n, dtype=np.float64)
        rc = _lib().dp_compute_exact(self._h, n, _dp(cfg.pos), _ip(cfg.type), _dp(cfg.h),
                                     _u8(cfg.periodic), C.byref(e), _dp(f), _dp(v), _dp(ae))
        _check(rc, self._h)
        return EvalResult(e.value, ae, f, v)

    def build_tables_gpu(self, h: float, install: bool = True) -> Tables:
        """build_tables (table.cpp:77-162) on the GPU from this handle's embedding nets."""
        n = C.c_uint64()
        xe = C.c_double()
        _check(_lib().dp_build_tables_gpu(self._h, h, C.byref(n), C.byref(xe), None, 0), self._h)
        m = 4 * self.model.shape.d1
        stride = ((m + 15) // 16) * 6 * 16
        coeffs = np.empty((self.model.shape.n_types, n.value * stride), dtype=np.float64)
        _check(_lib().dp_build_tables_gpu(self._h, h, C.byref(n), C.byref(xe), _dp(coeffs),
                                          1 if install else 0), self._h)
        tabs = Tables(0.0, h, n.value, m, 16, coeffs)
        if install:
            self.tables = tabs
        return tabs

    def rmse_sweep(self, h_list: Sequence[float], configs: Sequence[AtomicConfig]) -> List["SweepRow"]:
        """rmse_sweep (rmse.cpp:63-97): GPU tables per step vs the GPU exact path."""
        if len(h_list) == 0:
            raise InputError("sweep needs at least one step size")
        na = np.array([c.n_atoms for c in configs], dtype=np.int64)
        pos = np.ascontiguousarray(np.concatenate([c.pos.reshape(-1) for c in configs]) if configs else
                                   np.zeros(1), dtype=np.float64)
        typ = np.ascontiguousarray(np.concatenate([c.type for c in configs]) if configs else
                                   np.zeros(1, dtype=np.int32), dtype=np.int32)
        box = np.ascontiguousarray(np.concatenate([c.h.reshape(-1) for c in configs]) if configs else
                                   np.zeros(9), dtype=np.float64)
        pbc = np.ascontiguousarray(np.concatenate([c.periodic for c in configs]) if configs else
                                   np.zeros(3, dtype=np.uint8), dtype=np.uint8)
        hl = np.ascontiguousarray(h_list, dtype=np.float64)
        re = np.empty(len(hl), dtype=np.float64)
        rf = np.empty(len(hl), dtype=np.float64)
        _check(_lib().dp_rmse_sweep(self._h, len(configs), na.ctypes.data_as(C.POINTER(C.c_int64)), _dp(pos),
                                    _ip(typ), _dp(box), _u8(pbc), len(hl), _dp(hl), _dp(re), _dp(rf)),
               self._h)
        return [SweepRow(float(h), float(e), float(f)) for h, e, f in zip(hl, re, rf)]

    def neighbor_list(self, cfg: AtomicConfig, cutoff: float) -> NeighborList:
        total = C.c_int64()
        rc = _lib().dp_neighbor_list_build(self._h, cfg.n_atoms, _dp(cfg.pos), _ip(cfg.type),
                                           _dp(cfg.h), _u8(cfg.periodic), cutoff, C.byref(total))
        _check(rc, self._h)
        off = np.empty(cfg.n_atoms + 1, dtype=np.int64)
        j = np.empty(max(total.value, 1), dtype=np.int32)
        s = np.empty((max(total.value, 1), 3), dtype=np.int32)
        _check(_lib().dp_neighbor_list_get(self._h, off.ctypes.data_as(C.POINTER(C.c_int64)),
                                           _ip(j), _ip(s)), self._h)
        return NeighborList(cutoff, off, j[: total.value], s[: total.value])

    def run_md(self, cfg: AtomicConfig, vel: np.ndarray, mc: MDConfig) -> MDResult:
        """run_md (md.cpp:151-231) device resident; cfg.pos and vel are updated in place."""
        vel_arr = np.ascontiguousarray(vel, dtype=np.float64).reshape(-1, 3)
        if vel_arr.shape[0] != cfg.n_atoms:
            raise InputError("velocity array size mismatch")
        c = _MDConfig(mc.n_steps, mc.dt, mc.buffer, mc.rebuild_every, mc.thermo_every)
        cap = mc.n_steps // max(mc.thermo_every, 1) + 2
        th = (_Thermo * cap)()
        nth = C.c_int64()
        res = _MDResult()
        rc = _lib().dp_md_run(self._h, cfg.n_atoms, _dp(cfg.pos), _dp(vel_arr), _ip(cfg.type),
                              _dp(cfg.h), _u8(cfg.periodic), C.byref(c), th, cap, C.byref(nth),
                              C.byref(res))
        _check(rc, self._h)
        if vel_arr is not vel:
            np.copyto(vel, vel_arr.reshape(np.shape(vel)))
        return _md_result(th, nth.value, res)

    # split form for benchmarking (device-resident state between calls)
    def md_begin(self, cfg: AtomicConfig, vel: np.ndarray, mc: MDConfig) -> None:
        vel = np.ascontiguousarray(vel, dtype=np.float64)
        c = _MDConfig(mc.n_steps, mc.dt, mc.buffer, mc.rebuild_every, mc.thermo_every)
        rc = _lib().dp_md_begin(self._h, cfg.n_atoms, _dp(cfg.pos), _dp(vel), _ip(cfg.type),
                                _dp(cfg.h), _u8(cfg.periodic), C.byref(c))
        _check(rc, self._h)
        self._md_n = cfg.n_atoms
        self._md_cap = mc.n_steps // max(mc.thermo_every, 1) + 2

    def md_step(self, k: int) -> None:
        _check(_lib().dp_md_step(self._h, k), self._h)

    def md_end(self, pos_out: Optional[np.ndarray] = None, vel_out: Optional[np.ndarray] = None) -> MDResult:
        if pos_out is not None:
            assert pos_out.flags.c_contiguous and pos_out.dtype == np.float64
        if vel_out is not None:
            assert vel_out.flags.c_contiguous and vel_out.dtype == np.float64
        cap = self._md_cap
        th = (_Thermo * cap)()
        nth = C.c_int64()
        res = _MDResult()
        rc = _lib().dp_md_end(self._h, _dp(pos_out) if pos_out is not None else None,
                              _dp(vel_out) if vel_out is not None else None, th, cap,
                              C.byref(nth), C.byref(res))
        _check(rc, self._h)
        return _md_result(th, nth.value, res)


def _md_result(th, n, res: _MDResult) -> MDResult:
    recs = [ThermoRecord(int(th[k].step), th[k].ke, th[k].pe, th[k].temperature, th[k].pressure)
            for k in range(min(n, len(th)))]
    c = res.counters
    return MDResult(recs, int(res.force_evals), int(res.staleness_checks), res.max_drift_seen,
                    FusedCounters(c.rows_forward, c.rows_backward, c.extrapolations),
                    res.final_ke, res.final_pe, res.final_total)


def partition_domain(cfg: AtomicConfig, n_workers: int, margin: float):
    """partition_domain (domain.hpp:29): (owner[n], ghost_mask[n_workers, n]) on the host."""
    n = cfg.n_atoms
    owner = np.empty(n, dtype=np.int32)
    gm = np.empty((n_workers, n), dtype=np.uint8)
    _check(_lib().dp_partition_domain(n, _dp(cfg.pos), _dp(cfg.h), _u8(cfg.periodic), n_workers,
                                      margin, _ip(owner), _u8(gm)))
    return owner, gm.astype(bool)


def dist_plan(cfg: AtomicConfig, n_workers: int, rank: int, margin: float) -> dict:
    """Host plan of one rank of the decomposed run (local ids, centre mask, per-peer exchange)."""
    n = cfg.n_atoms
    I64P = C.POINTER(C.c_int64)
    nl = C.c_int64()
    lgid = np.empty(n, dtype=np.int64)
    cen = np.empty(n, dtype=np.uint8)
    so = np.empty(n_workers + 1, dtype=np.int64)
    ro = np.empty(n_workers + 1, dtype=np.int64)
    sg = np.empty(n, dtype=np.int64)
    rg = np.empty(n, dtype=np.int64)
    _check(_lib().dp_dist_plan(n, _dp(cfg.pos), _dp(cfg.h), _u8(cfg.periodic), n_workers, rank, margin,
                               C.byref(nl), lgid.ctypes.data_as(I64P), _u8(cen), so.ctypes.data_as(I64P),
                               sg.ctypes.data_as(I64P), ro.ctypes.data_as(I64P), rg.ctypes.data_as(I64P)))
    k = nl.value
    return {"lgid": lgid[:k], "center": cen[:k].astype(bool),
            "send": {p: sg[so[p]:so[p + 1]] for p in range(n_workers)},
            "recv": {p: rg[ro[p]:ro[p + 1]] for p in range(n_workers)}}


# ---------------------------------------------------------------- reference-named functions
_pots: dict = {}


def _pot(model: DPModel, tables: Tables) -> DeepPot:
    key = (id(model), id(tables))
    p = _pots.get(key)
    if p is None or p.model is not model or p.tables is not tables:
        p = DeepPot(model, tables)
        _pots[key] = p
    return p


def build_neighbor_list(cfg: AtomicConfig, cutoff: float, model: Optional[DPModel] = None,
                        tables: Optional[Tables] = None) -> NeighborList:
    """build_neighbor_list (neighbor.cpp:162-179) on the GPU; bit-exact canonical order."""
    if model is None:
        # any handle can build lists; use a 1-type dummy model of the smallest shape
        global _nl_pot
        try:
            pot = _nl_pot
        except NameError:
            m = make_test_model(1, 1, 1, 1, 1, [1], 1.0, 0.5, 1)
            t = build_tables(m, 0.5)
            pot = _nl_pot = DeepPot(m, t)
        cfg = AtomicConfig(cfg.pos, np.zeros(cfg.n_atoms, dtype=np.int32), cfg.h, cfg.periodic)
    else:
        pot = _pot(model, tables)
    return pot.neighbor_list(cfg, cutoff)


def compute_energy_forces_virial_tabulated(cfg: AtomicConfig, model: DPModel, tables: Tables,
                                           nlist=None, n_workers: int = 1,
                                           counters: Optional[FusedCounters] = None) -> EvalResult:
    """compute_energy_forces_virial_tabulated (fused.hpp:70-73) on the GPU.

    `nlist` may be a NeighborList or a cutoff; its entries beyond r_cut never contribute
    (env_mat.cpp:32), so results do not depend on it. n_workers is accepted for signature parity.
    """
    if n_workers < 1:
        raise InputError("worker count must be at least 1")
    pot = _pot(model, tables)
    cutoff = model.r_cut
    if isinstance(nlist, NeighborList):
        cutoff = nlist.cutoff
    elif nlist is not None:
        cutoff = float(nlist)
    pot.set_skin(max(0.0, cutoff - model.r_cut))
    res = pot.compute(cfg)
    if counters is not None:
        counters.rows_forward += pot.counters.rows_forward
        counters.rows_backward += pot.counters.rows_backward
        counters.extrapolations += pot.counters.extrapolations
    return res


def run_md(cfg: AtomicConfig, vel: np.ndarray, model: DPModel, tables: Tables,
           mc: MDConfig) -> MDResult:
    """run_md (md.hpp:58-60) on the GPU; cfg.pos and vel are updated in place."""
    if mc.n_workers < 1:
        raise InputError("worker count must be at least 1")
    return _pot(model, tables).run_md(cfg, vel, mc)


# ---------------------------------------------------------------- exact path and rmse tooling
@dataclass
class RmseReport:
    """RmseReport (rmse.hpp:15-19)."""
    rmse_e: float = 0.0
    rmse_f: float = 0.0
    n_configs: int = 0


@dataclass
class SweepRow:
    """SweepRow (rmse.hpp:24-28)."""
    h: float = 0.0
    rmse_e: float = 0.0
    rmse_f: float = 0.0


def _exact_pot(model: DPModel) -> DeepPot:
    key = ("exact", id(model))
    p = _pots.get(key)
    if p is None or p.model is not model:
        p = DeepPot(model, None)
        _pots[key] = p
    return p


def compute_energy_forces_virial(cfg: AtomicConfig, model: DPModel, nlist=None) -> EvalResult:
    """compute_energy_forces_virial (exact.cpp:155-173) on the GPU: full embedding nets."""
    pot = _exact_pot(model)
    cutoff = model.r_cut
    if isinstance(nlist, NeighborList):
        cutoff = nlist.cutoff
    elif nlist is not None:
        cutoff = float(nlist)
    pot.set_skin(max(0.0, cutoff - model.r_cut))
    return pot.compute_exact(cfg)


def build_tables_gpu(model: DPModel, h: float) -> Tables:
    """build_tables (table.cpp:77-162) evaluated on the GPU."""
    return _exact_pot(model).build_tables_gpu(h, install=False)


def rmse_compare(model: DPModel, tables: Tables, configs: Sequence[AtomicConfig],
                 n_workers: int = 1) -> RmseReport:
    """rmse_compare (rmse.cpp:48-59): tabulated vs exact energies / forces, both on the GPU."""
    sde2 = sdf2 = 0.0
    ncomp = 0
    nat = 0
    for cfg in configs:
        ref = compute_energy_forces_virial(cfg, model)
        tab = compute_energy_forces_virial_tabulated(cfg, model, tables, n_workers=n_workers)
        de = ref.energy - tab.energy
        sde2 += de * de
        df = np.asarray(ref.forces).reshape(-1) - np.asarray(tab.forces).reshape(-1)
        sdf2 += float(np.dot(df, df))
        ncomp += df.size
        nat = cfg.n_atoms
    r = RmseReport(n_configs=len(configs))
    if configs:
        r.rmse_e = float(np.sqrt(sde2 / len(configs)) / nat)
        r.rmse_f = float(np.sqrt(sdf2 / ncomp))
    return r


def rmse_sweep(model: DPModel, h_list: Sequence[float], configs: Sequence[AtomicConfig],
               n_workers: int = 1) -> List[SweepRow]:
    """rmse_sweep (rmse.cpp:63-97) on the GPU (a fresh handle; tables built per step on device)."""
    pot = DeepPot(model, None)
    try:
        return pot.rmse_sweep(h_list, configs)
    finally:
        pot.close()


def loglog_slope(rows: Sequence[SweepRow]) -> float:
    """loglog_slope (rmse.cpp:99-116): least-squares slope of log(rmse_e) vs log(h)."""
    sx = sy = sxx = sxy = 0.0
    n = 0
    for r in rows:
        if not (r.h > 0.0) or not (r.rmse_e > 0.0):
            continue
        x, y = math.log(r.h), math.log(r.rmse_e)
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
        n += 1
    if n < 2:
        return 0.0
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)
