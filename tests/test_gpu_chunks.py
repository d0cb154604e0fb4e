"""Chunked evaluation (engine.hpp "chunked evaluation"): the centres are evaluated in chunks of
consecutive slots with two buffer sets, so the per-step working set is bounded by the chunk
size instead of the system. Every per-centre computation is independent of the chunking
(same kernels, same per-centre summation order, same GEMM K order per row), so results must
be BITWISE equal to the one-chunk evaluation, and within 1e-10 of the oracle.
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_2201_01446_b200 as dp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cu():
    m = dp.gen_model("copper-like", 7)
    t = dp.build_tables(m, 0.01)
    return m, t


def same(a, b):
    assert a.energy == b.energy
    assert np.array_equal(a.forces, b.forces)
    assert np.array_equal(a.virial, b.virial)
    assert np.array_equal(a.per_atom_energy, b.per_atom_energy)


@pytest.mark.parametrize("chunk", [128, 384, 1024])
def test_c1_chunks_bitwise_and_oracle(cu, chunk):
    m, t = cu
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    whole = dp.DeepPot(m, t)
    r1 = whole.compute(c)
    pot = dp.DeepPot(m, t)
    pot.set_chunk_size(chunk)
    r = pot.compute(c)
    same(r, r1)
    assert pot.counters == whole.counters
    ro, co = O.or_compute(c, m, t)
    assert abs(r.energy - ro.energy) <= 1e-10 * abs(ro.energy)
    assert O.normwise(r.forces, ro.forces) <= 1e-10
    assert O.normwise(r.virial, ro.virial) <= 1e-10
    assert pot.counters == co


def test_c2_many_chunks_two_streams_bitwise(cu):
    # 32,000 centres: default plan = 2 chunks on two streams; 4,096 -> 8 chunks alternating
    m, t = cu
    c = dp.gen_config("copper-like", 20, 20, 20, 0.1, 11)
    a = dp.DeepPot(m, t)
    ra = a.compute(c)
    b = dp.DeepPot(m, t)
    b.set_chunk_size(4096)
    rb = b.compute(c)
    same(ra, rb)
    b.set_pipeline(False)  # same chunks, one stream
    same(ra, b.compute(c))
    b.set_chunk_size(1 << 20)  # one chunk
    same(ra, b.compute(c))
    assert a.counters == b.counters


def test_mixed_chunks_bitwise(cu):
    m, t = cu
    c = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    a = dp.DeepPot(m, t, precision="mixed")
    ra = a.compute(c)
    b = dp.DeepPot(m, t, precision="mixed")
    b.set_chunk_size(512)
    same(ra, b.compute(c))


def test_md_chunked_bitwise(cu):
    m, t = cu
    base = dp.gen_config("copper-like", 8, 8, 8, 0.1, 11)
    mc = dp.MDConfig(n_steps=30, dt=1.0, buffer=2.0, rebuild_every=10, thermo_every=5)
    runs = []
    for chunk in (0, 640):
        c = base.copy()
        v = dp.init_velocities(c, m, 330.0, 99)
        pot = dp.DeepPot(m, t)
        if chunk:
            pot.set_chunk_size(chunk)
        runs.append((pot.run_md(c, v, mc), c.pos.copy(), v.copy()))
    (ra, pa, va), (rb, pb, vb) = runs
    assert [x.pe for x in ra.thermo] == [x.pe for x in rb.thermo]
    assert np.array_equal(pa, pb) and np.array_equal(va, vb)


def test_exact_path_after_chunked(cu):
    # the exact (untabulated) path evaluates the whole system as one chunk, then the
    # tabulated path returns to its chunk plan
    m, t = cu
    c = dp.gen_config("copper-like", 6, 6, 6, 0.1, 5)
    pot = dp.DeepPot(m, t)
    pot.set_chunk_size(128)
    r1 = pot.compute(c)
    ex = pot.compute_exact(c)
    r2 = pot.compute(c)
    same(r1, r2)
    assert abs(ex.energy - r1.energy) <= 1e-4 * abs(r1.energy)


def test_chunk_size_rejects_negative(cu):
    m, t = cu
    pot = dp.DeepPot(m, t)
    with pytest.raises(dp.InputError):
        pot.set_chunk_size(-1)


def test_c3_chunk_size_bitwise_at_scale(cu):
    """BASELINE C3 size (1,048,576 atoms): 8 chunks of 131,072 vs 32 of 32,768 centres, both on
    two streams, bitwise equal; forces sum to zero (a size-independent property)."""
    m, t = cu
    c = dp.gen_config("copper-like", 64, 64, 64, 0.1, 11)
    pot = dp.DeepPot(m, t)
    a = pot.compute(c)
    pot.set_chunk_size(32768)
    b = pot.compute(c)
    same(a, b)
    fsum = np.abs(a.forces.sum(axis=0)).max()
    assert fsum <= 1e-9 * c.n_atoms * np.abs(a.forces).max()
    pot.close()
