"""Seeded input generators (paper_2204_04321_b200/meshgen.py): determinism,
validity of the footprints and the sizes of the BASELINE.json configs."""
import hashlib

import numpy as np
import pytest

from paper_2204_04321_b200 import meshgen as mg


def test_splitmix64_reference_vectors():
    # canonical splitmix64 outputs (Vigna's reference implementation)
    r = mg.SplitMix64(0)
    assert [int(x) for x in r.next_u64(2)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4]
    r = mg.SplitMix64(1234567)
    assert [int(x) for x in r.next_u64(5)] == [
        6457827717110365317, 3203168211198807973, 9817491932198370423,
        4593380528125082431, 16408922859458223821]
    u = mg.SplitMix64(5).uniform(100000)
    assert 0.0 < u.min() and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    z = mg.SplitMix64(5).normal(100001)
    assert abs(z.mean()) < 0.02 and abs(z.std() - 1.0) < 0.02


def _digest(fp):
    h = hashlib.sha256()
    for a in (fp.xy, fp.tri, fp.sigma, fp.thickness, fp.surface, fp.beta, fp.U):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _check_valid(fp):
    p = fp.xy[fp.tri]
    cross = (p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) - \
            (p[:, 2, 0] - p[:, 0, 0]) * (p[:, 1, 1] - p[:, 0, 1])
    assert (cross > 0).all()
    assert np.array_equal(np.unique(fp.tri), np.arange(fp.n_vert))
    e = np.concatenate([fp.tri[:, [0, 1]], fp.tri[:, [1, 2]], fp.tri[:, [2, 0]]])
    E = np.unique(np.sort(e, axis=1), axis=0)
    assert fp.n_vert - len(E) + fp.n_tri == 1          # simply connected
    assert fp.thickness.min() >= 10.0
    assert fp.sigma[0] == 0.0 and fp.sigma[-1] == 1.0 and np.all(np.diff(fp.sigma) > 0)
    assert np.isfinite(fp.U).all() and fp.U.size == fp.n_dof
    assert fp.tri.dtype == np.int32


@pytest.mark.parametrize("make", [mg.ismip_hom_a, lambda: mg.greenland_like(16.0),
                                  lambda: mg.antarctica_like(D_km=200.0)])
def test_generators_valid_and_deterministic(make):
    a, b = make(), make()
    _check_valid(a)
    assert _digest(a) == _digest(b)


def test_c1_counts():
    fp = mg.ismip_hom_a()
    assert (fp.n_vert, fp.n_tri, fp.n_layers, fp.n_elem, fp.n_dof) == (441, 800, 5, 4000, 5292)


def test_c3_size_matches_paper_triangle_count():
    """C3: N_t within 2% of the paper's 479,930, 10 layers."""
    fp = mg.greenland_like_1_10()
    _check_valid(fp)
    assert abs(fp.n_tri - 479930) <= 0.02 * 479930
    assert fp.n_layers == 10
    # floating margin columns exist (bed below flotation)
    assert (fp.params["rho"] * fp.thickness < -fp.params["rho_w"] * fp.bed).any()


def test_c5_has_floating_embayments():
    fp = mg.antarctica_like(D_km=200.0)
    fl = fp.params["rho"] * fp.thickness < -fp.params["rho_w"] * fp.bed
    assert fl.mean() > 0.01


def test_hilbert_order_is_local():
    """consecutive triangles are spatially close (compact contiguous ranges)."""
    fp = mg.greenland_like(16.0)
    cen = fp.xy[fp.tri].mean(axis=1)
    step = np.hypot(*np.diff(cen, axis=0).T)
    assert np.median(step) < 3 * 16e3


def test_sub_footprint_slices_consistently():
    fp = mg.greenland_like(40.0, n_layers=3)
    sub = mg.sub_footprint(fp, 10, 60)
    assert sub.n_tri == 50
    verts = np.unique(fp.tri[10:60])
    assert np.array_equal(sub.xy, fp.xy[verts])
    assert np.array_equal(sub.U.reshape(-1, 4, 2), fp.U.reshape(-1, 4, 2)[verts])
    assert np.array_equal(verts[sub.tri], fp.tri[10:60])
