"""Host-side checks of the owner-computes scatter plan (csrc/fo_plan.cpp) with
the library's own planner and no device (fo_plan_check_host): every CSR slot
and residual of a column with rows is written exactly once by a store or by
RED partial sums onto a zero-filled column, and every element entry is gathered
exactly once by the pair of its (column, slot)."""
import numpy as np
import pytest

from paper_2204_04321_b200 import fo, meshgen as mg


def _wheel(spokes):
    th = 2 * np.pi * np.arange(spokes) / spokes
    xy = np.vstack([[0.0, 0.0], np.stack([2e4 * np.cos(th), 2e4 * np.sin(th)], axis=1)])
    tri = np.array([[0, 1 + i, 1 + (i + 1) % spokes] for i in range(spokes)], dtype=np.int32)
    return xy, tri


@pytest.mark.parametrize("case", ["C1", "gris-40km", "C5-small", "wheel-200", "C2"])
def test_plan_covers_every_entry_once(case):
    if case == "wheel-200":
        xy, tri = _wheel(200)
        L = 3
    else:
        fp = {"C1": mg.ismip_hom_a, "gris-40km": lambda: mg.greenland_like(40.0),
              "C5-small": lambda: mg.sub_footprint(mg.antarctica_like(D_km=150.0, n_layers=3), 0, 6000),
              "C2": lambda: mg.greenland_like(16.0)}[case]()
        xy, tri, L = fp.xy, fp.tri, fp.n_layers
    st = fo.plan_check_host(xy, tri, L)
    assert st["bad_slots"] == 0 and st["bad_entries"] == 0, st
    assert st["contributions"] == 9 * tri.shape[0]
    assert st["patches"] >= (tri.shape[0] + 127) // 128


@pytest.mark.parametrize("P", [2, 3])
def test_plan_covers_part_meshes(P):
    fp = mg.greenland_like(40.0, n_layers=4)
    part = fo.partition(fp.n_tri, P)
    for p in range(P):
        st = fo.plan_check_host(fp.xy, fp.tri, fp.n_layers, part=part, n_parts=P, my_part=p)
        assert st["bad_slots"] == 0 and st["bad_entries"] == 0, (p, st)
        assert st["contributions"] == 9 * int((part == p).sum())


def test_plan_c3_statistics():
    """C3: the patch decomposition the bench runs (3 749 patches of <= 128
    triangles, ~38% of the columns zero-filled boundary columns, ~3% of them
    touched by three or more patches)."""
    fp = mg.greenland_like_1_10()
    st = fo.plan_check_host(fp.xy, fp.tri, fp.n_layers)
    assert st["bad_slots"] == 0 and st["bad_entries"] == 0
    assert 0.30 < st["zero_cols"] / fp.n_vert < 0.45
    assert 0.01 < st["multi"] / fp.n_vert < 0.06
    assert st["plan_bytes"] <= 233472 // 2


@pytest.mark.parametrize("case", ["C2", "C3"])
def test_patch_classes_match_the_plan(case):
    """the GPU test's column classes (tests/test_gpu_parity._patch_classes:
    patches touching each column) agree with the library's plan: columns
    touched by >= 2 patches are its zero-filled boundary columns, by >= 3 its
    multi columns -- so the targeted full-size parity samples what it claims.
    The plan halves the few ranges whose plan exceeds the shared-memory budget,
    which only ADDS boundaries: the classes are a lower bound, within 0.5%."""
    from test_gpu_parity import _patch_classes
    fp = mg.greenland_like(16.0) if case == "C2" else mg.greenland_like_1_10()
    st = fo.plan_check_host(fp.xy, fp.tri, fp.n_layers)
    npatch = _patch_classes(fp)
    for got, want in ((int((npatch >= 2).sum()), st["zero_cols"]), (int((npatch >= 3).sum()), st["multi"])):
        assert want * 0.995 <= got <= want


@pytest.mark.parametrize("case", ["C1-quads", "quads-40x40", "quads-33x33-distorted", "quads-700x700"])
def test_quad_plan_covers_every_entry_once(case):
    """NEXT-f4 hexahedra: the quad-patch plan of KH-patch (fo_plan_check_quad_host,
    no device) gathers each of the 16 corner-pair entries of every quad once and
    writes every slot / residual once (store, RED onto a zero fill, or multi
    fix-up); 700 x 700 is the timed mesh (~5 100 patches of <= 96 quads)."""
    fp = {"C1-quads": lambda: mg.to_quads(mg.ismip_hom_a(nx=10, n_layers=5), 10),
          "quads-40x40": lambda: mg.to_quads(mg.ismip_hom_a(nx=40, n_layers=3), 40),
          "quads-33x33-distorted": lambda: mg.to_quads(mg.slab(nx=33, n_layers=2, distort=0.2), 33),
          "quads-700x700": lambda: mg.to_quads(mg.ismip_hom_a(nx=700, n_layers=10), 700)}[case]()
    st = fo.plan_check_quad_host(fp.xy, fp.tri, fp.n_layers)
    assert st["bad_slots"] == 0 and st["bad_entries"] == 0, st
    assert st["contributions"] == 16 * fp.tri.shape[0]
    assert st["patches"] >= (fp.tri.shape[0] + 95) // 96
