"""C-ABI library (libfo.so): loads, exports every symbol include/fo.h declares,
host-side graph construction is bit-exact against the oracle's brute force,
and the product path refuses to run without a GPU (no CPU fallback)."""
import ctypes as C

import numpy as np
import pytest

from paper_2204_04321_b200 import fo
from paper_2204_04321_b200 import meshgen as mg


@pytest.fixture(scope="module")
def lib():
    from paper_2204_04321_b200 import _build
    _build.build()
    return fo.lib()


def test_exports_every_declared_symbol(lib):
    names = fo.declared_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), n
    # and the binding wraps all of them
    assert set(names) == set(fo._SIGS) | set(fo._VOID) | {"fo_last_error"}


@pytest.mark.parametrize("name", ["C1", "C1-L1", "gris", "slab-distorted"])
def test_graph_bit_exact_vs_oracle(lib, ora_mod, name):
    fp = {"C1": mg.ismip_hom_a, "C1-L1": lambda: mg.ismip_hom_a(n_layers=1),
          "gris": lambda: mg.greenland_like(60.0, n_layers=6),
          "slab-distorted": lambda: mg.slab(nx=6, n_layers=4, distort=0.2)}[name]()
    rp, col = fo.graph_host(fp.n_vert, fp.tri, fp.n_layers)
    orp, ocol = ora_mod.Oracle(fp).graph()
    assert rp.tobytes() == orp.tobytes()
    assert col.tobytes() == ocol.tobytes()


def test_partition_contiguous(lib):
    part = fo.partition(1001, 4)
    assert part[0] == 0 and part[-1] == 3
    assert np.all(np.diff(part) >= 0)
    assert np.array_equal(part, (np.arange(1001) * 4) // 1001)


def test_no_gpu_fails_loudly(lib):
    """without a CUDA device fo_mesh_create returns FO_ECUDA (there is no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    fp = mg.ismip_hom_a(nx=3, n_layers=2)
    with pytest.raises(fo.FoError) as ei:
        fo.Mesh.from_footprint(fp)
    assert ei.value.status == fo.FO_ECUDA


def test_validation_before_device(lib):
    """mesh validation errors are reported (FO_EMESH / FO_EINVAL) ahead of device use."""
    fp = mg.ismip_hom_a(nx=3, n_layers=2)
    fp.tri = fp.tri.copy()
    fp.tri[0] = fp.tri[0][[0, 2, 1]]
    with pytest.raises(fo.FoError) as ei:
        fo.Mesh.from_footprint(fp)
    assert ei.value.status == fo.FO_EMESH
    assert "CW" in str(ei.value)
    fp = mg.ismip_hom_a(nx=3, n_layers=2)
    with pytest.raises(fo.FoError) as ei:
        fo.Mesh.from_footprint(fp, params=dict(glen_n=-1.0))
    assert ei.value.status == fo.FO_EINVAL


def test_graph_host_rejects_bad_index(lib):
    tri = np.array([[0, 1, 5]], dtype=np.int32)
    with pytest.raises(fo.FoError):
        fo.graph_host(3, tri, 2)
