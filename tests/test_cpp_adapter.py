"""The C++ adapter (include/fastmtgp_b200.hpp) compiles against the C ABI, maps errors onto the
reference's exception types, and on a GPU reproduces the reference seam."""
import numpy as np
import pytest

from paper_2603_16014_b200.designs import Hyper, digital_design, lattice_design, normal
from tests import cpp_adapter


def _case(kind):
    dz = (lattice_design if kind == 0 else digital_design)(2, [5, 3], seed=3)
    hp = Hyper(gamma=1.2, eta=np.array([0.8, 0.5]), B=np.array([[0.7], [-0.4]]), t=np.array([0.3, 0.4]),
               xi=np.array([1e-4, 2e-4]), si_alpha=2, b=(0.5, 0.2, 0.1, 1.0))
    return dz, hp, normal(2, 1, np.arange(dz.N))


def test_adapter_builds_and_maps_missing_gpu_to_fastmtgperror():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu test")
    dz, hp, y = _case(0)
    out = cpp_adapter.run(dz, hp, hp.R, y)
    assert out["rc"] == 3 and "FastMtgpError" in out["stderr"]


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [0, 1])
def test_adapter_matches_reference_seam(ref, kind):
    dz, hp, y = _case(kind)
    out = cpp_adapter.run(dz, hp, hp.R, y)
    assert out["rc"] == 0, out["stderr"]
    x_ref, _, ld_ref, _, _ = ref.invert_solve(dz, hp, y)
    assert abs(out["logdet"] - ld_ref) <= 1e-8 * dz.N
    assert np.linalg.norm(out["x"] - x_ref) <= 1e-10 * np.linalg.norm(x_ref)
