"""The C++ multi-GPU KPM path (se_kpm_dos_multi / facade kpm_dos_devices / CLI --gpus N): probes
split over the listed GPUs, one thread + context per GPU, per-probe moments combined by ONE
ncclAllReduce of a zero-padded probe-major array.  On the one-GPU test box the device list is
[0]: NCCL still initialises a communicator and runs the all-reduce, and the curve must equal the
single-GPU kpm_dos bit for bit (the exactness argument -- x + 0 = x -- is what makes the N-GPU
result equal too)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_nccl_resolves(gpu_ctx):
    from paper_1802_05215_b200 import api
    assert api.nccl_version() >= 21800


@pytest.mark.parametrize("dims,m,nvec,probes,seed", [
    ([100, 100], 80, 20, "rademacher", 0),      # BASELINE cfg1 DOS
    ([64, 64, 64], 100, 40, "gaussian", 1234),  # BASELINE cfg2 DOS
    ([30, 30], 50, 37, "rademacher", 7),         # ragged: 2 full blocks + 5
])
def test_multi_gpu_kpm_equals_single_gpu_bitwise(gpu_ctx, dims, m, nvec, probes, seed):
    from paper_1802_05215_b200 import api
    a = api.gen_laplacian(dims)
    ev = api.laplacian_analytic_eigs(dims)
    b = api.SpectralBounds(float(ev[0]) - 1e-3, float(ev[-1]) + 1e-3)
    cfg = api.DosConfig(method="kpm", m=m, n_vec=nvec, npts=300, seed=seed, probes=probes)
    one = api.kpm_dos(api.make_operator(a), b, cfg)
    multi = api.kpm_dos_devices(a, b, cfg, [0])
    assert np.array_equal(one.xdos, multi.xdos)
    assert np.array_equal(one.ydos, multi.ydos)
    assert one.nev_est == multi.nev_est


def test_multi_gpu_kpm_errors(gpu_ctx):
    from paper_1802_05215_b200 import api
    a = api.gen_laplacian([10, 10])
    b = api.SpectralBounds(0.0, 8.0)
    with pytest.raises(ValueError):
        api.kpm_dos_devices(a, b, api.DosConfig(m=0, n_vec=4), [0])
    with pytest.raises(RuntimeError):  # a device that does not exist
        api.kpm_dos_devices(a, b, api.DosConfig(m=10, n_vec=4), [0, 97])
