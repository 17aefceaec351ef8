"""The product multi-rank path on a real GPU: two processes (one rank each, gloo for the
collectives -- there is one GPU here, and no rank's kernels wait on the other's) both run
pipeline.run with GpuBackend; breakpoints and every slice's eigenvalues must equal the
single-rank run bit for bit (bounds broadcast, KPM per-probe moments all-gathered in probe order,
deterministic device reductions), and only metadata crosses ranks."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CASES = {
    # BASELINE cfg1 (100^2, ChebLanNr, Jackson)
    "cfg1": (dict(xi=0.4, eta=1.6, ns=2, solver="nr", damping="jackson", dos_m=80, dos_nvec=20,
                  probes="rademacher", tol=1e-8, seed=0), [100, 100], None),
    # BASELINE cfg2 (64^3, ChebLanTr, 40 Gaussian probes), its two cheapest slices
    "cfg2": (dict(xi=0.6, eta=1.2, ns=8, solver="tr", damping="sigma", dos_m=100, dos_nvec=40,
                  probes="gaussian", tol=1e-8, seed=1234), [64, 64, 64], [4, 7]),
}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch.distributed as td
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1802_05215_b200.pipeline import Dist, GpuBackend, Plan, run
        plan_kw, dims, only = CASES[case]
        res = run(Plan(**plan_kw, only=only, want_vectors=True), GpuBackend(device=0, dims=dims),
                  Dist(rank, world, None))
        q.put((rank, res.lmin, res.lmax, res.breakpoints.tolist(),
               [(s.index, s.rank, s.eigenvalues.tolist(), s.error,
                 None if s.vectors is None else s.vectors.shape) for s in res.slices]))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("case", ["cfg1", "cfg2"])
def test_two_ranks_equal_single_rank_bitwise(case):
    import torch.multiprocessing as mp
    from paper_1802_05215_b200.pipeline import GpuBackend, Plan, run
    plan_kw, dims, only = CASES[case]
    single = run(Plan(**plan_kw, only=only), GpuBackend(device=0, dims=dims))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want = {s.index: s for s in single.slices}
    for rank, lmin, lmax, bp, slices in out:
        assert (lmin, lmax) == (single.lmin, single.lmax)
        assert bp == single.breakpoints.tolist()
        assert sorted(s[0] for s in slices) == sorted(want)
        for idx, owner, vals, err, vshape in slices:
            assert err is None, err
            assert vals == want[idx].eigenvalues.tolist(), (rank, idx)
            # eigenvectors stay with the owning rank: other ranks receive metadata only
            if owner == rank:
                assert tuple(vshape) == (int(np.prod(dims)), len(vals))
            else:
                assert vshape is None
    owners = {s[1] for _, _, _, _, sl in out for s in sl}
    if case == "cfg1":
        assert owners == {0, 1}
