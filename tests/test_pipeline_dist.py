"""Multi-rank plumbing of the pipeline (probe split + all-gather of per-probe moments, slice
ownership, result gather) on CPU with world_size 2 over gloo.  The compute backend here is the
TEST ORACLE (reference library / C restatement) so the plumbing runs without a GPU; the product
backend is pipeline.GpuBackend, exercised by the -m gpu tests and bench.py."""
import os
import socket
import types

import numpy as np
import pytest

from oracle import clib, reflib
from paper_1802_05215_b200 import api
from paper_1802_05215_b200.pipeline import (Dist, Plan, assign_lpt, probe_split, run, slice_owner,
                                            trim_to_slice)

DIMS = [24, 24]
PLAN = dict(xi=0.4, eta=1.6, ns=3, solver="nr", damping="jackson", dos_m=40, dos_nvec=7,
            probes="gaussian", tol=1e-8, seed=5)


class OracleBackend:
    """CPU stand-in for GpuBackend (test-only)."""

    def __init__(self, dims):
        self.rp, self.ci, self.v = clib.laplacian(dims)
        self.n = len(self.rp) - 1

    def bounds(self, seed):
        return reflib.lan_tr_bounds(self.rp, self.ci, self.v, 1e-4, 60, 40, seed)

    def moments(self, lmin, lmax, m, n_vec, seed, probes, first, count):
        kind = "normal" if probes == "gaussian" else "rademacher"
        return np.array([clib.kpm_moments(self.rp, self.ci, self.v, lmin, lmax, m, n_vec, seed,
                                          kind, first=l, count=1)
                         for l in range(first, first + count)]).reshape(count, m + 1)

    def curve(self, zeta, lmin, lmax, npts):
        x, y, nev = clib.kpm_curve(zeta, self.n, lmin, lmax, npts)
        return api.DosCurve(x, y, nev, self.n)

    def solve_slice(self, plan, lmin, lmax, lo, hi, est):
        r = reflib.cheb_lan(self.rp, self.ci, self.v, plan.solver, lo, hi, lmin, lmax,
                            damping=plan.damping, res_tol=plan.tol,
                            est_count=max(1, int(np.ceil(est))), seed=plan.seed)
        res = types.SimpleNamespace(eigenvalues=r["eigenvalues"], residuals=r["residuals"],
                                    vectors=None, niter=r["niter"], hit_max_its=r["hit_max_its"],
                                    counters=types.SimpleNamespace(n_A_matvec=r["n_A_matvec"],
                                                                   t_mv=0.0, t_orth=0.0))
        return r["degree"], res


def test_probe_split_and_ownership():
    for nvec in (1, 7, 40, 128):
        for world in (1, 2, 3, 8):
            spans = [probe_split(nvec, world, r) for r in range(world)]
            flat = [p for f, c in spans for p in range(f, f + c)]
            assert flat == list(range(nvec))  # contiguous, ordered, complete
    assert [slice_owner(i, 4) for i in range(8)] == [0, 1, 2, 3, 0, 1, 2, 3]
    # LPT: the identity at one slice per rank; balanced makespan when slices outnumber ranks
    assert assign_lpt([5, 1, 3], 8) == [0, 1, 2]
    costs = [8.0, 4.5, 5.1, 5.9, 4.0, 6.5, 7.9, 3.6]
    own = assign_lpt(costs, 2)
    loads = [sum(c for c, o in zip(costs, own) if o == r) for r in range(2)]
    assert max(loads) <= 23.0 < sum(costs[0::2])  # better than round-robin (25.0)


def test_trim_to_slice_seams():
    # sliceeig_main.cpp:422-442: a value within delta above an interior breakpoint goes below
    vals = np.array([1.0, 1.0 + 5e-11, 1.5, 2.0 + 5e-11, 2.5])
    keep = trim_to_slice(vals, vals, 1, 3, 1.0, 2.0, 1e-10)
    assert list(keep) == [2, 3]
    assert list(trim_to_slice(vals, vals, 0, 1, 1.0, 2.0, 1e-10)) == [0, 1, 2, 3, 4]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as td
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run(Plan(**PLAN), OracleBackend(DIMS), Dist(rank, world, None))
        q.put((rank, res.lmin, res.lmax, list(res.breakpoints),
               [(s.index, s.rank, list(s.eigenvalues)) for s in res.slices]))
    finally:
        td.destroy_process_group()


def test_two_rank_pipeline_matches_single_rank():
    import torch.multiprocessing as mp
    single = run(Plan(**PLAN), OracleBackend(DIMS), Dist())
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, lmin, lmax, bp, slices in out:
        assert (lmin, lmax) == (single.lmin, single.lmax)
        assert bp == list(single.breakpoints)  # moment gather in probe order: identical curve
        assert [s[0] for s in slices] == [0, 1, 2]
        assert sorted(set(s[1] for s in slices)) == [0, 1]  # both ranks own slices (LPT)
        for (idx, _, vals), ref in zip(slices, single.slices):
            assert vals == list(ref.eigenvalues)
    ev = api.laplacian_analytic_eigs(DIMS)
    assert single.n_found == api.count_in_interval(ev, 0.4, 1.6)


def test_windowed_slices_cover_the_spectrum_once():
    """Memory plan: slices above `window_est` are solved as DOS-mass sub-windows whose seams are
    trimmed like slice seams -- every analytic eigenvalue exactly once (run here through the
    reference library as the solver, so the window logic itself is what is tested)."""
    plan = Plan(**dict(PLAN, ns=2, window_est=12.0))
    res = run(plan, OracleBackend(DIMS), Dist())
    ev = api.laplacian_analytic_eigs(DIMS)
    truth = ev[(ev >= 0.4) & (ev <= 1.6)]
    assert all(len(s.windows) >= 2 for s in res.slices)
    for s in res.slices:
        wb = [w.lo for w in s.windows] + [s.windows[-1].hi]
        assert wb[0] == s.lo and wb[-1] == s.hi and all(np.diff(wb) > 0)
        assert max(w.est for w in s.windows) <= 12.0 + 1e-9
        assert sum(w.found for w in s.windows) >= s.eigenvalues.size
        assert all(s.error is None for s in res.slices)
    got = res.eigenvalues
    assert got.size == truth.size
    assert np.max(np.abs(np.sort(got) - truth)) <= 1e-10 * np.max(truth)


def test_window_sizing():
    from paper_1802_05215_b200.pipeline import concurrent_jobs, window_estimate
    # cfg2 (n = 64^3) on a 180 GB GPU: no split (the reference's 1,250 cap), all 8 slices at once
    assert window_estimate(262144, 180e9, 8) > 730  # largest cfg2 DOS estimate: 729.1
    assert concurrent_jobs(262144, 180e9, 8, 0) == 8
    # cfg5 (n = 128^3): one slice per GPU gets ~950-pair windows; 8 concurrent would not fit
    w = window_estimate(2097152, 180e9, 1)
    assert 900 < w < 1000
    assert concurrent_jobs(2097152, 180e9, 8, 0) == 2
    assert window_estimate(2097152, 180e9, 1, cap=500.0) == 500.0
