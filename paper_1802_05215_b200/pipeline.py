"""Sliced-solve pipeline (the semantics of `sliceeig solve`, tools/sliceeig_main.cpp:464-619), one
process per GPU.

    bounds (lan_tr_bounds tol 1e-4, 60, 40, seed; :128-136)
 -> KPM density: probes split across ranks, per-probe moments all-gathered and summed in probe
    order (so the curve is identical for any GPU count), curve + slicing on the host (:138-157)
 -> slice_clipped (:270-278): outer breakpoints reset to the user's interval
 -> per slice: est_count = max(1, ceil(est)) (:396-399), find_pol, cheb_lan_nr/tr (:394-418),
    trim_to_slice with delta = 1e-10 (lmax - lmin) (:422-442, :497)

Slices are independent: slice i runs on rank i % world, and the slices of one rank run
concurrently, one host thread + CUDA stream each (the reference's std::thread pool,
:494-523).  The only data-path collective is the KPM all-gather of per-probe moments.

The compute backend is pluggable only so the multi-rank plumbing can be exercised on CPU with
the test oracle (tests/test_pipeline_dist.py); the product backend is `GpuBackend`.
"""
from __future__ import annotations

import dataclasses
import math
import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import api


@dataclass
class Plan:
    xi: float
    eta: float
    ns: int = 1
    solver: str = "nr"            # nr | tr | si
    damping: str = "sigma"        # sigma | jackson | none
    dos_m: int = 60
    dos_nvec: int = 40
    dos_npts: int = 300
    probes: str = "rademacher"    # rademacher | gaussian
    tol: float = 1e-8
    seed: int = 1234
    bounds: Optional[tuple] = None  # fixed (lmin, lmax) skips the bounds stage
    solver_m: int = 0              # SolverConfig.m override (0: reference default)
    solver_max_its: int = 0        # SolverConfig.max_its override (0: 40 est + 300); a smaller
                                   # budget ends a slice early with hit_max_its, as in the reference
    jobs: int = 0                  # concurrent slices per rank (0: all of the rank's slices)
    only: Optional[Sequence[int]] = None  # debug/profiling: solve only these slice indices
    want_vectors: bool = False
    # memory plan (SURVEY.md §7 hard part 4): a DOS slice whose estimate exceeds `window_est` is
    # solved as consecutive sub-windows of near-equal DOS mass on its GPU (0: automatic -- the
    # reference's m = 4 est must stay within dense_sym_eig's 5,000 guard, dense_eig.hpp:114-117,
    # and each window's device footprint within the GPU's memory)
    window_est: float = 0.0


@dataclass
class Window:
    """One sub-window of a DOS slice (memory plan)."""
    lo: float
    hi: float
    est: float
    degree: int = 0
    found: int = 0
    niter: int = 0
    seconds: float = 0.0
    hit_max_its: bool = False


@dataclass
class SliceOutcome:
    index: int
    lo: float
    hi: float
    est: float
    degree: int = 0
    eigenvalues: np.ndarray = field(default_factory=lambda: np.zeros(0))
    residuals: np.ndarray = field(default_factory=lambda: np.zeros(0))
    vectors: Optional[np.ndarray] = None
    niter: int = 0
    n_A_matvec: int = 0
    hit_max_its: bool = False
    seconds: float = 0.0
    t_start: float = 0.0  # relative to the start of the solve stage
    t_mv: float = 0.0
    t_orth: float = 0.0
    error: Optional[str] = None
    rank: int = 0
    windows: List[Window] = field(default_factory=list)
    orth_passes: int = 0
    orth_cols: int = 0
    orth_bytes: float = 0.0


@dataclass
class PipelineResult:
    lmin: float
    lmax: float
    breakpoints: np.ndarray
    est_counts: np.ndarray
    slices: List[SliceOutcome]
    t_bounds: float
    t_dos: float
    t_solve: float
    t_total: float
    kernel_launches: int = 0

    @property
    def eigenvalues(self) -> np.ndarray:
        vals = [s.eigenvalues for s in sorted(self.slices, key=lambda s: s.index)]
        return np.concatenate(vals) if vals else np.zeros(0)

    @property
    def n_found(self) -> int:
        return int(sum(s.eigenvalues.size for s in self.slices))


class Dist:
    """Rank/world + the two collectives the pipeline needs (torch.distributed when initialised)."""

    def __init__(self, rank: int = 0, world: int = 1, device=None):
        self.rank, self.world, self.device = rank, world, device

    @classmethod
    def from_torch(cls):
        import torch.distributed as td
        if td.is_available() and td.is_initialized():
            import torch
            dev = torch.device("cuda", torch.cuda.current_device()) if td.get_backend() == "nccl" else None
            return cls(td.get_rank(), td.get_world_size(), dev)
        return cls()

    def combine_probe_rows(self, local: np.ndarray, first: int, total: int) -> np.ndarray:
        """The full probe-major (total, width) moment array from every rank's rows
        [first, first + len(local)): ONE all-reduce (NCCL under the nccl backend) of an array that
        is zero outside each rank's rows.  Adding exact zeros is exact in any order, so the result
        is the per-probe matrix bit for bit (one allreduce of the moments)."""
        width = local.shape[1]
        full = np.zeros((total, width), np.float64)
        full[first:first + local.shape[0]] = local
        if self.world == 1:
            return full
        import torch
        import torch.distributed as td
        t = torch.from_numpy(full)
        if self.device is not None:
            t = t.to(self.device)
        td.all_reduce(t, op=td.ReduceOp.SUM)
        return t.cpu().numpy()

    def broadcast_f64(self, vals: np.ndarray) -> np.ndarray:
        if self.world == 1:
            return vals
        import torch
        import torch.distributed as td
        t = torch.from_numpy(np.ascontiguousarray(vals, np.float64).copy())
        if self.device is not None:
            t = t.to(self.device)
        td.broadcast(t, 0)
        return t.cpu().numpy()

    def gather_objects(self, obj):
        if self.world == 1:
            return [obj]
        import torch.distributed as td
        out = [None] * self.world
        td.all_gather_object(out, obj)
        return out


def probe_split(n_vec: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous probe range [first, first+count) of `rank` (probe order is preserved)."""
    base, rem = divmod(n_vec, world)
    first = rank * base + min(rank, rem)
    return first, base + (1 if rank < rem else 0)


def slice_owner(index: int, world: int) -> int:
    return index % world


def slice_cost(est: float, degree: int, n: int, nnz: int) -> float:
    """Modelled device bytes of one slice solve: ~3.7 est Lanczos steps (measured on cfg2), each
    k filter degrees (12 nnz + 40 n bytes) plus two CGS passes over ~m/2 = 2 est columns
    (32 n * 2 est bytes)."""
    steps = 3.7 * max(est, 1.0)
    return steps * (degree * (12.0 * nnz + 40.0 * n) + 64.0 * n * max(est, 1.0))


def assign_lpt(costs: Sequence[float], world: int) -> List[int]:
    """Longest-processing-time-first assignment of slices to ranks (ties -> lowest rank), so the
    makespan of uneven DOS slices is balanced when there are more slices than GPUs.  With one
    slice per rank or more ranks than slices this is the identity / round-robin."""
    if world <= 1:
        return [0] * len(costs)
    if len(costs) <= world:
        return [i % world for i in range(len(costs))]
    load = [0.0] * world
    owner = [0] * len(costs)
    for i in sorted(range(len(costs)), key=lambda q: (-costs[q], q)):
        r = min(range(world), key=lambda q: (load[q], q))
        owner[i] = r
        load[r] += costs[i]
    return owner


def trim_to_slice(vals, res, index: int, ns: int, lo: float, hi: float, delta: float):
    """sliceeig_main.cpp:422-442: an eigenvalue within delta of an interior breakpoint belongs to
    the slice below it.  Returns the kept positions."""
    keep = []
    for i, v in enumerate(vals):
        if index > 0 and v <= lo + delta:
            continue
        if index + 1 < ns and v > hi + delta:
            continue
        keep.append(i)
    return np.asarray(keep, dtype=np.int64)


def slice_clipped(curve: api.DosCurve, xi: float, eta: float, ns: int, slicer=None):
    """sliceeig_main.cpp:187-193 + 270-278."""
    lo, hi = max(xi, curve.xdos[0]), min(eta, curve.xdos[-1])
    if not lo < hi:
        raise ValueError("requested interval does not meet the sampled spectrum")
    s = (slicer or api.slice_spectrum)(curve, lo, hi, ns)
    bp = np.array(s.breakpoints, np.float64)
    bp[0], bp[-1] = xi, eta
    return bp, np.asarray(s.est_counts, np.float64)


# ---- memory plan -----------------------------------------------------------------------------------
# The reference sizes a slice solve as m = max(4 est, 80) basis columns (eigensolvers.hpp:144) and
# its projected eigensolve refuses m > 5,000 (dense_eig.hpp:114-117), so a slice estimated above
# 1,250 eigenpairs cannot run as one Lanczos window.  At BASELINE cfg4/cfg5 sizes (n ~ 2M, 5-13k
# pairs per DOS slice) one window would also need 80-170 GB.  A large slice is therefore solved
# as consecutive sub-windows of near-equal DOS mass, each an ordinary cheb_lan_* call whose result
# is seam-trimmed exactly like neighbouring slices (sliceeig_main.cpp:422-442), with eigenvectors
# copied to host memory as each window finishes, so device memory holds one window at a time.
REF_WINDOW_EST = 1250.0      # 4 est <= 5,000 (dense_eig.hpp:114-117)
MIN_WINDOW_EST = 100.0
WINDOW_BYTES_PER_PAIR_ROW = 72.0  # 8 B x (m = 4 est basis + est locked + 2 x m/2 candidates)


def window_estimate(n: int, mem_bytes: Optional[float], jobs: int, cap: float = 0.0) -> float:
    """Largest DOS estimate one window may hold: the reference's m-guard limit, and a device
    footprint of ~72 n est bytes (basis, locked set, Ritz candidates) within 80% of the GPU's
    memory shared by `jobs` concurrent slices."""
    if cap > 0.0:  # explicit (Plan.window_est)
        return cap
    est = REF_WINDOW_EST
    if mem_bytes:
        est = min(est, 0.8 * mem_bytes / (WINDOW_BYTES_PER_PAIR_ROW * n * max(jobs, 1)))
    return max(est, MIN_WINDOW_EST)


def capped_basis(n: int, mem_bytes: Optional[float], jobs: int, est: float) -> int:
    """For a slice too large for the reference's m = 4 est but whose locked set still fits:
    the basis width m (<= 5,000: "explicit m <= 5,000") that fits next to
    the locked set (~1.15 est columns), the thick-restart staging block (m / 2) and the
    chunked candidate buffers (8 GB), in 85% of the device memory per concurrent slice.
    0 when even that does not fit (the slice is then solved as DOS-mass windows): a slice
    solved in one window keeps the filter of the whole slice, while w windows need w times the
    filter degree (each window is w times narrower)."""
    if not mem_bytes:
        return 0
    col = 8.0 * n
    room = 0.85 * mem_bytes / max(jobs, 1) - col * 1.15 * est - 8e9
    m = int(min(5000, 4 * math.ceil(est), room / (1.5 * col)))
    return m if m >= max(MIN_BASIS, 0.4 * est) else 0


MIN_BASIS = 400


def concurrent_jobs(n: int, mem_bytes: Optional[float], nslices: int, requested: int) -> int:
    """Slices solved at once on one GPU: all of them unless their windows would shrink below
    ~4x MIN_WINDOW_EST (narrow windows need high filter degrees); then as many as fit."""
    if requested > 0:
        return requested
    if not mem_bytes or nslices <= 1:
        return max(1, nslices)
    fit = int(0.8 * mem_bytes // (WINDOW_BYTES_PER_PAIR_ROW * n * 4 * MIN_WINDOW_EST))
    return max(1, min(nslices, fit))


def window_breakpoints(curve: api.DosCurve, lo: float, hi: float, est: float,
                       max_est: float) -> np.ndarray:
    """Split [lo, hi] into ceil(est / max_est) windows of equal DOS mass (bisection on
    dos_count, dos.hpp:212-218; the DOS grid is too coarse for slice_spectrum inside one slice)."""
    nw = max(1, int(math.ceil(est / max_est))) if est > max_est else 1
    bp = [lo]
    if nw > 1:
        x0, x1 = float(curve.xdos[0]), float(curve.xdos[-1])
        clo, chi = max(lo, x0), min(hi, x1)
        total = api.dos_count(curve, clo, chi)
        for i in range(1, nw):
            target = total * i / nw
            a, b = max(bp[-1], clo), chi
            for _ in range(100):
                mid = 0.5 * (a + b)
                if api.dos_count(curve, clo, mid) < target:
                    a = mid
                else:
                    b = mid
            bp.append(b)
    bp.append(hi)
    return np.asarray(bp, np.float64)


class GpuBackend:
    """The product path: every stage runs through libsliceeig_cuda.so on this rank's GPU."""

    def __init__(self, device: int = 0, matrix=None, dims=None, ctx=None):
        self.device = device
        self.ctx = ctx or api.default_context(device)
        if dims is not None:
            self.A = api.DeviceCsr.laplacian(dims, self.ctx)
        elif isinstance(matrix, api.DeviceCsr):
            self.A = matrix
        else:
            self.A = api.DeviceCsr.upload(matrix, self.ctx)
        self.n = self.A.n
        self._thread_ctx = {}

    def _ctx(self):
        import threading
        tid = threading.get_ident()
        if tid not in self._thread_ctx:
            self._thread_ctx[tid] = api.Context(self.device)
        return self._thread_ctx[tid]

    def launches(self) -> int:
        return self.ctx.kernel_launches() + sum(c.kernel_launches() for c in self._thread_ctx.values())

    def resident(self) -> bool:
        """True when a filter application is one resident cooperative launch (resident.cu) whose
        tiles fill more than half of every SM's shared memory: such a launch owns the GPU while
        it runs, so this GPU's slices are solved one at a time.  Small matrices (cfg1, the 32^3
        proxy) leave room for several launches and keep their slices concurrent."""
        return api.resident_tile_smem(self.A) > 110 * 1024

    def memory(self) -> float:
        """Total device memory in bytes (sizes the memory plan's windows)."""
        return float(api.device_memory(self.device)[1])

    def bounds(self, seed: int):
        b = api.lan_tr_bounds(self.A, 1e-4, 60, 40, seed)
        return b.lmin, b.lmax

    def moments(self, lmin, lmax, m, n_vec, seed, probes, first, count):
        if count == 0:
            return np.zeros((0, m + 1))
        return api.kpm_moments_probes(self.A, api.SpectralBounds(lmin, lmax), m, n_vec, seed,
                                      probes, first, count)

    def curve(self, zeta, lmin, lmax, npts):
        return api.kpm_curve(zeta, self.n, api.SpectralBounds(lmin, lmax), npts)

    def solve_slice(self, plan: Plan, lmin, lmax, lo, hi, est, m: int = 0):
        ctx = self._ctx()
        A = api.DeviceCsr(self.A.handle, ctx)  # se_csr is shareable across contexts on a device
        try:
            f = api.find_pol(lo, hi, api.SpectralBounds(lmin, lmax), api.PolyOpts(damping=plan.damping))
            cfg = api.SolverConfig(m=m or plan.solver_m, max_its=plan.solver_max_its,
                                   res_tol=plan.tol, seed=plan.seed,
                                   est_count=max(1, int(math.ceil(est))))
            if plan.solver == "si":  # filtered subspace iteration (eigensolvers.hpp:760-940)
                r = api.cheb_si(A, None, f, lo, hi, cfg.est_count, cfg, want_vectors=plan.want_vectors)
            elif plan.solver in ("tr", "nr"):
                drv = api.cheb_lan_tr if plan.solver == "tr" else api.cheb_lan_nr
                r = drv(A, None, f, lo, hi, cfg, want_vectors=plan.want_vectors)
            else:
                raise ValueError(f"unknown solver {plan.solver!r} (nr | tr | si)")
        finally:
            A.handle = None  # borrowed handle: do not free
        return f.k, r


def run(plan: Plan, backend, dist: Optional[Dist] = None, sink=None) -> PipelineResult:
    """Full sliced solve; every rank returns the gathered result (slices in index order).

    sink(slice_index, window_index, window, eigenvalues, residuals, vectors): optional consumer
    called on the owning rank as each solve window finishes (seam-trimmed; vectors (n, k) on the
    host when plan.want_vectors, else None -- or, with api.SAMPLE_VECTORS set, the pair
    (positions, (n, s) sample vectors) for spot checks of a result too large to download).  With a sink the eigenvectors are streamed to it -- e.g. written
    out like the CLI's vectors_<i>.bin -- instead of being accumulated, so neither device nor host
    memory has to hold a whole large slice.  A sink returning True stops that slice after the
    current window (a bounded partial solve)."""
    dist = dist or Dist()
    t0 = time.perf_counter()
    # bounds: deterministic on every rank; rank 0's copy is broadcast so all ranks agree bitwise
    if plan.bounds is not None:
        lmin, lmax = plan.bounds
    else:
        lmin, lmax = backend.bounds(plan.seed)
        lmin, lmax = (float(v) for v in dist.broadcast_f64(np.array([lmin, lmax])))
    t1 = time.perf_counter()
    # KPM: this rank's contiguous probe range, then one all-reduce of the per-probe moments
    first, count = probe_split(plan.dos_nvec, dist.world, dist.rank)
    mine = backend.moments(lmin, lmax, plan.dos_m, plan.dos_nvec, plan.seed, plan.probes, first,
                           count)
    allp = dist.combine_probe_rows(np.asarray(mine, np.float64).reshape(count, plan.dos_m + 1),
                                   first, plan.dos_nvec)
    zeta = np.zeros(plan.dos_m + 1)
    for row in allp:  # probe order (dos.hpp:100-106)
        zeta += row
    zeta /= float(plan.dos_nvec) * backend.n  # dos.hpp:110
    curve = backend.curve(zeta, lmin, lmax, plan.dos_npts)
    if plan.ns <= 1:
        lo, hi = max(plan.xi, curve.xdos[0]), min(plan.eta, curve.xdos[-1])
        est0 = api.dos_count(curve, lo, hi) if lo < hi else 0.0
        bp, est = np.array([plan.xi, plan.eta]), np.array([est0])
    else:
        bp, est = slice_clipped(curve, plan.xi, plan.eta, plan.ns)
    t2 = time.perf_counter()
    ns = len(est)
    delta = 1e-10 * (lmax - lmin)
    # LPT over modelled slice costs (degrees are cheap host computations, identical on every rank)
    degs = [api.find_pol(bp[i], bp[i + 1], api.SpectralBounds(lmin, lmax),
                         api.PolyOpts(damping=plan.damping)).k for i in range(ns)]
    nnz = getattr(getattr(backend, "A", None), "nnz", 7 * backend.n)
    owners = assign_lpt([slice_cost(est[i], degs[i], backend.n, nnz) for i in range(ns)], dist.world)
    mine_idx = [i for i in range(ns) if owners[i] == dist.rank
                and (plan.only is None or i in plan.only)]

    mem = backend.memory() if hasattr(backend, "memory") else None
    jobs = concurrent_jobs(backend.n, mem, len(mine_idx), plan.jobs)
    if plan.jobs <= 0 and plan.solver in ("tr", "nr") and getattr(backend, "resident", lambda: False)():
        jobs = 1  # the resident filter owns the whole GPU while it runs; concurrency buys nothing
    max_west = window_estimate(backend.n, mem, min(jobs, max(1, len(mine_idx))), plan.window_est)

    def work(i):
        out = SliceOutcome(i, float(bp[i]), float(bp[i + 1]), float(est[i]), rank=dist.rank)
        ts = time.perf_counter()
        out.t_start = ts - t2
        try:
            m_cap = 0
            if out.est > max_west and plan.window_est <= 0:
                m_cap = capped_basis(backend.n, mem, jobs, out.est)
            wbp = (np.array([out.lo, out.hi]) if m_cap else
                   window_breakpoints(curve, out.lo, out.hi, out.est, max_west))
            nw = len(wbp) - 1
            vals, ress, vecs = [], [], []
            for w in range(nw):
                tw = time.perf_counter()
                wlo, whi = float(wbp[w]), float(wbp[w + 1])
                west = out.est if nw == 1 else api.dos_count(
                    curve, max(wlo, curve.xdos[0]), min(whi, curve.xdos[-1]))
                k, r = backend.solve_slice(plan, lmin, lmax, wlo, whi, west,
                                           **({"m": m_cap} if m_cap else {}))
                # window seams follow the slice-seam rule (sliceeig_main.cpp:422-442)
                wk = trim_to_slice(r.eigenvalues, r.residuals, w, nw, wlo, whi, delta)
                vals.append(np.asarray(r.eigenvalues)[wk])
                ress.append(np.asarray(r.residuals)[wk])
                wv = None
                if plan.want_vectors and r.vectors is not None:
                    # seam trimming drops at most a few columns, usually none: no copy then
                    # (a fancy-indexed copy of a 1 GB block costs more than its D2H)
                    wv = np.asarray(r.vectors)
                    if wk.size != wv.shape[1]:
                        wv = wv[:, wk]
                if wv is not None and sink is None:
                    vecs.append(wv)
                out.degree = max(out.degree, k)
                out.niter += r.niter
                out.n_A_matvec += r.counters.n_A_matvec
                out.hit_max_its = out.hit_max_its or r.hit_max_its
                out.t_mv += r.counters.t_mv
                out.t_orth += r.counters.t_orth
                orth = getattr(r, "orth", None)
                if orth is not None:
                    out.orth_passes += orth.passes
                    out.orth_cols += orth.cols
                    out.orth_bytes += orth.bytes
                out.windows.append(Window(wlo, whi, float(west), k, int(wk.size), r.niter,
                                          time.perf_counter() - tw, r.hit_max_its))
                if wv is None and getattr(r, "sample_vectors", None) is not None:
                    # want_vectors=False with api.SAMPLE_VECTORS: the spot-check sample, as
                    # (positions into this window's kept eigenvalues, (n, s) vectors)
                    pos = {int(j): q for q, j in enumerate(wk)}
                    sel = [q for q, j in enumerate(r.sample_index) if int(j) in pos]
                    wv = (np.array([pos[int(r.sample_index[q])] for q in sel], np.int64),
                          r.sample_vectors[:, sel])
                del r
                stop = sink is not None and sink(i, w, out.windows[-1], vals[-1], ress[-1], wv)
                del wv
                if stop:  # the sink asked for no more windows of this slice (partial solve)
                    break
            allv = np.concatenate(vals) if vals else np.zeros(0)
            keep = trim_to_slice(allv, None, i, ns, out.lo, out.hi, delta)
            out.eigenvalues = allv[keep]
            out.residuals = np.concatenate(ress)[keep] if ress else np.zeros(0)
            if vecs:
                allvec = vecs[0] if len(vecs) == 1 else np.concatenate(vecs, axis=1)
                out.vectors = allvec if keep.size == allvec.shape[1] else allvec[:, keep]
        except Exception as e:  # per-slice failure is recorded (sliceeig_main.cpp:506-514)
            out.error = f"{type(e).__name__}: {e}"
        out.seconds = time.perf_counter() - ts
        return out

    if jobs == 1 or len(mine_idx) <= 1:
        local = [work(i) for i in mine_idx]
    else:
        with ThreadPoolExecutor(max_workers=jobs) as ex:
            local = list(ex.map(work, mine_idx))
    t3 = time.perf_counter()
    # only metadata crosses ranks (values, residuals, counters): eigenvectors stay with the rank
    # that owns the slice, so a multi-GPU run never ships vector blocks
    meta = [dataclasses.replace(s, vectors=None) for s in local]
    gathered = dist.gather_objects(meta)
    own = {s.index: s for s in local}
    slices = sorted([own.get(s.index, s) if s.rank == dist.rank else s
                     for part in gathered for s in part], key=lambda s: s.index)
    t4 = time.perf_counter()
    return PipelineResult(lmin, lmax, bp, est, slices, t1 - t0, t2 - t1, t3 - t2, t4 - t0,
                          backend.launches() if hasattr(backend, "launches") else 0)
