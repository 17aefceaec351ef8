#!/usr/bin/env python
"""bench.py -- eigenpairs/s of the full sliced solve (BASELINE.json metric) on B200.

Workload (BASELINE.json configs[1], "cfg2"): 3-D 7-point Laplacian 64^3 (n = 262,144, fp64 CSR),
KPM DOS with 100 moments and 40 seeded Gaussian probes, [0.6, 1.2] sliced into 8 by the DOS,
every slice solved with ChebLanTr (thick-restart filtered Lanczos, sigma damping), tol 1e-8.
One step = one full pipeline pass: bounds -> KPM -> slicing -> 8 filtered-Lanczos slice solves.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  (N > 1: launched by torch.distributed.run, one rank per GPU; slice i runs on rank i % N and the
   KPM probes are split across ranks with one all-gather of the per-probe moments.)

`value`  : eigenpairs/s with the matrix already resident in HBM (device generator) at t0.
`e2e`    : the same pipeline through the public API from a pinned HOST CSR: H2D of the matrix and
           D2H of all eigenpairs (values + vectors) inside the timed region.
`roofline`: the dominant kernel class on cfg2, the CGS2 step on the row-major basis (T1 + fused
           MID + N2, bytes 24 n k + 40 n), and beside it the fused Chebyshev-filter SpMV (bytes Abytes + 40 n per
           degree) on the workload matrix and on 160^3 (A > L2); all timed live with
           CUDA events on the launching stream, graph-captured as in production.
`cpu_baseline` / `--impl reference`: the unmodified reference (oracle/_ref, compiled from
           /root/reference headers) timed on this host's cores on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os

# before anything initialises CUDA (see paper_1802_05215_b200/__init__.py)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CFG2 = dict(dims=[64, 64, 64], xi=0.6, eta=1.2, ns=8, solver="tr", damping="sigma", dos_m=100,
            dos_nvec=40, probes="gaussian", tol=1e-8, seed=1234)
# CPU-boundable proxy of the same recipe (used only for the reference arm / cpu_baseline): the
# largest grid whose full reference pipeline stays near 20-30 s per step on 8 host threads (per-
# eigenpair cost grows ~n^2 with the grid: the 64^3 cfg2 itself takes ~2 h)
PROXY = dict(CFG2, dims=[32, 32, 32])
# side measurements (other BASELINE configs, reported under "other_configs")
CFGS_OTHER = {"cfg1": dict(dims=[100, 100], xi=0.4, eta=1.6, ns=2, solver="nr", damping="jackson",
                           dos_m=80, dos_nvec=20, probes="rademacher", tol=1e-8, seed=0)}
METRIC = "eigenpairs/sec for full sliced solve"
UNIT = "eigenpairs/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as td
        torch.cuda.set_device(local)
        td.init_process_group("nccl", device_id=torch.device("cuda", local))
    return rank, world, local


def _barrier(world):
    if world > 1:
        import torch.distributed as td
        td.barrier()


def _max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as td
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    td.all_reduce(t, op=td.ReduceOp.MAX)
    return float(t.item())


def _sum_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as td
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    td.all_reduce(t)
    return float(t.item())


def _plan(cfg, **kw):
    from paper_1802_05215_b200.pipeline import Plan
    keys = ("xi", "eta", "ns", "solver", "damping", "dos_m", "dos_nvec", "probes", "tol", "seed")
    return Plan(**{k: cfg[k] for k in keys}, **kw)


def kernel_rooflines(local_gpu: int, dims, cfg2_mean_cols: int):
    """Live CUDA-event timings (graph-captured, as in production) of the two kernel classes of the
    path: the reorthogonalisation pass (k_gemvt + k_gemvn, dominant on cfg2; bytes 16 n k + 24 n)
    and the fused Chebyshev-filter SpMV (bytes Abytes + 40 n per degree)."""
    import ctypes as C
    from paper_1802_05215_b200 import _lib, api
    peak, peak_kind = _peaks()
    ctx = api.Context(local_gpu)
    out = {}
    # the CGS2 step on the workload's basis shape (n = 64^3, k = mean active columns), re-pass
    # forced as in TR: row-major basis, T1 + fused MID + N2 = three reads of W (rowgs.cu)
    n = int(np.prod(dims))
    ms = C.c_double()
    reps = 20
    _lib.call("se_cgs2_bench", ctx.handle, n, cfg2_mean_cols, reps, 2, C.byref(ms))
    per = ms.value / reps * 1e-3
    by = 24.0 * n * cfg2_mean_cols + 40.0 * n
    out["cgs"] = (by / per / 1e9, per, by)
    # the column-major two-pass step it replaced (four reads of W), same shape, for reference
    ms0 = C.c_double()
    _lib.call("se_cgs2_bench", ctx.handle, n, cfg2_mean_cols, reps, 0, C.byref(ms0))
    out["cgs_colmajor"] = ms0.value / reps * 1e-3
    # filter SpMV on the workload matrix (L2-resident) and on 160^3 (A = 359 MB > L2)
    for tag, dd in (("workload", dims), ("hbm", [160, 160, 160])):
        A = api.DeviceCsr.laplacian(dd, ctx)
        f = api.find_pol(1.1691525, 1.2, api.SpectralBounds(0.0, 12.0))
        s, keep = f._c()
        ms2, nl, byt = C.c_double(), C.c_long(), C.c_double()
        _lib.call("se_filter_bench", ctx.handle, A.handle, C.byref(s), 3, C.byref(ms2), C.byref(nl),
                  C.byref(byt))
        out[tag] = (byt.value / (ms2.value * 1e-3) / 1e9, ms2.value * 1e-3 / nl.value, byt.value / nl.value)
        if tag == "workload":
            out["workload_resident"] = api.resident_tiles(A) > 0
            # the same chain as one launch per degree (the resident filter switched off)
            api.set_resident_filter(0)
            try:
                _lib.call("se_filter_bench", ctx.handle, A.handle, C.byref(s), 3, C.byref(ms2),
                          C.byref(nl), C.byref(byt))
                out["workload_per_degree_us"] = ms2.value * 1e3 / nl.value
            finally:
                api.set_resident_filter(1)
        else:  # the 8-vector block filter (cheb_si / block apply_pol) on the same matrix
            msb = C.c_double()
            _lib.call("se_block_filter_bench", ctx.handle, A.handle, 60, 3, C.byref(msb))
            per_b = msb.value / (60 * 3) * 1e-3
            by_b = 12.0 * A.nnz + 4.0 * (A.n + 1) + 40.0 * A.n * 8
            out["block"] = (by_b / per_b / 1e9, per_b, by_b)
        A.free()
    # Rayleigh-Ritz contraction U = W Y on the workload's widest slice (fp64 tensor cores)
    gm, gn, gk = n, 720, 2880
    g_ms = api.mult_cols_bench(gm, gn, gk, a_rowmajor=True, reps=2, ctx=ctx)
    out["gemm"] = (2.0 * gm * gn * gk / (g_ms * 1e-3) / 1e12, g_ms, (gm, gn, gk))
    # KPM block-step (K3) on BASELINE cfg3's matrix (160^3, 16 Rademacher probes per block,
    # doubling recurrence: bytes Abytes + 24 n b per step)
    A = api.DeviceCsr.laplacian([160, 160, 160], ctx)
    b3 = api.SpectralBounds(0.0, 12.0)
    api.kpm_moments(A, b3, 8, 16, seed=0)  # warm
    _lib.call("se_ctx_filter_timing", ctx.handle, 1, None, None, None)
    api.kpm_moments(A, b3, 80, 16, seed=0)
    ms3, nl3, by3 = C.c_double(), C.c_long(), C.c_double()
    _lib.call("se_ctx_filter_timing", ctx.handle, 0, C.byref(ms3), C.byref(nl3), C.byref(by3))
    out["kpm"] = (by3.value / (ms3.value * 1e-3) / 1e9, ms3.value * 1e-3 / nl3.value, by3.value / nl3.value)
    A.free()
    ctx.close()
    g, per, by = out["cgs"]
    traffic = {}
    tpath = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r1_ncu_traffic.json")
    if os.path.exists(tpath):  # dram bytes per launch from the committed ncu --set full captures
        with open(tpath) as fh:
            traffic = json.load(fh)
    def _t(key):
        return traffic.get(key, {}).get("traffic_bytes")
    roof = {"bound": "hbm",
            "kernel": "CGS2 step on the row-major Krylov basis: k_rw_stream T1 + fused MID (N1, "
                      "||t1||, T2) + N2 with their finishing reductions (orth.hpp:63-80, rowgs.cu)",
            "achieved": round(g, 1), "peak": peak, "unit": "GB/s", "frac": round(g / peak, 4),
            "peak_kind": peak_kind,
            # ncu capture at k = 1,440 columns (traffic 1.001 x algorithmic), scaled to this shape
            "traffic": (round(_t("rw_cgs2_step_n262144") * by /
                              traffic["rw_cgs2_step_n262144"]["algorithmic_bytes"])
                        if _t("rw_cgs2_step_n262144") else None),
            "traffic_capture": traffic.get("rw_cgs2_step_n262144"),
            "shape": f"n={n}, k={cfg2_mean_cols} basis columns (mean over the cfg2 run), re-pass forced",
            "us_per_step": round(per * 1e6, 2), "bytes_per_step": by,
            "algorithmic_bytes": "24 n k + 40 n (three reads of W; t read by T1, read+written by MID and N2)",
            "column_major_4read_us": round(out["cgs_colmajor"] * 1e6, 2),
            "filter_spmv": {"kernel": "k_spmv_cheb<kNext> (fused filter degree)",
                            "hbm_160^3": {"achieved": round(out["hbm"][0], 1),
                                          "frac": round(out["hbm"][0] / peak, 4),
                                          "us_per_launch": round(out["hbm"][1] * 1e6, 2),
                                          "traffic": _t("spmv_cheb_160cubed")},
                            "workload_64^3_L2_resident": {
                                "kernel": ("k_cheb_resident: all degrees of one filter application "
                                           "in one cooperative launch, matrix tiles in shared memory"
                                           if out.get("workload_resident") else "k_spmv_cheb per degree"),
                                "achieved": round(out["workload"][0], 1),
                                "us_per_degree": round(out["workload"][1] * 1e6, 2),
                                "us_per_degree_one_launch_per_degree":
                                    round(out.get("workload_per_degree_us", 0.0), 2)}},
            "block_filter": {"kernel": "k_cheb_ell_block (8-vector filter degree, row-major block; "
                                       "filter_poly.hpp:256-277 per column)",
                             "shape": "160^3, 8 vectors", "achieved": round(out["block"][0], 1),
                             "frac": round(out["block"][0] / peak, 4),
                             "us_per_degree": round(out["block"][1] * 1e6, 2),
                             "bytes_per_degree": round(out["block"][2]),
                             "traffic": _t("cheb_ell_block_160cubed_v8")},
            "ritz_gemm": {"kernel": "k_ritz_gemm (DMMA m8n8k4 f64): U = W Y, eigensolvers.hpp:275-283",
                          "bound": "tensor (fp64)", "shape": list(out["gemm"][2]),
                          "achieved_tflops_fp64": round(out["gemm"][0], 1),
                          "ms": round(out["gemm"][1], 2),
                          "traffic": _t("ritz_gemm_262144x720x2880")},
            "kpm_block_step": {"kernel": "k_kpm_ell (16-probe block, padded rows, doubling; dos.hpp:96-110)",
                               "shape": "160^3 (BASELINE cfg3 matrix), b=16",
                               "achieved": round(out["kpm"][0], 1), "frac": round(out["kpm"][0] / peak, 4),
                               "us_per_step": round(out["kpm"][1] * 1e6, 2),
                               "bytes_per_step": round(out["kpm"][2]),
                               "traffic": _t("kpm_ell_160cubed_b16")}}
    return roof


def other_configs(local_gpu: int):
    """The other BASELINE configs that fit a short run, measured on the same GPU after the timed
    region (not part of the headline): cfg1 (2-D 100^2, full NR pipeline) and cfg3 (KPM only:
    160^3, 300 moments x 128 Rademacher probes in blocks of 16, bounds fixed to [0, 12])."""
    import time as _time
    import ctypes as C
    from paper_1802_05215_b200 import _lib, api
    from paper_1802_05215_b200.pipeline import GpuBackend, run
    out = {}
    c1 = CFGS_OTHER["cfg1"]
    be = GpuBackend(device=local_gpu, dims=c1["dims"])
    run(_plan(c1), be)  # warm
    t0 = _time.perf_counter()
    r = run(_plan(c1), be)
    el = _time.perf_counter() - t0
    out["cfg1"] = {"workload": "2-D 100x100 Laplacian, KPM 80x20 Rademacher, [0.4,1.6] in 2 slices, "
                               "ChebLanNr (Jackson) tol 1e-8",
                   "eigenpairs": int(r.n_found), "seconds": round(el, 3),
                   "eigenpairs_per_s": round(r.n_found / el, 1),
                   "counts": [int(s.eigenvalues.size) for s in r.slices]}
    # the reference arm's bounded sample (cfg2 recipe on the 32^3 proxy) on this GPU, so the
    # two arms can also be compared on one identical workload
    bp = GpuBackend(device=local_gpu, dims=PROXY["dims"])
    run(_plan(PROXY), bp)  # warm
    t0 = _time.perf_counter()
    r = run(_plan(PROXY), bp)
    el = _time.perf_counter() - t0
    out["cfg2_proxy"] = {"workload": f"cfg2 recipe on the {PROXY['dims'][0]}^3 proxy (the "
                                     f"reference arm's sample)",
                         "eigenpairs": int(r.n_found), "seconds": round(el, 3),
                         "eigenpairs_per_s": round(r.n_found / el, 1)}
    bp.A.free()
    ctx = api.Context(local_gpu)
    A = api.DeviceCsr.laplacian([160, 160, 160], ctx)
    b3 = api.SpectralBounds(0.0, 12.0)
    api.kpm_moments(A, b3, 8, 16, seed=0)  # warm
    _lib.call("se_ctx_filter_timing", ctx.handle, 1, None, None, None)
    t0 = _time.perf_counter()
    api.kpm_moments(A, b3, 300, 128, seed=0)
    el = _time.perf_counter() - t0
    ms, nl, by = C.c_double(), C.c_long(), C.c_double()
    _lib.call("se_ctx_filter_timing", ctx.handle, 0, C.byref(ms), C.byref(nl), C.byref(by))
    out["cfg3"] = {"workload": "KPM: 160^3 Laplacian, 300 moments x 128 Rademacher probes (8 blocks of 16)",
                   "wall_s": round(el, 3), "device_s": round(ms.value * 1e-3, 3),
                   "block_steps": int(nl.value),
                   "device_GBps_algorithmic": round(by.value / (ms.value * 1e-3) / 1e9, 1),
                   "probe_moments_per_s": round(128 * 301 / el, 1)}
    A.free()
    ctx.close()
    return out


def arm_config(cfg, n, world):
    """The workload an arm actually ran (grid, n) -- the reference arm's bounded sample is the
    cfg2 recipe on the 32^3 proxy and says so."""
    tag = "cfg2" if cfg["dims"] == CFG2["dims"] else "cfg2 recipe on the CPU-boundable proxy grid"
    return {"workload": f"{tag}: {cfg['dims'][0]}^3 7-pt Laplacian, KPM 100x40 Gaussian, "
                        f"[0.6,1.2] in 8 slices, ChebLanTr tol 1e-8",
            "dims": list(cfg["dims"]), "n": n, "slices": cfg["ns"],
            "parallelism": f"slices{world}",
            "l2": "working set (Krylov bases ~1-6 GB per slice) >> 126 MB L2; no flush"}


CACHED_CPU = os.path.join(ROOT, "profiles", "r2_cpu_reference_cfg2.json")


def cached_cpu_reference():
    """The full cfg2 reference run (oracle/_ref, 8 slice threads), timed once in the build
    container by scripts/cpu_reference_cfg2.py (~2 h: too long for a bench run)."""
    if not os.path.exists(CACHED_CPU):
        return None
    with open(CACHED_CPU) as f:
        c = json.load(f)
    return {"value": c["eigenpairs_per_s"], "unit": UNIT, "cores": c["machine"]["jobs"],
            "host_cores": c["machine"]["cores"], "kind": "reference-cached",
            "sample": f"the full cfg2 workload ({c['eigenpairs']} eigenpairs in {c['wall_s']} s, "
                      f"{c['machine']['jobs']} slice threads on {c['machine']['cpu']}), "
                      f"{os.path.relpath(CACHED_CPU, ROOT)}"}


def run_reference(args, rank, world):
    """--impl reference: the unmodified reference pipeline (oracle/_ref) on this host's cores."""
    if rank != 0:
        return
    from oracle import reflib
    cfg = PROXY
    cores = os.cpu_count() or 1
    rp, ci, v = reflib.laplacian(cfg["dims"])
    res = None
    for _ in range(args.warmup):
        reflib.solve(rp, ci, v, cfg["xi"], cfg["eta"], cfg["ns"], cfg["solver"], cfg["damping"],
                     cfg["dos_m"], cfg["dos_nvec"], 300, "normal", cfg["tol"], cfg["seed"],
                     jobs=min(cores, cfg["ns"]))
    t0 = time.perf_counter()
    found = 0
    for _ in range(args.steps):
        res = reflib.solve(rp, ci, v, cfg["xi"], cfg["eta"], cfg["ns"], cfg["solver"],
                           cfg["damping"], cfg["dos_m"], cfg["dos_nvec"], 300, "normal", cfg["tol"],
                           cfg["seed"], jobs=min(cores, cfg["ns"]))
        found += sum(len(s["eigenvalues"]) for s in res["slices"])
    el = time.perf_counter() - t0
    val = found / el
    sample = (f"reference `sliceeig solve` semantics (bounds, KPM 100x40 Gaussian, 8 slices, "
              f"ChebLanTr tol 1e-8, {min(cores, cfg['ns'])} slice threads) on the CPU-boundable "
              f"{cfg['dims'][0]}^3 proxy of cfg2 ({found // args.steps} eigenpairs/step); the full "
              f"64^3 cfg2 takes ~2 h on 8 CPU threads (SURVEY.md §6.2)")
    line = {"impl": "reference", "metric": METRIC, "value": round(val, 4), "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(arm_config(cfg, int(np.prod(cfg["dims"])), args.gpus),
                           same_config_as_gpu_arm=False,
                           sample=f"bounded sample: the cfg2 recipe on the {cfg['dims'][0]}^3 proxy; "
                                  f"the GPU arm reports the same proxy under other_configs.cfg2_proxy"),
            "cpu_baseline": {"value": round(val, 4), "unit": UNIT, "cores": min(cores, cfg["ns"]),
                             "host_cores": cores, "kind": "reference", "sample": sample,
                             "cached_same_config": cached_cpu_reference()},
            "e2e": {"value": round(val, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    from oracle import reflib
    if not reflib.available():
        return None
    cfg = PROXY
    cores = os.cpu_count() or 1
    rp, ci, v = reflib.laplacian(cfg["dims"])
    t0 = time.perf_counter()
    res = reflib.solve(rp, ci, v, cfg["xi"], cfg["eta"], cfg["ns"], cfg["solver"], cfg["damping"],
                       cfg["dos_m"], cfg["dos_nvec"], 300, "normal", cfg["tol"], cfg["seed"],
                       jobs=min(cores, cfg["ns"]))
    el = time.perf_counter() - t0
    found = sum(len(s["eigenvalues"]) for s in res["slices"])
    return {"value": round(found / el, 4), "unit": UNIT, "cores": min(cores, cfg["ns"]),
            "host_cores": cores, "kind": "reference",
            "sample": f"full reference pipeline of the cfg2 recipe on the {cfg['dims'][0]}^3 proxy "
                      f"({found} eigenpairs in {el:.1f} s, {min(cores, cfg['ns'])} slice threads)",
            "cached_same_config": cached_cpu_reference()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--proxy", action="store_true", help="run the GPU arm on the CPU proxy size")
    ap.add_argument("--jobs", type=int, default=0, help="concurrent slices per GPU (0: all)")
    ap.add_argument("--no-others", action="store_true", help="skip the cfg1 / cfg3 side measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        # the reference is CPU code: rank 0 runs it on the host cores, other ranks exit at once
        run_reference(args, int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")))
        return
    rank, world, local = _dist_init()
    import torch
    from paper_1802_05215_b200 import api
    from paper_1802_05215_b200.pipeline import Dist, GpuBackend, run
    torch.cuda.set_device(local)
    cfg = PROXY if args.proxy else CFG2
    dist = Dist.from_torch() if world > 1 else Dist()
    backend = GpuBackend(device=local, dims=cfg["dims"])
    plan = _plan(cfg, jobs=args.jobs)
    for _ in range(args.warmup):
        res = run(plan, backend, dist)
    # ---- timed region: matrix resident in HBM ------------------------------------------------
    clocks = ClockSampler(local)
    l0 = backend.launches()
    _barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    found = 0
    for _ in range(args.steps):
        res = run(plan, backend, dist)
        found += sum(s.eigenvalues.size for s in res.slices if s.rank == rank)
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    _barrier(world)
    clk = clocks.stop()
    ms = _max_over_ranks(e0.elapsed_time(e1), world)
    found_all = _sum_over_ranks(found, world)
    launches = int(_sum_over_ranks(backend.launches() - l0, world))
    value = found_all / (ms * 1e-3)
    per_slice = [{"slice": s.index, "lo": round(s.lo, 8), "hi": round(s.hi, 8), "est": round(s.est, 1),
                  "found": int(s.eigenvalues.size), "degree": s.degree, "niter": s.niter,
                  "seconds": round(s.seconds, 3), "rank": s.rank, "error": s.error}
                 for s in res.slices]
    # ---- end to end through the public API from host buffers ---------------------------------
    e2e = None
    if not args.no_e2e:
        host = api.gen_laplacian(cfg["dims"])
        pinned = {}
        for nm in ("row_ptr", "col_idx", "vals"):
            arr = getattr(host, nm)
            t = torch.from_numpy(arr).pin_memory()
            pinned[nm] = t.numpy()
        hcsr = api.CsrMatrix(host.n, pinned["row_ptr"], pinned["col_idx"], pinned["vals"])
        plan_v = _plan(cfg, want_vectors=True)
        h2d = hcsr.row_ptr.nbytes + hcsr.col_idx.nbytes + hcsr.vals.nbytes
        # one untimed end-to-end step first: the pinned result blocks (8.6 GB a step) come from
        # torch's caching host allocator, and their first cudaHostAlloc is not part of a step
        be = GpuBackend(device=local, matrix=hcsr)
        r2 = run(plan_v, be, dist)
        be.A.free()
        del r2
        _barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d2h = 0
        got = 0
        for _ in range(args.steps):
            be = GpuBackend(device=local, matrix=hcsr)  # H2D of the CSR
            r2 = run(plan_v, be, dist)
            mine = [s for s in r2.slices if s.rank == rank]
            got += sum(s.eigenvalues.size for s in mine)
            d2h += sum(s.eigenvalues.nbytes + s.residuals.nbytes +
                       (s.vectors.nbytes if s.vectors is not None else 0) for s in mine)
            be.A.free()
            del r2, mine  # the step's pinned result blocks go back to the host caching allocator
        torch.cuda.synchronize()
        el = _max_over_ranks(time.perf_counter() - t0, world)
        got_all = _sum_over_ranks(got, world)
        e2e = {"value": round(got_all / el, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": int(_sum_over_ranks(d2h, world) / args.steps)}
    # mean active basis width over the run's reorthogonalisation passes (device counters of the
    # last timed step, all slices), and the orthogonalisation's share of the step in situ
    passes = sum(s.orth_passes for s in res.slices)
    cols = sum(s.orth_cols for s in res.slices)
    obytes = sum(s.orth_bytes for s in res.slices)
    mean_cols = max(1, int(round(cols / max(passes, 1))))
    roof = kernel_rooflines(local, cfg["dims"], mean_cols) if rank == 0 else None
    if roof is not None:
        step_s = ms * 1e-3 / args.steps
        rate = obytes / step_s / 1e9
        roof["in_situ"] = {
            "what": "CGS2 bytes of one timed step (every streamed basis column, 8 n each, + vector "
                    "traffic; device counters of all slices) / that step's wall time: the rate the "
                    "dominant kernel class sustains inside the whole step (filter and Ritz "
                    "extraction included in the denominator)",
            "orth_bytes_per_step": obytes, "orth_passes": passes, "mean_cols": mean_cols,
            "step_s": round(step_s, 3), "achieved": round(rate, 1),
            "frac": round(rate / roof["peak"], 4)}
    others = other_configs(local) if rank == 0 and not args.no_others else None
    cpu = cpu_baseline_sample() if (rank == 0 and world == 1 and not args.no_cpu) else None
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (generated Laplacian, seeded Gaussian/normal probes)",
                "config": arm_config(cfg, backend.n, world),
                "eigenpairs_per_step": int(found_all / args.steps),
                "per_slice": per_slice, "t_bounds": round(res.t_bounds, 3),
                "t_dos": round(res.t_dos, 3), "t_solve": round(res.t_solve, 3),
                "e2e": e2e, "gpu_launches": launches, "roofline": roof, "clocks": clk,
                "cpu_baseline": cpu, "other_configs": others}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as td
        td.destroy_process_group()


if __name__ == "__main__":
    main()
