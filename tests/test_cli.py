"""The command-line caller (tools/sliceeig_b200): the reference's CLI test
cases (test_cli.cpp: gen round trip, bounds, dos counts, slice balance, solve oracle set / seams /
pool / determinism / tr driver, eigenvector sidecar, filter-dump, error exits) restated against the
B200 binary, plus report parity with the reference's cmd_solve (golden cli.npz)."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1802_05215_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "tools", "sliceeig_b200")


def run(args, cwd=None):
    r = subprocess.run([CLI, *args.split()], capture_output=True, text=True, timeout=900, cwd=cwd)
    return r.returncode, r.stdout, r.stderr


def ok_json(args):
    rc, out, err = run(args)
    assert rc == 0, err[-2000:]
    return json.loads(out)


def union(rep):
    return np.sort(np.concatenate([np.asarray(s["eigenvalues"]) for s in rep["slices"] if "eigenvalues" in s]))


def strip_times(j):
    if isinstance(j, dict):
        return {k: strip_times(v) for k, v in j.items() if k not in ("times", "timings")}
    if isinstance(j, list):
        return [strip_times(v) for v in j]
    return j


@pytest.fixture(scope="module", autouse=True)
def _binary():
    if not os.path.exists(CLI):
        from paper_1802_05215_b200 import build
        build.build(verbose=False)
    assert os.path.exists(CLI)


# ---- host-only cases (no GPU) -------------------------------------------------------------------
def read_mtx(path):
    with open(path) as f:
        head = f.readline().split()
        assert head[:4] == ["%%MatrixMarket", "matrix", "coordinate", "real"]
        line = f.readline()
        while line.startswith("%"):
            line = f.readline()
        n, _, nnz = (int(x) for x in line.split())
        ent = [f.readline().split() for _ in range(nnz)]
    dense = np.zeros((n, n))
    for i, j, v in ent:
        dense[int(i) - 1, int(j) - 1] = float(v)
        dense[int(j) - 1, int(i) - 1] = float(v)
    return n, dense


def test_gen_writes_laplacian_that_reads_back(tmp_path):
    small = ok_json(f"gen --dims 2 --out {tmp_path}")
    assert small["schema"] == 1 and small["n"] == 2
    rep = ok_json(f"gen --dims 12,12 --out {tmp_path}")
    assert rep["n"] == 144 and rep["nnz"] == 672
    n, dense = read_mtx(rep["path"])
    ref = api.gen_laplacian([12, 12])
    want = np.zeros((144, 144))
    for i in range(144):
        for p in range(ref.row_ptr[i], ref.row_ptr[i + 1]):
            want[i, ref.col_idx[p]] = ref.vals[p]
    assert n == 144 and np.array_equal(dense, want)


@pytest.mark.parametrize("args,code", [
    ("bounds", 2),                                    # no input source
    ("bounds --dims 4 --matrix nosuch.mtx", 2),       # two input sources
    ("bounds --matrix nosuch.mtx", 1),                # missing file
    ("solve --dims 6,6 --interval 0.6,0.4 --out {d}", 2),  # malformed interval
    ("solve --dims 6,6 --out {d}", 2),                # interval required
    ("solve --dims 6,6 --interval 0.4,0.6 --solver xx --out {d}", 2),
    ("solve --dims 6,6 --interval 0.4,0.6 --filter rat --solver si --out {d}", 1),  # no rational si
    ("frobnicate --dims 4", 2),
    ("gen --dims 4 --bogus 1", 2),
])
def test_bad_invocations_fail(tmp_path, args, code):
    rc, _, err = run(args.format(d=tmp_path))
    assert rc == code and "error:" in err


# ---- device cases --------------------------------------------------------------------------------

@pytest.mark.gpu
def test_bounds_enclose_spectrum():
    rep = ok_json("bounds --dims 20,20")
    ev = api.laplacian_analytic_eigs([20, 20])
    spread = ev[-1] - ev[0]
    assert rep["lmin"] <= ev[0] + 1e-10 and rep["lmax"] >= ev[-1] - 1e-10
    assert rep["lmin"] >= ev[0] - 0.2 * spread and rep["lmax"] <= ev[-1] + 0.2 * spread


@pytest.mark.gpu
def test_dos_counts_track_analytic(tmp_path):
    whole = ok_json(f"dos --dims 60,60 --interval 0,8 --out {tmp_path}")
    assert abs(whole["nev_est"] - 3600) <= 0.10 * 3600
    assert (tmp_path / "dos_curve.csv").exists()
    ev = api.laplacian_analytic_eigs([20, 20])
    truth = api.count_in_interval(ev, 0.0, 2.0)
    for method in ("kpm", "lanczos"):
        rep = ok_json(f"dos --dims 20,20 --interval 0,2 --method {method} --out {tmp_path}")
        assert abs(rep["nev_est"] - truth) <= 0.15 * truth
    rc, out, _ = run(f"dos --dims 8,8 --format csv --out {tmp_path}")
    assert rc == 0 and out.startswith("t,phi\n")


@pytest.mark.gpu
def test_slice_single_and_balanced(tmp_path):
    one = ok_json(f"slice --dims 10,10 --interval 0.3,0.9 --slices 1 --out {tmp_path}")
    assert len(one["slices"]) == 1
    assert one["slices"][0]["lo"] == 0.3 and one["slices"][0]["hi"] == 0.9
    rep = ok_json(f"slice --dims 20,20 --interval 0,2 --slices 4 --out {tmp_path}")
    ev = api.laplacian_analytic_eigs([20, 20])
    counts, prev = [], 0.0
    for s in rep["slices"]:
        assert s["lo"] == prev
        prev = s["hi"]
        counts.append(np.count_nonzero((ev > s["lo"]) & (ev <= s["hi"])))
    assert prev == 2.0
    mean = np.mean(counts)
    assert all(abs(c - mean) <= 0.25 * mean for c in counts)
    assert json.loads((tmp_path / "slices.json").read_text()) == rep


@pytest.mark.gpu
def test_solve_oracle_set_seams_pool_determinism(tmp_path):
    ev = api.laplacian_analytic_eigs([30, 30])
    oracle = ev[(ev >= 0.4) & (ev <= 0.6)]
    assert oracle.size == 13
    base = "solve --dims 30,30 --interval 0.4,0.6"
    poly = ok_json(f"{base} --out {tmp_path}/p")
    assert poly["converged"] is True
    vp = union(poly)
    assert vp.size == 13 and np.all(np.abs(vp - oracle) <= 1e-8)
    assert all(r <= 1e-8 for s in poly["slices"] for r in s["residuals"])
    for extra in (" --slices 4", " --slices 4 --jobs 4"):
        sl = ok_json(f"{base}{extra} --out {tmp_path}/s")
        assert sl["totals"]["found"] == 13
        assert np.all(np.abs(union(sl) - oracle) <= 1e-8)
    again = ok_json(f"{base} --out {tmp_path}/p")
    assert strip_times(poly) == strip_times(again)
    tr = ok_json(f"{base} --solver tr --out {tmp_path}/tr")
    assert np.all(np.abs(union(tr) - oracle) <= 1e-8)
    si = ok_json(f"{base} --solver si --out {tmp_path}/si")
    vsi = union(si)
    assert vsi.size == 13 and np.all(np.abs(vsi - oracle) <= 1e-7)
    rep = json.loads((tmp_path / "p" / "report.json").read_text())
    assert strip_times(rep) == strip_times(again)
    for i in range(len(rep["slices"])):
        assert json.loads((tmp_path / "p" / f"slice_{i}.json").read_text())["slice"] == i


@pytest.mark.gpu
@pytest.mark.parametrize("solver", ["nr", "tr", "si"])
def test_solve_report_matches_reference_cmd_solve(tmp_path, golden, solver):
    """Same arguments through the reference's cmd_solve (golden cli.npz): identical breakpoints,
    per-slice counts, eigenvalues within 1e-10 relative, iteration counts and filter degrees."""
    g = golden("cli")
    rc, out, err = run(f"solve --dims 30,30 --interval 0.4,0.6 --slices 4 --jobs 4 --solver {solver} "
                       f"--out {tmp_path}")
    rep = json.loads(out)
    # exit status 0 iff every slice converged -- as the reference run did (si slice 1 runs out of
    # cycles there too, exit 1)
    ref_ok = [not int(g[f"{solver}_slice{i}_meta"][3]) for i in range(len(rep["slices"]))]
    assert [s["converged"] for s in rep["slices"]] == ref_ok
    assert rc == (0 if all(ref_ok) else 1), err[-2000:]
    assert np.allclose([rep["bounds"]["lmin"], rep["bounds"]["lmax"]], g[f"{solver}_bounds"], rtol=1e-10)
    bp = [s["lo"] for s in rep["slices"]] + [rep["slices"][-1]["hi"]]
    assert np.allclose(bp, g[f"{solver}_bp"], rtol=1e-12, atol=0)
    assert np.allclose([s["est_count"] for s in rep["slices"]], g[f"{solver}_est"], rtol=1e-9)
    for i, s in enumerate(rep["slices"]):
        ref = g[f"{solver}_slice{i}_vals"]
        vals = np.asarray(s["eigenvalues"])
        assert vals.size == ref.size
        assert np.all(np.abs(vals - ref) <= 1e-10 * np.abs(ref))
        if solver != "si":  # subspace-iteration cycle counts hinge on residuals at the tolerance
            assert s["niter"] == int(g[f"{solver}_slice{i}_meta"][0])


@pytest.mark.gpu
def test_vectors_sidecar_round_trip(tmp_path):
    rep = ok_json(f"solve --dims 10,10 --interval 0.5,0.7 --vectors --out {tmp_path}")
    s0 = rep["slices"][0]
    side = s0["vectors"]
    n, count = side["n"], side["count"]
    assert count == len(s0["eigenvalues"]) and side["layout"] == "column-major"
    raw = np.fromfile(tmp_path / side["file"], dtype="<f8")
    assert raw.size == n * count
    u = raw[:n]
    a = api.gen_laplacian([10, 10])
    lam, res = api.rayleigh_and_residual(a, None, u)
    assert abs(lam - s0["eigenvalues"][0]) <= 1e-10 and res <= 1e-8
    assert abs(np.linalg.norm(u) - 1.0) <= 1e-10


@pytest.mark.gpu
def test_filter_dump_curve(tmp_path):
    rep = ok_json(f"filter-dump --dims 10,10 --interval 0.4,0.6 --filter poly --out {tmp_path}")
    assert rep["degree"] > 0 and rep["bar"] > 0.0
    lines = (tmp_path / "filter_curve.csv").read_text().splitlines()
    assert lines[0] == "t,rho" and len(lines) == 1001


@pytest.mark.gpu
def test_solve_errors(tmp_path):
    assert run(f"solve --dims 6,6 --interval 50,60 --out {tmp_path}")[0] != 0  # outside spectrum
    assert run(f"solve --dims 6,6 --interval 0.4,0.6 --filter rat --out {tmp_path}")[0] != 0


def _write_mtx(path, rp, ci, v):
    """Symmetric MatrixMarket (lower triangle), as the reference's write_matrix_market."""
    n = len(rp) - 1
    ent = [(i + 1, int(ci[p]) + 1, float(v[p])) for i in range(n) for p in range(rp[i], rp[i + 1])
           if ci[p] <= i]
    with open(path, "w") as f:
        f.write(f"%%MatrixMarket matrix coordinate real symmetric\n{n} {n} {len(ent)}\n")
        for i, j, x in ent:
            f.write(f"{i} {j} {x:.17g}\n")


@pytest.mark.gpu
def test_solve_generalized_pencil(tmp_path, golden):
    """test_cli.cpp:226-241: `solve --matrix a.mtx --bmatrix b.mtx --method lanczos`, here with a
    non-diagonal SPD B (the linear-element mass matrix of tests/golden/pencil_general.npz): the
    pencil's closed-form eigenvalues in the interval, slices seam-trimmed, exit status 0; KPM
    refuses a pencil as the reference does."""
    g = golden("pencil_general")
    a = api.gen_laplacian([30, 30])
    _write_mtx(tmp_path / "a.mtx", a.row_ptr, a.col_idx, a.vals)
    _write_mtx(tmp_path / "b.mtx", g["brp"], g["bci"], g["bv"])
    rep = ok_json(f"solve --matrix {tmp_path}/a.mtx --bmatrix {tmp_path}/b.mtx --method lanczos "
                  f"--interval 2.0,3.0 --slices 2 --solver tr --out {tmp_path}")
    ev = g["analytic"]
    truth = ev[(ev >= 2.0) & (ev <= 3.0)]
    got = union(rep)
    assert got.size == truth.size and np.all(np.abs(got - truth) <= 1e-10 * truth)
    assert rep["converged"] is True
    rc, _, err = run(f"solve --matrix {tmp_path}/a.mtx --bmatrix {tmp_path}/b.mtx --method kpm "
                     f"--interval 2.0,3.0 --out {tmp_path}")
    assert rc == 1 and "pencil" in err
