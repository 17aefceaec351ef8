// sliceeig_b200: the command-line caller of the polynomial-filtering path,
// built on the C++ drop-in facade (include/sliceeig/*.hpp) and therefore on libsliceeig_cuda.so.
// Subcommands, options, report layout and exit status follow the reference front end
// (tools/sliceeig_main.cpp:42-107 manifest/options, :200-377 gen/bounds/dos/slice/filter-dump,
// :382-619 solve): reports are JSON on stdout (or CSV with --format csv) plus files under --out
// (dos_curve.csv, slices.json, filter_curve.csv, slice_<i>.json, report.json, vectors_<i>.bin).
// Exit status is 0 only when every requested slice converged.
//
// In scope: polynomial filters with the nr / tr / si drivers, KPM or Lanczos densities, standard
// problems and generalized pencils (--bmatrix: a sparse SPD B, solved on the device as
// S = P A P with P ~ B^-1/2).  Rational filters are reported as errors (nonzero exit), as the
// reference does for invalid combinations.  B200 extension: --gpus N spreads the slice pool over
// N GPUs of the node (worker thread w on GPU w mod N) and splits the KPM probes over them with one
// NCCL all-reduce of the moments (kpm_dos_devices).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <map>
#include <optional>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "json_out.hpp"
#include "sliceeig/matrix_market.hpp"
#include "sliceeig/sliceeig_b200.hpp"

using namespace sliceeig;
using sejson::Json;
namespace fs = std::filesystem;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

double since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// ---- options -------------------------------------------------------------------------------
struct Manifest {
  std::string matrix_path, bmatrix_path;
  std::vector<int> dims;
  std::vector<double> interval;
  int slices = 1;
  std::string filter = "poly", damping = "sigma", solver = "nr", method = "kpm";
  int poles = 1, repeats = 2;
  double tol = 1e-8;
  unsigned long seed = 1234;
  int jobs = 1, gpus = 1;
  std::string out_dir = ".", format = "json";
  bool write_vectors = false;
  int dos_deg = 60, dos_vecs = 40, dos_npts = 300;

  Json input_json() const {
    Json j = Json::object();
    if (!dims.empty())
      j["dims"] = Json(dims);
    else
      j["matrix"] = matrix_path;
    if (!bmatrix_path.empty()) j["bmatrix"] = bmatrix_path;
    return j;
  }
  void require_interval() const {
    if (interval.size() != 2 || !(interval[0] < interval[1]))
      throw UsageError("--interval: expected LO,HI with LO < HI");
  }
};

template <class T>
std::vector<T> split_list(const std::string& s, const std::string& opt) {
  std::vector<T> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ',')) {
    std::istringstream is(item);
    T v{};
    if (!(is >> v) || !(is >> std::ws).eof()) throw UsageError(opt + ": bad value '" + item + "'");
    out.push_back(v);
  }
  if (out.empty()) throw UsageError(opt + ": empty list");
  return out;
}
template <class T>
T scalar(const std::string& s, const std::string& opt) {
  auto v = split_list<T>(s, opt);
  if (v.size() != 1) throw UsageError(opt + ": expected one value");
  return v[0];
}
int positive(const std::string& s, const std::string& opt) {
  const int v = scalar<int>(s, opt);
  if (v < 1) throw UsageError(opt + ": must be positive");
  return v;
}
void member(const std::string& v, std::initializer_list<const char*> allowed, const std::string& opt) {
  for (const char* a : allowed)
    if (v == a) return;
  throw UsageError(opt + ": '" + v + "' is not one of the allowed values");
}

// per-subcommand option sets (tools/sliceeig_main.cpp:623-681)
const std::map<std::string, std::set<std::string>>& option_table() {
  static const std::set<std::string> input{"--matrix", "--dims", "--bmatrix"};
  static const std::set<std::string> dosf{"--method", "--deg", "--vecs", "--npts"};
  static const std::set<std::string> outf{"--out", "--format"};
  auto join = [](std::initializer_list<std::set<std::string>> parts, std::set<std::string> extra) {
    for (const auto& p : parts) extra.insert(p.begin(), p.end());
    return extra;
  };
  static const std::map<std::string, std::set<std::string>> t{
      {"gen", {"--dims", "--out"}},
      {"bounds", join({input}, {"--seed"})},
      {"dos", join({input, dosf, outf}, {"--interval", "--seed"})},
      {"slice", join({input, dosf, outf}, {"--interval", "--slices", "--seed"})},
      {"filter-dump", join({input, outf}, {"--interval", "--filter", "--damping", "--poles", "--repeats", "--seed"})},
      {"solve", join({input, dosf, outf}, {"--interval", "--slices", "--filter", "--damping", "--poles", "--repeats",
                                           "--solver", "--tol", "--seed", "--jobs", "--vectors", "--gpus"})}};
  return t;
}

Manifest parse(const std::string& cmd, const std::vector<std::string>& args) {
  const auto& tab = option_table();
  auto it = tab.find(cmd);
  if (it == tab.end()) throw UsageError("unknown subcommand '" + cmd + "'");
  Manifest m;
  for (std::size_t i = 0; i < args.size(); ++i) {
    std::string opt = args[i], val;
    const std::size_t eq = opt.find('=');
    if (eq != std::string::npos) {
      val = opt.substr(eq + 1);
      opt = opt.substr(0, eq);
    }
    if (!it->second.count(opt)) throw UsageError("unknown option '" + opt + "' for " + cmd);
    if (opt == "--vectors") {
      m.write_vectors = true;
      continue;
    }
    if (eq == std::string::npos) {
      if (i + 1 >= args.size()) throw UsageError(opt + ": missing value");
      val = args[++i];
    }
    if (opt == "--matrix") m.matrix_path = val;
    else if (opt == "--bmatrix") m.bmatrix_path = val;
    else if (opt == "--dims") m.dims = split_list<int>(val, opt);
    else if (opt == "--interval") m.interval = split_list<double>(val, opt);
    else if (opt == "--slices") m.slices = positive(val, opt);
    else if (opt == "--filter") { member(val, {"poly", "rat"}, opt); m.filter = val; }
    else if (opt == "--damping") { member(val, {"sigma", "jackson", "none"}, opt); m.damping = val; }
    else if (opt == "--poles") m.poles = positive(val, opt);
    else if (opt == "--repeats") m.repeats = positive(val, opt);
    else if (opt == "--solver") { member(val, {"nr", "tr", "si"}, opt); m.solver = val; }
    else if (opt == "--method") { member(val, {"kpm", "lanczos"}, opt); m.method = val; }
    else if (opt == "--tol") {
      m.tol = scalar<double>(val, opt);
      if (!(m.tol > 0)) throw UsageError("--tol: must be positive");
    }
    else if (opt == "--seed") m.seed = scalar<unsigned long>(val, opt);
    else if (opt == "--jobs") m.jobs = positive(val, opt);
    else if (opt == "--gpus") m.gpus = positive(val, opt);
    else if (opt == "--out") m.out_dir = val;
    else if (opt == "--format") { member(val, {"json", "csv"}, opt); m.format = val; }
    else if (opt == "--deg") m.dos_deg = scalar<int>(val, opt);
    else if (opt == "--vecs") m.dos_vecs = scalar<int>(val, opt);
    else if (opt == "--npts") m.dos_npts = scalar<int>(val, opt);
  }
  if (cmd == "gen" && m.dims.empty()) throw UsageError("--dims: gen requires grid dimensions");
  if ((cmd == "slice" || cmd == "filter-dump" || cmd == "solve") && m.interval.empty())
    throw UsageError("--interval is required");
  return m;
}

// ---- shared pipeline stages (sliceeig_main.cpp:112-195) ---------------------------------------
// The problem of a run: A, and B for a generalized pencil (--bmatrix, sliceeig_main.cpp:112-125).
struct Problem {
  CsrMatrix a;
  std::optional<CsrMatrix> b;
  const CsrMatrix* bp() const { return b ? &*b : nullptr; }
};

Problem load_problem(const Manifest& m) {
  if (m.matrix_path.empty() == m.dims.empty())
    throw UsageError("input: exactly one of --matrix and --dims is required");
  Problem p;
  p.a = m.dims.empty() ? read_matrix_market(m.matrix_path) : gen_laplacian(m.dims);
  if (!m.bmatrix_path.empty()) {
    p.b = read_matrix_market(m.bmatrix_path);
    if (p.b->n() != p.a.n()) throw std::invalid_argument("A and B sizes differ");
  }
  return p;
}

// Bounds in the problem's inner product (sliceeig_main.cpp:128-136); for a pencil the device
// path uses B's CSR matrix instead of a Cholesky solve.
SpectralBounds estimate_bounds(const Problem& p, unsigned long seed) {
  const Operator opa = make_operator(p.a);
  if (!p.b) return lan_tr_bounds(opa, InnerProduct{}, 1e-4, 60, 40, seed);
  const Operator opb = make_operator(*p.b);
  InnerProduct ip;
  ip.b = &opb;
  return lan_tr_bounds(opa, ip, 1e-4, 60, 40, seed);
}

DosCurve estimate_dos(const Problem& p, const SpectralBounds& b, const Manifest& m) {
  DosConfig cfg;
  cfg.method = m.method == "kpm" ? DosMethod::Kpm : DosMethod::Lanczos;
  cfg.m = m.dos_deg;
  cfg.n_vec = m.dos_vecs;
  cfg.npts = m.dos_npts;
  cfg.seed = m.seed;
  const Operator op = make_operator(p.a);
  if (!p.b) return cfg.method == DosMethod::Kpm ? kpm_dos(op, b, cfg) : lan_dos(op, b, cfg);
  if (cfg.method == DosMethod::Kpm)
    throw std::invalid_argument("kpm density estimation handles standard problems only; "
                                "use --method lanczos for a pencil");
  const Operator opb = make_operator(*p.b);
  return dos_generalized(op, opb, opb, opb, b, cfg);
}

void write_text(const fs::path& path, const std::string& body) {
  std::ofstream os(path);
  if (!os) throw std::runtime_error("cannot write " + path.string());
  os << body;
  if (!os) throw std::runtime_error("write failed: " + path.string());
}

std::string curve_csv(const DosCurve& c) {
  std::ostringstream os;
  os.precision(17);
  os << "t,phi\n";
  for (std::size_t i = 0; i < c.xdos.size(); ++i) os << c.xdos[i] << "," << c.ydos[i] << "\n";
  return os.str();
}

fs::path out_dir(const Manifest& m) {
  fs::path d(m.out_dir);
  fs::create_directories(d);
  return d;
}

struct Overlap {
  double lo = 0, hi = 0;
  bool empty = true;
};
Overlap clip(const DosCurve& c, double lo, double hi) {  // density lives on [lmin, lmax] only
  Overlap o;
  o.lo = std::max(lo, c.xdos.front());
  o.hi = std::min(hi, c.xdos.back());
  o.empty = !(o.lo < o.hi);
  return o;
}

void emit(const Json& j) { std::cout << j.dump(2) << "\n"; }

Damping damping_of(const std::string& s) {
  return s == "sigma" ? Damping::LanczosSigma : s == "jackson" ? Damping::Jackson : Damping::None;
}

void require_poly(const Manifest& m) {
  if (m.filter != "poly")
    throw std::invalid_argument("rational filters (--filter rat) are outside the B200 build");
}

// ---- subcommands ----------------------------------------------------------------------------
int cmd_gen(const Manifest& m) {
  const CsrMatrix a = gen_laplacian(m.dims);
  std::string name = "laplacian_";
  for (std::size_t i = 0; i < m.dims.size(); ++i) name += (i ? "x" : "") + std::to_string(m.dims[i]);
  const fs::path path = out_dir(m) / (name + ".mtx");
  write_matrix_market(a, path.string());
  Json r = Json::object();
  r["schema"] = 1;
  r["command"] = "gen";
  r["path"] = path.string();
  r["n"] = a.n();
  r["nnz"] = a.nnz();
  emit(r);
  return 0;
}

int cmd_bounds(const Manifest& m) {
  const Problem a = load_problem(m);
  const SpectralBounds b = estimate_bounds(a, m.seed);
  Json r = Json::object();
  r["schema"] = 1;
  r["command"] = "bounds";
  r["input"] = m.input_json();
  r["lmin"] = b.lmin;
  r["lmax"] = b.lmax;
  emit(r);
  return 0;
}

int cmd_dos(const Manifest& m) {
  const Problem a = load_problem(m);
  const SpectralBounds b = estimate_bounds(a, m.seed);
  const DosCurve curve = estimate_dos(a, b, m);
  double nev = curve.nev_est;
  if (!m.interval.empty()) {
    m.require_interval();
    const Overlap o = clip(curve, m.interval[0], m.interval[1]);
    nev = o.empty ? 0.0 : dos_count(curve, o.lo, o.hi);
  }
  const fs::path cp = out_dir(m) / "dos_curve.csv";
  write_text(cp, curve_csv(curve));
  Json r = Json::object();
  r["schema"] = 1;
  r["command"] = "dos";
  r["input"] = m.input_json();
  r["method"] = m.method;
  r["lmin"] = b.lmin;
  r["lmax"] = b.lmax;
  r["nev_est"] = nev;
  r["curve_file"] = cp.string();
  if (m.format == "csv")
    std::cout << curve_csv(curve);
  else
    emit(r);
  return 0;
}

// Breakpoints from the clipped interval, outer edges reset to the request (sliceeig_main.cpp:270-278)
SliceSet slice_clipped(const DosCurve& curve, double xi, double eta, int ns) {
  const Overlap o = clip(curve, xi, eta);
  if (o.empty) throw std::invalid_argument("requested interval does not meet the sampled spectrum");
  SliceSet s = slice_spectrum(curve, o.lo, o.hi, ns);
  s.breakpoints.front() = xi;
  s.breakpoints.back() = eta;
  return s;
}

int cmd_slice(const Manifest& m) {
  m.require_interval();
  const Problem a = load_problem(m);
  const SpectralBounds b = estimate_bounds(a, m.seed);
  const DosCurve curve = estimate_dos(a, b, m);
  const SliceSet s = slice_clipped(curve, m.interval[0], m.interval[1], m.slices);
  Json arr = Json::array();
  for (int i = 0; i < s.ns(); ++i) {
    Json e = Json::object();
    e["lo"] = s.breakpoints[i];
    e["hi"] = s.breakpoints[i + 1];
    e["est_count"] = s.est_counts[i];
    arr.push_back(e);
  }
  Json r = Json::object();
  r["schema"] = 1;
  r["command"] = "slice";
  r["input"] = m.input_json();
  r["method"] = m.method;
  r["interval"] = Json(m.interval);
  r["slices"] = arr;
  write_text(out_dir(m) / "slices.json", r.dump(2) + "\n");
  if (m.format == "csv") {
    std::ostringstream os;
    os.precision(17);
    os << "lo,hi,est_count\n";
    for (int i = 0; i < s.ns(); ++i) os << s.breakpoints[i] << "," << s.breakpoints[i + 1] << "," << s.est_counts[i] << "\n";
    std::cout << os.str();
  } else {
    emit(r);
  }
  return 0;
}

int cmd_filter_dump(const Manifest& m) {
  m.require_interval();
  require_poly(m);
  const Problem a = load_problem(m);
  const SpectralBounds b = estimate_bounds(a, m.seed);
  const double lo = m.interval[0], hi = m.interval[1];
  PolyOpts po;
  po.damping = damping_of(m.damping);
  const PolynomialFilter f = find_pol(lo, hi, b, po);
  constexpr int kPts = 1000;
  std::ostringstream os;
  os.precision(17);
  os << "t,rho\n";
  for (int i = 0; i < kPts; ++i) {
    const double x = b.lmin + (b.lmax - b.lmin) * i / (kPts - 1);
    os << x << "," << eval_pol(f, std::clamp(f.map.to_ref(x), -1.0, 1.0)) << "\n";
  }
  write_text(out_dir(m) / "filter_curve.csv", os.str());
  Json r = Json::object();
  r["schema"] = 1;
  r["command"] = "filter-dump";
  r["kind"] = m.filter;
  r["interval"] = Json(m.interval);
  r["lmin"] = b.lmin;
  r["lmax"] = b.lmax;
  r["degree"] = f.k;
  r["bar"] = f.bar;
  r["center"] = f.map.c + f.map.d * f.gamma;
  r["damping"] = m.damping;
  if (m.format == "csv")
    std::cout << os.str();
  else
    emit(r);
  return 0;
}

// ---- solve: the slice pool ---------------------------------------------------------------------
// One unit of work per DOS slice.  Workers are host threads pinned round-robin to the node's GPUs
// (one slice context per thread); slices are handed out largest estimate first so a GPU does not
// finish the run alone on the most expensive slice (reports stay in slice order).
struct SliceJob {
  int index = 0;
  double lo = 0, hi = 0, est = 0;
};
struct SliceRun {
  EigenResults res;
  std::string error;   // non-empty: the driver threw (the slice is reported as failed)
  int gpu = 0;
  double seconds = 0;
  bool converged() const { return error.empty() && !res.hit_max_its; }
};

// Which eigenvalues a slice reports.  Neighbouring windows overlap by the filter's slack, so a
// pair near an interior breakpoint b can come back from both sides; it is assigned to the slice
// whose window (b_i + delta, b_{i+1} + delta] contains it, the outermost windows open-ended
// (the reference's seam rule, sliceeig_main.cpp:420-442, with delta = 1e-10 (lmax - lmin)).
struct SeamOwner {
  int ns = 1;
  double delta = 0;
  bool owns(const SliceJob& j, double v) const {
    const bool above_lo = j.index == 0 || v > j.lo + delta;
    const bool below_hi = j.index + 1 == ns || v <= j.hi + delta;
    return above_lo && below_hi;
  }
};

// the columns `pick` of a result (eigenvalues, residuals and vectors together)
EigenResults select_pairs(const EigenResults& r, const std::vector<int>& pick) {
  EigenResults out;
  out.niter = r.niter;
  out.counters = r.counters;
  out.hit_max_its = r.hit_max_its;
  out.vectors = DenseMat(r.vectors.rows(), 0);
  out.eigenvalues.reserve(pick.size());
  out.residuals.reserve(pick.size());
  for (int c : pick) {
    out.eigenvalues.push_back(r.eigenvalues[c]);
    out.residuals.push_back(r.residuals[c]);
    out.vectors.push_col(r.vectors.col_vec(c));
  }
  return out;
}

using SliceDriver = EigenResults (*)(const Problem&, const PolynomialFilter&, const SliceJob&,
                                     const SolverConfig&);
SliceDriver driver_for(const std::string& solver) {
  if (solver == "tr")
    return [](const Problem& p, const PolynomialFilter& f, const SliceJob& j, const SolverConfig& c) {
      return cheb_lan_tr(p.a, p.bp(), f, j.lo, j.hi, c);
    };
  if (solver == "si")
    return [](const Problem& p, const PolynomialFilter& f, const SliceJob& j, const SolverConfig& c) {
      return cheb_si(p.a, p.bp(), f, j.lo, j.hi, c.est_count, c);
    };
  return [](const Problem& p, const PolynomialFilter& f, const SliceJob& j, const SolverConfig& c) {
    return cheb_lan_nr(p.a, p.bp(), f, j.lo, j.hi, c);
  };
}

class SlicePool {
 public:
  SlicePool(const Problem& a, const SpectralBounds& b, const Manifest& m, SeamOwner seams)
      : a_(a), bounds_(b), m_(m), seams_(seams), drive_(driver_for(m.solver)) {}

  std::vector<SliceRun> run(const std::vector<SliceJob>& jobs, int workers) {
    std::vector<SliceRun> runs(jobs.size());
    std::vector<int> order(jobs.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int x, int y) { return jobs[x].est > jobs[y].est; });
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> threads;
    for (int w = 0; w < workers; ++w)
      threads.emplace_back([&, w] {
        const int gpu = w % std::max(1, m_.gpus);
        if (m_.gpus > 1) set_thread_device(gpu);
        for (std::size_t q; (q = next.fetch_add(1)) < order.size();) {
          const SliceJob& job = jobs[order[q]];
          SliceRun& out = runs[order[q]];
          out.gpu = gpu;
          const auto t0 = std::chrono::steady_clock::now();
          try {
            out.res = solve_one(job);
          } catch (const std::exception& e) {
            out.error = e.what();
          }
          out.seconds = since(t0);
        }
      });
    for (auto& t : threads) t.join();
    return runs;
  }

 private:
  EigenResults solve_one(const SliceJob& job) const {
    SolverConfig cfg;
    cfg.res_tol = m_.tol;
    cfg.seed = m_.seed;
    cfg.est_count = std::max(1, (int)std::lround(std::ceil(job.est)));
    PolyOpts po;
    po.damping = damping_of(m_.damping);
    const PolynomialFilter f = find_pol(job.lo, job.hi, bounds_, po);
    EigenResults r = drive_(a_, f, job, cfg);
    std::vector<int> mine;
    for (int c = 0; c < (int)r.eigenvalues.size(); ++c)
      if (seams_.owns(job, r.eigenvalues[c])) mine.push_back(c);
    return mine.size() == r.eigenvalues.size() ? std::move(r) : select_pairs(r, mine);
  }

  const Problem& a_;
  const SpectralBounds& bounds_;
  const Manifest& m_;
  SeamOwner seams_;
  SliceDriver drive_;
};

// pool width: the request (at least one thread per GPU), capped by the slice count and by the
// SLICEEIG_THREADS environment variable of the reference front end
int pool_width(const Manifest& m, int nslices) {
  int want = std::max(m.jobs, m.gpus);
  if (const char* e = std::getenv("SLICEEIG_THREADS"))
    if (std::atoi(e) >= 1) want = std::min(want, std::atoi(e));
  return std::max(1, std::min(want, nslices));
}

// ---- solve: reports -------------------------------------------------------------------------
Json counters_json(const Counters& c) {
  Json j = Json::object();
  j["n_A_matvec"] = c.n_A_matvec;
  j["n_B_matvec"] = c.n_B_matvec;
  j["n_B_solve"] = c.n_B_solve;
  j["n_shift_solve"] = c.n_shift_solve;
  return j;
}
Json times_json(const Counters& c) {
  Json j = Json::object();
  j["t_mv"] = c.t_mv;
  j["t_orth"] = c.t_orth;
  j["t_sv"] = c.t_sv;
  j["t_total"] = c.t_total;
  return j;
}

// vectors_<i>.bin: the slice's eigenvectors as raw little-endian float64, column-major n x count,
// described by a sidecar object in slice_<i>.json
Json write_vector_block(const fs::path& dir, int slice, const DenseMat& v) {
  const std::string name = "vectors_" + std::to_string(slice) + ".bin";
  std::ofstream os(dir / name, std::ios::binary);
  os.write(reinterpret_cast<const char*>(v.data()),
           (std::streamsize)(sizeof(double) * (std::size_t)v.rows() * v.cols()));
  if (!os) throw std::runtime_error("cannot write " + (dir / name).string());
  Json d = Json::object();
  d["file"] = name;
  d["n"] = v.rows();
  d["count"] = v.cols();
  d["element"] = "float64";
  d["byte_order"] = "little-endian";
  d["layout"] = "column-major";
  return d;
}

Json slice_report(const SliceJob& job, const SliceRun& run, const fs::path& dir, bool vectors) {
  Json sj = Json::object();
  sj["schema"] = 1;
  sj["slice"] = job.index;
  sj["lo"] = job.lo;
  sj["hi"] = job.hi;
  sj["est_count"] = job.est;
  if (!run.error.empty()) {
    sj["error"] = run.error;
    sj["converged"] = false;
    return sj;
  }
  const EigenResults& r = run.res;
  sj["found"] = (long)r.eigenvalues.size();
  sj["eigenvalues"] = Json(r.eigenvalues);
  sj["residuals"] = Json(r.residuals);
  sj["niter"] = r.niter;
  sj["converged"] = !r.hit_max_its;
  sj["counters"] = counters_json(r.counters);
  sj["times"] = times_json(r.counters);
  if (vectors) sj["vectors"] = write_vector_block(dir, job.index, r.vectors);
  return sj;
}

Json solve_config_json(const Manifest& m, int workers) {
  Json cfg = Json::object();
  cfg["input"] = m.input_json();
  cfg["interval"] = Json(m.interval);
  cfg["slices"] = m.slices;
  cfg["filter"] = m.filter;
  cfg["damping"] = m.damping;
  cfg["poles"] = m.poles;
  cfg["repeats"] = m.repeats;
  cfg["solver"] = m.solver;
  cfg["method"] = m.method;
  cfg["tol"] = m.tol;
  cfg["seed"] = m.seed;
  cfg["jobs_requested"] = m.jobs;
  cfg["jobs"] = workers;
  cfg["gpus"] = m.gpus;
  return cfg;
}

std::string pairs_csv(const std::vector<SliceRun>& runs) {
  std::ostringstream os;
  os.precision(17);
  os << "slice,index,eigenvalue,residual\n";
  for (std::size_t i = 0; i < runs.size(); ++i) {
    if (!runs[i].error.empty()) continue;
    const EigenResults& r = runs[i].res;
    for (std::size_t k = 0; k < r.eigenvalues.size(); ++k)
      os << i << "," << k << "," << r.eigenvalues[k] << "," << r.residuals[k] << "\n";
  }
  return os.str();
}

// The density for solve: with --gpus N > 1 and KPM the probes are split over the GPUs and the
// moments combined by one NCCL all-reduce (bit-identical to the single-GPU curve).
DosCurve solve_dos(const Problem& a, const SpectralBounds& b, const Manifest& m) {
  if (m.gpus <= 1 || m.method != "kpm" || a.b) return estimate_dos(a, b, m);
  DosConfig cfg;
  cfg.m = m.dos_deg;
  cfg.n_vec = m.dos_vecs;
  cfg.npts = m.dos_npts;
  cfg.seed = m.seed;
  std::vector<int> devices(m.gpus);
  for (int g = 0; g < m.gpus; ++g) devices[g] = g;
  return kpm_dos_devices(a.a, b, cfg, devices);
}

int cmd_solve(const Manifest& m) {
  const auto t0 = std::chrono::steady_clock::now();
  m.require_interval();
  require_poly(m);
  const double xi = m.interval[0], eta = m.interval[1];
  const Problem a = load_problem(m);
  const double t_load = since(t0);
  auto tb = std::chrono::steady_clock::now();
  const SpectralBounds bounds = estimate_bounds(a, m.seed);
  const double t_bounds = since(tb);
  tb = std::chrono::steady_clock::now();
  const DosCurve curve = solve_dos(a, bounds, m);
  std::vector<SliceJob> jobs;
  if (m.slices > 1) {
    const SliceSet s = slice_clipped(curve, xi, eta, m.slices);
    for (int i = 0; i < s.ns(); ++i) jobs.push_back({i, s.breakpoints[i], s.breakpoints[i + 1], s.est_counts[i]});
  } else {
    const Overlap o = clip(curve, xi, eta);
    jobs.push_back({0, xi, eta, o.empty ? 0.0 : dos_count(curve, o.lo, o.hi)});
  }
  const double t_dos = since(tb);
  const fs::path dir = out_dir(m);
  write_text(dir / "dos_curve.csv", curve_csv(curve));

  const int ns = (int)jobs.size();
  const int workers = pool_width(m, ns);
  tb = std::chrono::steady_clock::now();
  SlicePool pool(a, bounds, m, SeamOwner{ns, 1e-10 * (bounds.lmax - bounds.lmin)});
  const std::vector<SliceRun> runs = pool.run(jobs, workers);
  const double t_solve = since(tb);

  Json slices = Json::array();
  Counters total;
  long found = 0, niter = 0;
  bool all_ok = true;
  for (int i = 0; i < ns; ++i) {
    const Json sj = slice_report(jobs[i], runs[i], dir, m.write_vectors);
    write_text(dir / ("slice_" + std::to_string(i) + ".json"), sj.dump(2) + "\n");
    slices.push_back(sj);
    all_ok = all_ok && runs[i].converged();
    if (runs[i].error.empty()) {
      found += (long)runs[i].res.eigenvalues.size();
      niter += runs[i].res.niter;
      total += runs[i].res.counters;
    }
  }
  Json rep = Json::object();
  rep["schema"] = 1;
  rep["command"] = "solve";
  rep["config"] = solve_config_json(m, workers);
  Json bj = Json::object();
  bj["lmin"] = bounds.lmin;
  bj["lmax"] = bounds.lmax;
  rep["bounds"] = bj;
  Json dj = Json::object();
  dj["method"] = m.method;
  dj["curve_file"] = (dir / "dos_curve.csv").string();
  rep["dos"] = dj;
  rep["slices"] = slices;
  Json tot = Json::object();
  tot["found"] = found;
  tot["niter"] = niter;
  tot["counters"] = counters_json(total);
  tot["times"] = times_json(total);
  rep["totals"] = tot;
  rep["converged"] = all_ok;
  Json tj = Json::object();
  tj["t_load"] = t_load;
  tj["t_bounds"] = t_bounds;
  tj["t_dos"] = t_dos;
  tj["t_solve"] = t_solve;
  tj["t_total"] = since(t0);
  rep["timings"] = tj;
  write_text(dir / "report.json", rep.dump(2) + "\n");
  if (m.format == "csv")
    std::cout << pairs_csv(runs);
  else
    emit(rep);
  return all_ok ? 0 : 1;
}

void usage(std::ostream& os) {
  os << "usage: sliceeig_b200 {gen|bounds|dos|slice|filter-dump|solve} [options]\n"
        "  input:  --dims d1[,d2[,d3]] | --matrix FILE.mtx\n"
        "  dos:    --method kpm|lanczos --deg M --vecs N --npts P\n"
        "  output: --out DIR --format json|csv\n"
        "  solve:  --interval LO,HI --slices S --damping sigma|jackson|none --solver nr|tr|si\n"
        "          --tol T --seed S --jobs J --gpus G --vectors\n";
}

}  // namespace

int main(int argc, char** argv) {
  // 32 hardware work queues for the slice contexts' streams (before CUDA initialises)
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
  if (argc < 2) {
    usage(std::cerr);
    return 2;
  }
  const std::string cmd = argv[1];
  if (cmd == "-h" || cmd == "--help") {
    usage(std::cout);
    return 0;
  }
  try {
    const Manifest m = parse(cmd, std::vector<std::string>(argv + 2, argv + argc));
    if (cmd == "gen") return cmd_gen(m);
    if (cmd == "bounds") return cmd_bounds(m);
    if (cmd == "dos") return cmd_dos(m);
    if (cmd == "slice") return cmd_slice(m);
    if (cmd == "filter-dump") return cmd_filter_dump(m);
    return cmd_solve(m);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    usage(std::cerr);
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
}
