// ORACLE — TEST INFRASTRUCTURE ONLY. C entry points over skrylov_oracle.hpp so
// the pytest suite (tests/) and bench.py's CPU-baseline leg can drive the CPU
// restatement through ctypes (oracle/pyoracle.py). Never linked by the product.
#include "skrylov_oracle.hpp"
#include "skrylov_oracle_complex.hpp"

#include <chrono>
#include <cstring>
#include <memory>
#include <string>

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}

struct Csr {
  std::shared_ptr<const SparseMatrix> A;
};
struct Krylov {
  KrylovState st;
  Counters c;
};
}  // namespace

extern "C" {

typedef struct {
  int64_t m, t, k, s;
  double tol, safety_init;
  int32_t max_restarts, variant;
  uint64_t sketch_seed;
  double rank_tol, breakdown_tol;
} orc_config;

const char* orc_last_error() { return g_err.c_str(); }

// ---- rng
void orc_mt_stream(uint64_t seed, int64_t n, uint64_t* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void orc_gaussian_vector(int64_t n, uint64_t seed, double* out) {
  Vec v = gaussian_vector(n, seed);
  std::memcpy(out, v.data(), sizeof(double) * static_cast<size_t>(n));
}
void orc_gaussian_stream(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.gaussian();
}
void orc_uniform_stream(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.uniform();
}
int orc_uniform_below_stream(uint64_t seed, uint64_t bound, int64_t n, uint64_t* out) {
  return guard([&] {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform_below(bound);
  });
}
void orc_sign_stream(uint64_t seed, int64_t n, double* out) {
  Rng r(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = r.sign();
}
int orc_sample_without_replacement(int64_t n, int64_t k, uint64_t seed, int64_t* out) {
  return guard([&] {
    Rng r(seed);
    auto v = r.sample_without_replacement(n, k);
    std::memcpy(out, v.data(), sizeof(int64_t) * v.size());
  });
}

// ---- matrices
void* orc_csr_create(int64_t rows, int64_t cols, const int64_t* off, const int64_t* col, const double* val) {
  Csr* h = nullptr;
  const int rc = guard([&] {
    const int64_t nnz = rows >= 0 ? off[rows] : 0;
    std::vector<Index> o(off, off + rows + 1), c(col, col + std::max<int64_t>(nnz, 0));
    Vec v(val, val + std::max<int64_t>(nnz, 0));
    h = new Csr{std::make_shared<const SparseMatrix>(rows, cols, std::move(o), std::move(c), std::move(v))};
  });
  return rc == 0 ? h : nullptr;
}
void* orc_csr_from_triplets(int64_t rows, int64_t cols, int64_t n, const int64_t* r, const int64_t* c, const double* v) {
  Csr* h = nullptr;
  const int rc = guard([&] {
    std::vector<Triplet> t(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) t[static_cast<size_t>(i)] = {r[i], c[i], v[i]};
    h = new Csr{std::make_shared<const SparseMatrix>(SparseMatrix::from_triplets(rows, cols, std::move(t)))};
  });
  return rc == 0 ? h : nullptr;
}
void* orc_gen_convdiff(int64_t n, double alpha) {
  Csr* h = nullptr;
  guard([&] { h = new Csr{std::make_shared<const SparseMatrix>(gen_convdiff(n, alpha))}; });
  return h;
}
void* orc_gen_neumann(int64_t g, double shift) {
  Csr* h = nullptr;
  guard([&] { h = new Csr{std::make_shared<const SparseMatrix>(gen_neumann(g, shift))}; });
  return h;
}
void* orc_gen_convdiff2d(int64_t n, double bx, double by, double shift, const double* diag_rel) {
  Csr* h = nullptr;
  guard([&] {
    Vec rel;
    if (diag_rel) rel.assign(diag_rel, diag_rel + n * n);
    h = new Csr{std::make_shared<const SparseMatrix>(gen_convdiff2d(n, bx, by, shift, diag_rel ? &rel : nullptr))};
  });
  return h;
}
void* orc_gen_convdiff3d(int64_t n, double bx, double by, double bz) {
  Csr* h = nullptr;
  guard([&] { h = new Csr{std::make_shared<const SparseMatrix>(gen_convdiff3d(n, bx, by, bz))}; });
  return h;
}
int64_t orc_csr_rows(void* h) { return static_cast<Csr*>(h)->A->rows(); }
int64_t orc_csr_cols(void* h) { return static_cast<Csr*>(h)->A->cols(); }
int64_t orc_csr_nnz(void* h) { return static_cast<Csr*>(h)->A->nonzeros(); }
void orc_csr_export(void* h, int64_t* off, int64_t* col, double* val) {
  const auto& A = *static_cast<Csr*>(h)->A;
  std::memcpy(off, A.offsets().data(), sizeof(int64_t) * A.offsets().size());
  std::memcpy(col, A.columns().data(), sizeof(int64_t) * A.columns().size());
  std::memcpy(val, A.values().data(), sizeof(double) * A.values().size());
}
int orc_csr_apply(void* h, const double* x, int64_t xlen, double* y) {
  return guard([&] { static_cast<Csr*>(h)->A->apply(x, xlen, y); });
}
void orc_csr_free(void* h) { delete static_cast<Csr*>(h); }

// ---- sketches
void* orc_sketch_srdct(int64_t n, int64_t s, uint64_t seed, int backend) {
  SketchOperator* h = nullptr;
  guard([&] { h = new SketchOperator(SketchOperator::subsampled_dct(n, s, seed, static_cast<SketchBackend>(backend))); });
  return h;
}
void* orc_sketch_identity(int64_t n) {
  SketchOperator* h = nullptr;
  guard([&] { h = new SketchOperator(SketchOperator::identity(n)); });
  return h;
}
void* orc_sketch_sparse_sign(int64_t n, int64_t s, uint64_t seed, int64_t zeta) {
  SketchOperator* h = nullptr;
  guard([&] { h = new SketchOperator(SketchOperator::sparse_sign(n, s, seed, zeta)); });
  return h;
}
int orc_sketch_apply(void* h, const double* x, int64_t n, double* out) {
  return guard([&] { static_cast<SketchOperator*>(h)->apply(x, n, out); });
}
int64_t orc_sketch_dim(void* h) { return static_cast<SketchOperator*>(h)->sketch_dim(); }
int64_t orc_sketch_input_dim(void* h) { return static_cast<SketchOperator*>(h)->input_dim(); }
void orc_sketch_rows(void* h, int64_t* out) {
  const auto& r = static_cast<SketchOperator*>(h)->rows();
  std::memcpy(out, r.data(), sizeof(int64_t) * r.size());
}
void orc_sketch_signs(void* h, double* out) {
  const auto& s = static_cast<SketchOperator*>(h)->signs();
  std::memcpy(out, s.data(), sizeof(double) * s.size());
}
void orc_sketch_sparse_entries(void* h, int64_t j0, int64_t count, int64_t* rows, double* signs) {
  const auto* S = static_cast<SketchOperator*>(h);
  const Index z = S->zeta();
  for (int64_t j = 0; j < count; ++j)
    for (Index l = 0; l < z; ++l) {
      Index r;
      double sg;
      S->sparse_entry(j0 + j, l, &r, &sg);
      rows[j * z + l] = r;
      signs[j * z + l] = sg;
    }
}
void orc_sketch_free(void* h) { delete static_cast<SketchOperator*>(h); }

// ---- truncated Arnoldi (test_arnoldi restatement driver)
void* orc_krylov_run(void* csr, const double* r0, int64_t n, void* sketch, int64_t t, int64_t m, int64_t steps,
                     double breakdown_tol) {
  Krylov* h = nullptr;
  const int rc = guard([&] {
    auto k = std::make_unique<Krylov>();
    const auto& S = *static_cast<SketchOperator*>(sketch);
    OperatorRef op(*static_cast<Csr*>(csr)->A);
    k->st = init_krylov(Vec(r0, r0 + n), S, t, m, &k->c);
    for (int64_t q = 0; q < steps && !k->st.breakdown && k->st.j < m; ++q) arnoldi_step(k->st, op, S, &k->c, breakdown_tol);
    h = k.release();
  });
  return rc == 0 ? h : nullptr;
}
void orc_krylov_info(void* h, int64_t* j, int32_t* breakdown, double* r0_norm, int64_t* counters) {
  const auto* k = static_cast<Krylov*>(h);
  *j = k->st.j;
  *breakdown = k->st.breakdown ? 1 : 0;
  *r0_norm = k->st.r0_norm;
  counters[0] = k->c.matvecs;
  counters[1] = k->c.inner_products;
  counters[2] = k->c.sketch_applies;
}
/// which: 0 V (n x m+1), 1 H (m+1 x m), 2 SV (s x m+1), 3 SAV (s x m); column-major.
void orc_krylov_get(void* h, int which, double* out) {
  const auto* k = static_cast<Krylov*>(h);
  const Mat* M[4] = {&k->st.V, &k->st.H, &k->st.SV, &k->st.SAV};
  std::memcpy(out, M[which]->a.data(), sizeof(double) * M[which]->a.size());
}
void orc_krylov_free(void* h) { delete static_cast<Krylov*>(h); }

/// CPU baseline sample (bench.py): the per-step work of solve_cycle
/// (solver.hpp:165-179) with an empty recycle space — init_krylov, then per
/// step arnoldi_step + IncrementalQR::append + solve — timed on the steps
/// alone (steady clock). Returns the steps taken; seconds in *step_s and
/// *init_s.
int64_t orc_step_sample(void* csr, const double* r0, int64_t n, void* sketch, int64_t t, int64_t steps,
                        double* init_s, double* step_s) {
  int64_t done = -1;
  guard([&] {
    const auto& S = *static_cast<SketchOperator*>(sketch);
    OperatorRef op(*static_cast<Csr*>(csr)->A);
    Counters c;
    const auto t0 = std::chrono::steady_clock::now();
    KrylovState st = init_krylov(Vec(r0, r0 + n), S, t, steps, &c);
    const Index s = S.sketch_dim();
    Vec sr0(static_cast<size_t>(s));
    for (Index r = 0; r < s; ++r) sr0[static_cast<size_t>(r)] = st.SV(r, 0) * st.r0_norm;
    IncrementalQR qr(s, steps, 1e-12);
    const auto t1 = std::chrono::steady_clock::now();
    double sres = 0.0;
    while (st.j < steps && !st.breakdown) {
      arnoldi_step(st, op, S, &c, 1e-14);
      const auto info = qr.append(st.SAV.col(st.j - 1), s);
      if (info.rank_deficient) qr.exclude(info.column);
      sres += qr.solve(sr0).residual_norm;
    }
    const auto t2 = std::chrono::steady_clock::now();
    *init_s = std::chrono::duration<double>(t1 - t0).count();
    *step_s = std::chrono::duration<double>(t2 - t1).count();
    (void)sres;
    done = st.j;
  });
  return done;
}

// ---- harmonic extraction (test_recycle restatement driver)
int orc_harmonic(const double* SAW, const double* SW, int64_t s, int64_t p, int64_t k, double rank_tol,
                 int64_t* rank_out, int64_t* k_eff, int32_t* flags, double* coeffs /* p x (k+1) */,
                 double* mu_re, double* mu_im, double* sigma /* p */) {
  return guard([&] {
    Mat a(s, p), w(s, p);
    std::memcpy(a.a.data(), SAW, sizeof(double) * static_cast<size_t>(s * p));
    std::memcpy(w.a.data(), SW, sizeof(double) * static_cast<size_t>(s * p));
    HarmonicPencil pen = truncated_svd(a, rank_tol);
    fill_pencil(pen, w);
    HarmonicPairs hp = harmonic_pairs(pen, k);
    *rank_out = pen.rank();
    *k_eff = hp.k_effective;
    flags[0] = hp.pair_extended;
    flags[1] = hp.rank_limited;
    std::memcpy(coeffs, hp.coeffs.a.data(), sizeof(double) * hp.coeffs.a.size());
    for (size_t i = 0; i < hp.mu.size(); ++i) {
      mu_re[i] = hp.mu[i].real();
      mu_im[i] = hp.mu[i].imag();
    }
    for (size_t i = 0; i < pen.sigma.size(); ++i) sigma[i] = pen.sigma[i];
  });
}

// ---- recycle spaces
void* orc_space_create() { return new RecycleSpace(); }
void orc_space_free(void* h) { delete static_cast<RecycleSpace*>(h); }
int64_t orc_space_dim(void* h) { return static_cast<RecycleSpace*>(h)->dim(); }
int64_t orc_space_rows(void* h) { return static_cast<RecycleSpace*>(h)->U.rows; }
int64_t orc_space_srows(void* h) { return static_cast<RecycleSpace*>(h)->SU.rows; }
int orc_space_provenance(void* h) { return static_cast<int>(static_cast<RecycleSpace*>(h)->provenance); }
void orc_space_get(void* h, double* U, double* SU, double* SAU) {
  const auto* sp = static_cast<RecycleSpace*>(h);
  if (U) std::memcpy(U, sp->U.a.data(), sizeof(double) * sp->U.a.size());
  if (SU) std::memcpy(SU, sp->SU.a.data(), sizeof(double) * sp->SU.a.size());
  if (SAU) std::memcpy(SAU, sp->SAU.a.data(), sizeof(double) * sp->SAU.a.size());
}
void orc_space_set(void* h, int64_t n, int64_t s, int64_t k, const double* U, const double* SU, const double* SAU, int prov) {
  auto* sp = static_cast<RecycleSpace*>(h);
  sp->U = Mat(n, k);
  sp->SU = Mat(s, k);
  sp->SAU = Mat(s, k);
  std::memcpy(sp->U.a.data(), U, sizeof(double) * static_cast<size_t>(n * k));
  std::memcpy(sp->SU.a.data(), SU, sizeof(double) * static_cast<size_t>(s * k));
  std::memcpy(sp->SAU.a.data(), SAU, sizeof(double) * static_cast<size_t>(s * k));
  sp->provenance = static_cast<RecycleSpace::Provenance>(prov);
}

// ---- solves
static SolverConfig to_cfg(const orc_config* c) {
  SolverConfig cfg;
  cfg.m = c->m;
  cfg.t = c->t;
  cfg.k = c->k;
  cfg.s = c->s;
  cfg.tol = c->tol;
  cfg.safety_init = c->safety_init;
  cfg.max_restarts = c->max_restarts;
  cfg.variant = static_cast<SequenceVariant>(c->variant);
  cfg.sketch_seed = c->sketch_seed;
  cfg.rank_tol = c->rank_tol;
  cfg.breakdown_tol = c->breakdown_tol;
  return cfg;
}

void* orc_solve(void* csr, const double* b, int64_t n, const orc_config* c, void* space, void* sketch,
                const double* x0, double* x_out) {
  SolveReport* rep = nullptr;
  guard([&] {
    const SparseMatrix& A = *static_cast<Csr*>(csr)->A;
    OperatorRef op(A);
    Vec bb(b, b + n), xx0;
    if (x0) xx0.assign(x0, x0 + n);
    RecycleSpace sp = space ? *static_cast<RecycleSpace*>(space) : RecycleSpace{};
    SolveResult r = solve(op, bb, to_cfg(c), std::move(sp), static_cast<SketchOperator*>(sketch), x0 ? &xx0 : nullptr);
    std::memcpy(x_out, r.x.data(), sizeof(double) * r.x.size());
    if (space) *static_cast<RecycleSpace*>(space) = std::move(r.space);
    rep = new SolveReport(std::move(r.report));
  });
  return rep;
}

/// solve() on a callable operator (OperatorRef(rows, cols, Apply),
/// operator_ref.hpp:22-25): apply(x, y, user) on host vectors.
void* orc_solve_callable(int64_t rows, int64_t cols, int (*apply)(const double*, double*, void*), void* user,
                         const double* b, int64_t n, const orc_config* c, void* space, void* sketch, double* x_out) {
  SolveReport* rep = nullptr;
  guard([&] {
    OperatorRef op(rows, cols, [apply, user](const double* x, double* y) {
      if (apply(x, y, user) != 0) throw std::runtime_error("OperatorRef: apply callback failed");
    });
    Vec bb(b, b + n);
    RecycleSpace sp = space ? *static_cast<RecycleSpace*>(space) : RecycleSpace{};
    SolveResult r = solve(op, bb, to_cfg(c), std::move(sp), static_cast<SketchOperator*>(sketch), nullptr);
    std::memcpy(x_out, r.x.data(), sizeof(double) * r.x.size());
    if (space) *static_cast<RecycleSpace*>(space) = std::move(r.space);
    rep = new SolveReport(std::move(r.report));
  });
  return rep;
}

void* orc_baseline_gmres(void* csr, const double* b, int64_t n, int64_t m, double tol, int32_t max_restarts,
                         double breakdown_tol, const double* x0, double* x_out) {
  SolveReport* rep = nullptr;
  guard([&] {
    const SparseMatrix& A = *static_cast<Csr*>(csr)->A;
    OperatorRef op(A);
    Vec bb(b, b + n), xx0;
    if (x0) xx0.assign(x0, x0 + n);
    BaselineConfig cfg;
    cfg.m = m;
    cfg.tol = tol;
    cfg.max_restarts = max_restarts;
    cfg.breakdown_tol = breakdown_tol;
    SolveResult r = baseline_gmres(op, bb, cfg, x0 ? &xx0 : nullptr);
    std::memcpy(x_out, r.x.data(), sizeof(double) * r.x.size());
    rep = new SolveReport(std::move(r.report));
  });
  return rep;
}

int orc_solve_sequence(int32_t nprob, void** mats, const double** rhs, const double** x0s, const double* tols,
                       int32_t shared, const orc_config* c, void* sketch, void* space, double** x_outs,
                       void** reports_out) {
  return guard([&] {
    ProblemSequence seq;
    seq.shared_matrix = shared != 0;
    for (int32_t i = 0; i < nprob; ++i) {
      ProblemInstance p;
      if (mats[i]) {
        p.matrix = static_cast<Csr*>(mats[i])->A;
        const Index n = p.matrix->rows();
        p.rhs.assign(rhs[i], rhs[i] + n);
        if (x0s && x0s[i]) p.x0.assign(x0s[i], x0s[i] + n);
      }
      p.target_tol = tols ? tols[i] : 0.0;
      seq.problems.push_back(std::move(p));
    }
    RecycleSpace sp = space ? *static_cast<RecycleSpace*>(space) : RecycleSpace{};
    SequenceResult r = solve_sequence(seq, to_cfg(c), static_cast<SketchOperator*>(sketch), std::move(sp));
    for (int32_t i = 0; i < nprob; ++i) {
      if (x_outs && x_outs[i] && !r.solutions[static_cast<size_t>(i)].empty())
        std::memcpy(x_outs[i], r.solutions[static_cast<size_t>(i)].data(), sizeof(double) * r.solutions[static_cast<size_t>(i)].size());
      reports_out[i] = new SolveReport(std::move(r.reports[static_cast<size_t>(i)]));
    }
    if (space) *static_cast<RecycleSpace*>(space) = std::move(r.space);
  });
}

int orc_report_status(void* r) { return static_cast<int>(static_cast<SolveReport*>(r)->status); }
int64_t orc_report_iterations(void* r) { return static_cast<SolveReport*>(r)->iterations; }
int32_t orc_report_cycles(void* r) { return static_cast<SolveReport*>(r)->cycles; }
double orc_report_rhs_norm(void* r) { return static_cast<SolveReport*>(r)->rhs_norm; }
double orc_report_final_rel(void* r) { return static_cast<SolveReport*>(r)->final_relative_residual; }
double orc_report_seconds(void* r) { return static_cast<SolveReport*>(r)->seconds; }
void orc_report_counters(void* r, int64_t* c) {
  const auto& k = static_cast<SolveReport*>(r)->counters;
  c[0] = k.matvecs;
  c[1] = k.inner_products;
  c[2] = k.sketch_applies;
}
int64_t orc_report_n_samples(void* r, int which) {
  const auto* p = static_cast<SolveReport*>(r);
  return static_cast<int64_t>(which == 0 ? p->sketched_residuals.size() : p->true_residuals.size());
}
void orc_report_samples(void* r, int which, int64_t* it, double* val) {
  const auto* p = static_cast<SolveReport*>(r);
  const auto& v = which == 0 ? p->sketched_residuals : p->true_residuals;
  for (size_t i = 0; i < v.size(); ++i) {
    it[i] = v[i].iteration;
    val[i] = v[i].value;
  }
}
int64_t orc_report_n_cycle_stats(void* r) { return static_cast<int64_t>(static_cast<SolveReport*>(r)->cycle_stats.size()); }
/// out: steps, entry_residual, sketched_entry, exit_sres, exit_residual, safety_after, basis_cond, deflation_rank
void orc_report_cycle_stats(void* r, int64_t i, double* out) {
  const auto& c = static_cast<SolveReport*>(r)->cycle_stats[static_cast<size_t>(i)];
  out[0] = static_cast<double>(c.steps);
  out[1] = c.entry_residual;
  out[2] = c.sketched_entry;
  out[3] = c.exit_sres;
  out[4] = c.exit_residual;
  out[5] = c.safety_after;
  out[6] = c.basis_cond;
  out[7] = static_cast<double>(c.deflation_rank);
}
int64_t orc_report_n_notes(void* r) { return static_cast<int64_t>(static_cast<SolveReport*>(r)->notes.size()); }
const char* orc_report_note(void* r, int64_t i) { return static_cast<SolveReport*>(r)->notes[static_cast<size_t>(i)].c_str(); }
const char* orc_report_error(void* r) { return static_cast<SolveReport*>(r)->error.c_str(); }
void orc_report_free(void* r) { delete static_cast<SolveReport*>(r); }

// ---- complex GMRES-SDR (skrylov_oracle_complex.hpp; interleaved (re, im) arrays)
void* orc_zcsr_create(int64_t n, const int64_t* off, const int64_t* col, const double* val) {
  auto* A = new cplx::ZCsr();
  A->n = n;
  A->off.assign(off, off + n + 1);
  A->col.assign(col, col + off[n]);
  A->val.resize(static_cast<size_t>(off[n]));
  for (int64_t p = 0; p < off[n]; ++p) A->val[static_cast<size_t>(p)] = {val[2 * p], val[2 * p + 1]};
  return A;
}
void orc_zcsr_free(void* h) { delete static_cast<cplx::ZCsr*>(h); }
void orc_zcsr_apply(void* h, const double* x, double* y) {
  const auto* A = static_cast<cplx::ZCsr*>(h);
  A->apply(reinterpret_cast<const cplx::Z*>(x), reinterpret_cast<cplx::Z*>(y));
}
void* orc_zspace_create() { return new cplx::RecycleSpace(); }
void orc_zspace_free(void* h) { delete static_cast<cplx::RecycleSpace*>(h); }
int64_t orc_zspace_dim(void* h) { return static_cast<cplx::RecycleSpace*>(h)->dim(); }
/// U (n x k), SU / SAU (s x k), column-major interleaved complex.
void orc_zspace_get(void* h, double* U, double* SU, double* SAU) {
  const auto* sp = static_cast<cplx::RecycleSpace*>(h);
  std::memcpy(U, sp->U.a.data(), sizeof(cplx::Z) * sp->U.a.size());
  std::memcpy(SU, sp->SU.a.data(), sizeof(cplx::Z) * sp->SU.a.size());
  std::memcpy(SAU, sp->SAU.a.data(), sizeof(cplx::Z) * sp->SAU.a.size());
}
void orc_zspace_set(void* h, int64_t n, int64_t s, int64_t k, const double* U, const double* SU, const double* SAU) {
  auto* sp = static_cast<cplx::RecycleSpace*>(h);
  sp->U = cplx::ZMat(n, k);
  sp->SU = cplx::ZMat(s, k);
  sp->SAU = cplx::ZMat(s, k);
  std::memcpy(sp->U.a.data(), U, sizeof(cplx::Z) * n * k);
  std::memcpy(sp->SU.a.data(), SU, sizeof(cplx::Z) * s * k);
  std::memcpy(sp->SAU.a.data(), SAU, sizeof(cplx::Z) * s * k);
}
void* orc_zsolve(void* A, const double* b, const orc_config* c, void* space, void* sketch, double* x_out) {
  SolveReport* rep = nullptr;
  guard([&] {
    const auto& M = *static_cast<cplx::ZCsr*>(A);
    cplx::ZVec bb(reinterpret_cast<const cplx::Z*>(b), reinterpret_cast<const cplx::Z*>(b) + M.n);
    cplx::RecycleSpace tmp;
    cplx::RecycleSpace& sp = space ? *static_cast<cplx::RecycleSpace*>(space) : tmp;
    auto r = cplx::solve(M, bb, to_cfg(c), sp, *static_cast<SketchOperator*>(sketch));
    std::memcpy(x_out, r.x.data(), sizeof(cplx::Z) * r.x.size());
    rep = new SolveReport(std::move(r.report));
  });
  return rep;
}
int orc_zrefresh(void* space, void* A, void* sketch, int64_t* counters3) {
  return guard([&] {
    Counters cn;
    cplx::refresh_exact(*static_cast<cplx::RecycleSpace*>(space), *static_cast<cplx::ZCsr*>(A),
                        *static_cast<SketchOperator*>(sketch), cn);
    counters3[0] = cn.matvecs;
    counters3[1] = cn.inner_products;
    counters3[2] = cn.sketch_applies;
  });
}
}
