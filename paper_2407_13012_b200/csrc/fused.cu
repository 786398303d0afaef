// Host orchestration of the fused hot path: sweep planning, simulate,
// expectation, value_and_grad (adjoint walk over exactly two vectors) and the
// Rx layer.  Reference: circuit.py:98-113, adjoint.py:37-77, backend.py:200-207.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "sweep.cuh"

using namespace qsb;

namespace qsb {
// ops.cu
int launch_rx_qubit(qsb_ctx* ctx, double2* amps, uint64_t len, int j, double c, double s);
int launch_fill_plus(qsb_ctx* ctx, double2* amps, uint64_t len);
int launch_phase_lut(qsb_ctx* ctx, qsb_table* t, double2* amps);
int launch_phase_sincos(qsb_ctx* ctx, double2* amps, const double* table, uint64_t len, double gamma);
int expectation_exact(qsb_ctx* ctx, const double* table, const double2* amps, uint64_t len, double* out);
int diag_inner_exact(qsb_ctx* ctx, const double2* a, const double* table, const double2* b, uint64_t len,
                     double* out2);
int xsum_exact(qsb_ctx* ctx, const double2* a, const double2* b, uint64_t len, int nq, double* out2);
}  // namespace qsb

extern "C" int qsb_table_phase(qsb_ctx* ctx, qsb_table* t, double* amps, double gamma);
extern "C" int qsb_diag_scale(qsb_ctx* ctx, double* amps, const double* table, uint64_t len);

namespace {

// ------------------------------------------------------------------ planning
struct SweepShape {
  bool is_a;
  int lo;      // first target qubit
  int hi;      // last target qubit
  int glo;     // global bit of local bit 3 (B sweeps)
};

// sweeps applying gates to qubits [lo, hi] of an n-qubit array: an A sweep for the
// part below 12, then 9-qubit B windows (the last window slides down to n-9)
std::vector<SweepShape> plan_range(int n, int lo, int hi) {
  std::vector<SweepShape> out;
  if (lo < kSweepT) out.push_back({true, lo, std::min(hi, kSweepT - 1), 0});
  for (int s = std::max(lo, kSweepT); s <= hi; s += 9) {
    const int e = std::min(s + 8, hi);
    out.push_back({false, s, e, std::min(s, n - 9)});
  }
  return out;
}

std::vector<SweepShape> plan_sweeps(int n) { return plan_range(n, 0, n - 1); }

// register-bit family of the fast sweeps (QSB_SWEEP_R1 / QSB_SWEEP_R2 override)
int sweep_family(int nv) {
  static int fam[3] = {0, 0, 0};
  if (!fam[nv]) {
    const char* e = getenv(nv == 1 ? "QSB_SWEEP_R1" : "QSB_SWEEP_R2");
    int r = e ? atoi(e) : 0;
    if (nv == 2 && r == 5) r = 0;  // two vectors of 32 amplitudes do not fit in registers
    if (r < 3 || r > 5) r = 4;  // measured best for both kinds on B200 (profiles/)
    fam[nv] = r;
  }
  return fam[nv];
}

// Fill the tile/phase part of SweepArgs for one sweep. Returns the number of gates.
int build_shape(const SweepShape& sh, int n, int nv, bool exact, SweepArgs& a, int gates_before_phase[kMaxPhases]) {
  int gl[kSweepT];
  for (int i = 0; i < kSweepT; ++i) gl[i] = sh.is_a ? i : (i < 3 ? i : sh.glo + i - 3);
  const int shape = pick_shape(exact, sh.is_a, sweep_family(nv));
  const int np = shape_np(shape);
  PhaseSpec ps[kMaxPhases];
  for (int p = 0; p < np; ++p) ps[p] = shape_phase(shape, p);
  a.shape = shape;
  a.glo = sh.is_a ? 3 : sh.glo;
  const int R = shape_r(shape);
  const int W = shape_w(shape);
  bool applied[kSweepT] = {false};
  int gates = 0;
  a.nphase = np;
  for (int p = 0; p < np; ++p) {
    PhaseMap& m = a.ph[p];
    memset(&m, 0, sizeof(m));
    for (int b = 0; b < 5; ++b) {
      m.lane_l[b] = (uint8_t)ps[p].lanes[b];
      m.lane_g[b] = (uint8_t)gl[ps[p].lanes[b]];
    }
    for (int b = 0; b < W; ++b) {
      m.warp_l[b] = (uint8_t)ps[p].warps[b];
      m.warp_g[b] = (uint8_t)gl[ps[p].warps[b]];
    }
    m.reg_l = (uint8_t)ps[p].reg_l;
    m.reg_g = (uint8_t)gl[ps[p].reg_l];
    gates_before_phase[p] = gates;
    uint8_t apply = 0;
    for (int b = 0; b < R; ++b) {
      const int loc = ps[p].reg_l + b;
      const int g = gl[loc];
      if (g != gl[ps[p].reg_l] + b) return -1;  // register bits must be consecutive globally
      if (ps[p].allow && !applied[loc] && g >= sh.lo && g <= sh.hi) {
        apply |= (uint8_t)(1u << b);
        applied[loc] = true;
        ++gates;
      }
    }
    m.apply = apply;
  }
  // cp.async load mapping: lanes <-> local 0..4, warps <-> next W bits, R register bits on top
  {
    PhaseMap& m = a.ld;
    memset(&m, 0, sizeof(m));
    for (int b = 0; b < 5; ++b) {
      m.lane_l[b] = (uint8_t)b;
      m.lane_g[b] = (uint8_t)gl[b];
    }
    for (int b = 0; b < W; ++b) {
      m.warp_l[b] = (uint8_t)(5 + b);
      m.warp_g[b] = (uint8_t)gl[5 + b];
    }
    m.reg_l = (uint8_t)(5 + W);
    m.reg_g = (uint8_t)gl[5 + W];
    for (int b = 0; b < R; ++b)
      if (gl[5 + W + b] != gl[5 + W] + b) return -1;
  }
  a.cshift = gl[3];
  // tile index -> global base: the non-tile bits as contiguous runs
  a.nruns = 0;
  auto add_run = [&](int pos, int len) {
    if (len > 0) {
      a.run_pos[a.nruns] = (uint8_t)pos;
      a.run_len[a.nruns] = (uint8_t)len;
      a.nruns++;
    }
  };
  if (sh.is_a) {
    add_run(kSweepT, n - kSweepT);
  } else {
    add_run(3, sh.glo - 3);
    add_run(sh.glo + 9, n - sh.glo - 9);
  }
  a.ntiles = 1ull << (n - kSweepT);
  // whole window targeted -> the kernel uses the compile-time masks (shape_apply)
  a.full = sh.is_a ? (sh.lo == 0 && sh.hi == kSweepT - 1) : (sh.lo == sh.glo && sh.hi == sh.glo + 8);
  if (a.full)
    for (int p = 0; p < np; ++p)
      if (a.ph[p].apply != shape_apply(shape, p)) return -1;  // planner and kernel must agree
  return gates;
}

struct Gate {
  int form;
  double ga, gb;
  double sigma;  // true = sigma * computed, per gate
};

Gate make_gate(double theta, bool exact) {
  // c, s as backend.apply_rx_layer computes them (backend.py:202-203)
  const double c = cos(theta / 2.0), s = sin(theta / 2.0);
  Gate g;
  if (exact) {
    g.form = GF_EXACT;
    g.ga = c;
    g.gb = s;
    g.sigma = 1.0;
  } else if (fabs(c) >= fabs(s)) {
    g.form = GF_FACT_C;
    g.ga = 1.0;
    g.gb = s / c;
    g.sigma = c;
  } else {
    g.form = GF_FACT_S;
    g.ga = c / s;
    g.gb = 1.0;
    g.sigma = s;
  }
  return g;
}

double ipow(double x, int k) {
  double r = 1.0;
  for (int i = 0; i < k; ++i) r *= x;
  return r;
}

// per-call LUT staging: k-th LUT = t->d_lut + k * nvals
int prepare_luts(qsb_table* t, const std::vector<double>& ang_scales, const std::vector<double2>& extras, bool exact) {
  if (t->kind == 0 || ang_scales.empty()) return QSB_OK;
  qsb_ctx* ctx = t->ctx;
  const size_t need = ang_scales.size() * (size_t)t->nvals;
  // t->d_lut holds nvals entries from finish_table; grow to `need`
  static_assert(sizeof(double2) == 16, "");
  size_t cap = t->h_lutbuf.size() / 2;
  if (cap < need) {
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    if (t->d_lut) cudaFree(t->d_lut);
    t->d_lut = nullptr;
    QSB_CUDA(cudaMalloc(&t->d_lut, need * sizeof(double2)));
    t->h_lutbuf.assign(2 * need, 0.0);
  }
  double* h = t->h_lutbuf.data();
  for (size_t L = 0; L < ang_scales.size(); ++L) {
    for (int k = 0; k < t->nvals; ++k) {
      const double v = t->vmin + (double)k;
      const double ang = ang_scales[L] * v;
      double c = cos(ang), s = sin(ang);
      if (!exact) {
        const double2 e = extras[L];
        const double c2 = c * e.x - s * e.y, s2 = c * e.y + s * e.x;
        c = c2;
        s = s2;
      }
      h[2 * (L * t->nvals + k)] = c;
      h[2 * (L * t->nvals + k) + 1] = s;
    }
  }
  QSB_CUDA(cudaStreamSynchronize(ctx->stream));  // previous users of d_lut are done
  QSB_CUDA(cudaMemcpyAsync(t->d_lut, h, need * sizeof(double2), cudaMemcpyHostToDevice, ctx->stream));
  ctx->h2d_bytes += need * sizeof(double2);
  return QSB_OK;
}

void set_table(SweepArgs& a, qsb_table* t) {
  a.kind = t ? t->kind : 0;
  a.cidx = t ? t->cidx : nullptr;
  a.table = t ? t->values : nullptr;
  a.vmin = t ? t->vmin : 0.0;
  a.nlut = t ? t->nvals : 0;
}

// ------------------------------------------------------------------ small n (< 12): per-op kernels
int rx_layer_perop(qsb_ctx* ctx, double2* amps, int n, double theta) {
  const double c = cos(theta / 2.0), s = sin(theta / 2.0);
  for (int j = 0; j < n; ++j) QSB_TRY(launch_rx_qubit(ctx, amps, 1ull << n, j, c, s));
  return QSB_OK;
}

int simulate_perop(qsb_ctx* ctx, qsb_table* t, double2* amps, int p, const double* gammas, const double* betas,
                   unsigned flags) {
  const uint64_t len = 1ull << t->n;
  if (flags & QSB_FROM_PLUS) QSB_TRY(launch_fill_plus(ctx, amps, len));
  for (int i = 0; i < p; ++i) {
    QSB_TRY(qsb_table_phase(ctx, t, (double*)amps, gammas[i]));
    QSB_TRY(rx_layer_perop(ctx, amps, t->n, -2.0 * betas[i]));
  }
  return QSB_OK;
}

// ------------------------------------------------------------------ fused forward
struct PartialRef {
  int sweep;
  int slot;
};

struct Runner {
  qsb_ctx* ctx;
  qsb_table* t;
  int n;
  bool exact;
  std::vector<SweepShape> shapes;
  std::vector<unsigned> grids;  // per launched sweep
  int nsweeps_launched = 0;
  double* partials = nullptr;   // device, kSlots * maxgrid per sweep
  double plus_amp = 0.0;        // 0: 1/sqrt(2^n)
  unsigned maxgrid = 0;

  int init(int total_sweeps_upper) {
    shapes = plan_sweeps(n);
    unsigned g1, g2;
    QSB_TRY(sweep_grid(ctx, 1, exact, 1ull << (n - kSweepT), &g1));
    QSB_TRY(sweep_grid(ctx, 2, exact, 1ull << (n - kSweepT), &g2));
    maxgrid = std::max(g1, g2);
    QSB_TRY(ensure_scratch(ctx, (uint64_t)total_sweeps_upper * kSlots * maxgrid * sizeof(double) + 64));
    partials = ctx->d_scratch;
    return QSB_OK;
  }

  // algorithmic HBM bytes of one sweep: every amplitude read/written once,
  // plus one table read (compact index or f64) per fused table use
  double alg_bytes(int nv, uint32_t flags) const {
    const double N = (double)(1ull << n);
    const double tb = t ? (t->kind == 1 ? 1.0 : t->kind == 2 ? 2.0 : 8.0) : 0.0;
    double b = 0.0;
    if (nv == 1) {
      if (!(flags & SF_PLUS)) b += 16.0 * N;
      if (!(flags & SF_NO_STORE)) b += 16.0 * N;
      if (flags & SF_PRE_PHASE) b += tb * N;
      if (flags & SF_POST_EXPECT) b += tb * N;
    } else {
      b += (flags & SF_BRA_FROM_KET) ? 16.0 * N : 32.0 * N;
      if (!(flags & SF_NO_STORE)) b += 32.0 * N;
      if (flags & (SF_PRE_PHASE | SF_BRA_FROM_KET | SF_PRE_DINNER)) b += tb * N;
      if (flags & SF_POST_DINNER) b += tb * N;
    }
    return b;
  }

  // launch one sweep; returns its index for partial lookup
  int sweep(int nv, const SweepShape& sh, double2* v0, double2* v1, const Gate& g, uint32_t flags,
            const double2* lut, double pre_ang, double2 pre_extra, bool want_partials, int* idx_out) {
    SweepArgs a;
    memset(&a, 0, sizeof(a));
    int gbp[kMaxPhases];
    const int gates = build_shape(sh, n, nv, exact, a, gbp);
    if (gates < 0) return invalid("internal: bad sweep layout");
    a.v0 = v0;
    a.v1 = v1;
    set_table(a, t);
    const bool table_ops = flags & (SF_PRE_PHASE | SF_BRA_FROM_KET | SF_PRE_DINNER | SF_POST_EXPECT | SF_POST_DINNER);
    a.cmode = (t && t->kind != 0 && table_ops) ? ((!sh.is_a && t->kind == 1) ? 2 : 1) : 0;
    if (!sh.is_a) {  // TMA boxes for the strided B tiles
      QSB_TRY(encode_b_tile_map(&a.tm0, v0, n, sh.glo));
      if (nv == 2) QSB_TRY(encode_b_tile_map(&a.tm1, v1, n, sh.glo));
      if (a.cmode) QSB_TRY(encode_b_cidx_map(&a.tmc, t->cidx, t->kind == 1 ? 1 : 2, n, sh.glo));
    }
    a.lut = lut;
    a.pre_ang = pre_ang;
    a.pre_extra = pre_extra;
    a.form = g.form;
    a.ga = g.ga;
    a.gb = g.gb;
    a.plus_amp = plus_amp > 0.0 ? plus_amp : 1.0 / sqrt((double)(1ull << n));
    for (int p = 0; p < kMaxPhases; ++p) a.xs_w[p] = ipow(g.sigma * g.sigma, gbp[p]);
    a.post_scale = ipow(g.sigma, gates);
    if (!exact && gates > 0) flags |= SF_POST_SCALE;
    a.flags = flags;
    const int idx = nsweeps_launched++;
    a.partials = want_partials ? partials + (uint64_t)idx * kSlots * maxgrid : nullptr;
    unsigned grid = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof) QSB_TRY(prof_mark(ctx, &e0));
    QSB_TRY(launch_sweep(ctx, nv, exact, a, &grid));
    if (ctx->prof) {
      QSB_TRY(prof_mark(ctx, &e1));
      ctx->prof_recs.push_back({e0, e1, nv - 1, alg_bytes(nv, flags)});
    }
    grids.push_back(grid);
    if (idx_out) *idx_out = idx;
    return QSB_OK;
  }

  // sum a slot of a set of sweeps from the host copy of the partials, in a fixed order
  static double slot_sum(const std::vector<double>& h, unsigned maxgrid, const std::vector<unsigned>& grids, int sweep,
                         int slot) {
    const double* p = h.data() + (uint64_t)sweep * kSlots * maxgrid + (uint64_t)slot * grids[sweep];
    // pairwise (deterministic) sum
    std::vector<double> v(p, p + grids[sweep]);
    while (v.size() > 1) {
      std::vector<double> w((v.size() + 1) / 2);
      for (size_t i = 0; i < w.size(); ++i) w[i] = v[2 * i] + (2 * i + 1 < v.size() ? v[2 * i + 1] : 0.0);
      v.swap(w);
    }
    return v.empty() ? 0.0 : v[0];
  }

  int fetch(std::vector<double>& h) {
    h.assign((uint64_t)nsweeps_launched * kSlots * maxgrid, 0.0);
    if (nsweeps_launched) {
      QSB_CUDA(cudaMemcpyAsync(h.data(), partials, h.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      ctx->d2h_bytes += h.size() * sizeof(double);
    }
    QSB_CUDA(cudaStreamSynchronize(ctx->stream));
    return QSB_OK;
  }
};

// forward layers on `amps`; if expect_sweep != nullptr, the last sweep carries SF_POST_EXPECT
int forward_fused(Runner& R, double2* amps, int p, const double* gammas, const double* betas, unsigned flags,
                  int* expect_sweep, int lut_base) {
  const int ns = (int)R.shapes.size();
  for (int i = 0; i < p; ++i) {
    const Gate g = make_gate(-2.0 * betas[i], R.exact);
    for (int s = 0; s < ns; ++s) {
      uint32_t f = 0;
      const double2* lut = nullptr;
      if (s == 0) {
        f |= SF_PRE_PHASE;
        if (i == 0 && (flags & QSB_FROM_PLUS)) f |= SF_PLUS;
        if (R.t->kind != 0) lut = R.t->d_lut + (size_t)(lut_base + i) * R.t->nvals;
      }
      const bool last = (i == p - 1) && (s == ns - 1);
      if (last && expect_sweep) f |= SF_POST_EXPECT;
      QSB_TRY(R.sweep(1, R.shapes[s], amps, nullptr, g, f, lut, -gammas[i], make_double2(1.0, 0.0),
                      last && expect_sweep, last ? expect_sweep : nullptr));
    }
  }
  return QSB_OK;
}

int upper_sweeps(int n, int p) { return 2 * p * (int)plan_sweeps(n).size() + 4; }

}  // namespace

extern "C" {

// Gates Rx(theta) on qubits [lo, hi] of n-qubit array(s) v0 (and v1 when nv == 2),
// with the fused ops in `flags` (QSB_SW_*): pre ops on the first sweep, post ops and
// NO_STORE on the last, XSUM on all.  sums[0..2] = {<C> or post <bra|C|ket>, pre
// <bra|C|ket>, sum_j <bra|X_j|ket>} (imaginary parts for the bra/ket contractions).
// Building block of the sharded walk (dist.py): the gates of one layer are split
// around the index-bit swap.
int qsb_layer_sweeps(qsb_ctx* ctx, qsb_table* t, double* v0, double* v1, int nv, int n, int n_global, int lo,
                     int hi, double theta, unsigned flags, double phase_scale, double* sums) {
  if (!ctx || !t || !v0 || (nv == 2 && !v1) || !sums) return invalid("qsb_layer_sweeps: null argument");
  if (nv != 1 && nv != 2) return invalid("qsb_layer_sweeps: nv must be 1 or 2");
  if (n < kSweepT || n > 62 || n != t->n) return invalid("qsb_layer_sweeps: n=%d (table n=%d, need >= 12)", n, t->n);
  if (lo < 0 || hi >= n || lo > hi) return invalid("qsb_layer_sweeps: bad qubit range [%d, %d]", lo, hi);
  if (n_global < n || n_global > 62) return invalid("qsb_layer_sweeps: n_global=%d < n=%d", n_global, n);
  const bool exact = flags & QSB_SW_EXACT;
  Runner R{ctx, t, n, exact};
  R.plus_amp = 1.0 / sqrt((double)(1ull << n_global));  // |+> of the whole (sharded) register
  R.shapes = plan_range(n, lo, hi);
  unsigned g1 = ctx->num_sms;
  R.maxgrid = (unsigned)std::min<uint64_t>(g1, 1ull << (n - kSweepT));
  QSB_TRY(ensure_scratch(ctx, (uint64_t)(R.shapes.size() + 1) * kSlots * R.maxgrid * sizeof(double) + 64));
  R.partials = ctx->d_scratch;
  const double2* lut = nullptr;
  if ((flags & QSB_SW_PRE_PHASE) && t->kind != 0) {
    QSB_TRY(prepare_luts(t, {phase_scale}, {make_double2(1.0, 0.0)}, exact));
    lut = t->d_lut;
  }
  const Gate g = make_gate(theta, exact);
  const uint32_t pre = flags & (QSB_SW_PLUS | QSB_SW_PRE_PHASE | QSB_SW_BRA_FROM_KET | QSB_SW_PRE_DINNER);
  const uint32_t post = flags & (QSB_SW_POST_EXPECT | QSB_SW_POST_DINNER | QSB_SW_NO_STORE);
  const int ns = (int)R.shapes.size();
  for (int s = 0; s < ns; ++s) {
    uint32_t f = flags & QSB_SW_XSUM;
    if (s == 0) f |= pre;
    if (s == ns - 1) f |= post;
    QSB_TRY(R.sweep(nv, R.shapes[s], (double2*)v0, (double2*)v1, g, f, s == 0 ? lut : nullptr, phase_scale,
                    make_double2(1.0, 0.0), true, nullptr));
  }
  std::vector<double> h;
  QSB_TRY(R.fetch(h));
  for (int k = 0; k < kSlots; ++k) {
    double acc = 0.0;
    for (int sw = 0; sw < ns; ++sw) acc += Runner::slot_sum(h, R.maxgrid, R.grids, sw, k);
    sums[k] = acc;
  }
  return QSB_OK;
}

}  // extern "C"

namespace {

}  // namespace

extern "C" {

int qsb_rx_layer(qsb_ctx* ctx, double* amps, int n, double theta, unsigned flags) {
  if (!ctx || !amps) return invalid("qsb_rx_layer: null argument");
  if (n < 1 || n > 62) return invalid("qsb_rx_layer: n=%d out of range", n);
  const bool exact = flags & QSB_EXACT;
  if (n < kSweepT) return rx_layer_perop(ctx, (double2*)amps, n, theta);
  Runner R{ctx, nullptr, n, exact};
  QSB_TRY(R.init(upper_sweeps(n, 1)));
  const Gate g = make_gate(theta, exact);
  for (const SweepShape& sh : R.shapes)
    QSB_TRY(R.sweep(1, sh, (double2*)amps, nullptr, g, 0, nullptr, 0.0, make_double2(1, 0), false, nullptr));
  return QSB_OK;
}

// simulate with optional fused expectation (expect_out != NULL)
int qsb_simulate_expect(qsb_ctx* ctx, qsb_table* t, double* amps, int p, const double* gammas, const double* betas,
                        unsigned flags, double* expect_out) {
  if (!ctx || !t || !amps) return invalid("qsb_simulate: null argument");
  if (p < 0 || (p > 0 && (!gammas || !betas))) return invalid("qsb_simulate: bad parameters");
  const bool exact = flags & QSB_EXACT;
  const int n = t->n;
  double2* a = (double2*)amps;
  if (n < kSweepT || p == 0) {
    if (p == 0 && (flags & QSB_FROM_PLUS)) QSB_TRY(launch_fill_plus(ctx, a, t->len));
    else QSB_TRY(simulate_perop(ctx, t, a, p, gammas, betas, flags));
    if (expect_out) QSB_TRY(expectation_exact(ctx, t->values, a, t->len, expect_out));
    return QSB_OK;
  }
  Runner R{ctx, t, n, exact};
  QSB_TRY(R.init(upper_sweeps(n, p)));
  std::vector<double> scales;
  std::vector<double2> extras;
  for (int i = 0; i < p; ++i) {
    scales.push_back(-gammas[i]);
    extras.push_back(make_double2(1.0, 0.0));
  }
  QSB_TRY(prepare_luts(t, scales, extras, exact));
  const bool fused_e = expect_out && !exact;
  int esweep = -1;
  QSB_TRY(forward_fused(R, a, p, gammas, betas, flags, fused_e ? &esweep : nullptr, 0));
  if (expect_out) {
    if (fused_e) {
      std::vector<double> h;
      QSB_TRY(R.fetch(h));
      *expect_out = Runner::slot_sum(h, R.maxgrid, R.grids, esweep, 0);
    } else {
      QSB_TRY(expectation_exact(ctx, t->values, a, t->len, expect_out));
    }
  }
  return QSB_OK;
}

int qsb_simulate(qsb_ctx* ctx, qsb_table* t, double* amps, int p, const double* gammas, const double* betas,
                 unsigned flags) {
  return qsb_simulate_expect(ctx, t, amps, p, gammas, betas, flags, nullptr);
}

int qsb_expectation(qsb_ctx* ctx, qsb_table* t, const double* amps, unsigned flags, double* out) {
  (void)flags;
  if (!ctx || !t || !amps || !out) return invalid("qsb_expectation: null argument");
  // reference association (neighbour-pair tree of T*|psi|^2), circuit.py:106-113
  return expectation_exact(ctx, t->values, (const double2*)amps, t->len, out);
}

// Reference-order adjoint walk with the per-op kernels (bit-identical to the
// numba set): used for QSB_EXACT and for n < 12.
static int value_and_grad_perop(qsb_ctx* ctx, qsb_table* t, double2* ket, double2* bra, int p, const double* gammas,
                                const double* betas, unsigned flags, int skip_forward, double* value, double* dg,
                                double* db) {
  const uint64_t len = t->len;
  const int n = t->n;
  if (!skip_forward) QSB_TRY(qsb_simulate_expect(ctx, t, (double*)ket, p, gammas, betas, flags | QSB_FROM_PLUS, nullptr));
  if (value) QSB_TRY(expectation_exact(ctx, t->values, ket, len, value));
  QSB_CUDA(cudaMemcpyAsync(bra, ket, len * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream));
  QSB_TRY(qsb_diag_scale(ctx, (double*)bra, t->values, len));
  for (int i = p - 1; i >= 0; --i) {
    double xs[2], di[2];
    QSB_TRY(xsum_exact(ctx, bra, ket, len, n, xs));
    db[i] = -2.0 * xs[1];
    QSB_TRY(rx_layer_perop(ctx, bra, n, 2.0 * betas[i]));
    QSB_TRY(rx_layer_perop(ctx, ket, n, 2.0 * betas[i]));
    QSB_TRY(diag_inner_exact(ctx, bra, t->values, ket, len, di));
    dg[i] = 2.0 * di[1];
    QSB_TRY(qsb_table_phase(ctx, t, (double*)bra, -gammas[i]));
    QSB_TRY(qsb_table_phase(ctx, t, (double*)ket, -gammas[i]));
  }
  return QSB_OK;
}

int qsb_value_and_grad(qsb_ctx* ctx, qsb_table* t, double* ket_, double* bra_, int p, const double* gammas,
                       const double* betas, unsigned flags, int skip_forward, double* value, double* d_gammas,
                       double* d_betas) {
  if (!ctx || !t || !ket_ || !bra_ || !d_gammas || !d_betas) return invalid("qsb_value_and_grad: null argument");
  if (p < 1) return invalid("gradient needs depth p >= 1");
  if (!gammas || !betas) return invalid("qsb_value_and_grad: null parameters");
  const bool exact = flags & QSB_EXACT;
  const int n = t->n;
  double2* ket = (double2*)ket_;
  double2* bra = (double2*)bra_;
  if (exact || n < kSweepT)
    return value_and_grad_perop(ctx, t, ket, bra, p, gammas, betas, flags, skip_forward, value, d_gammas, d_betas);

  Runner R{ctx, t, n, false};
  QSB_TRY(R.init(upper_sweeps(n, p)));
  // LUTs: forward phases exp(-i g C) for layers 0..p-1, then inverse phases exp(+i g C) for layers 1..p-1
  std::vector<double> scales;
  std::vector<double2> extras;
  for (int i = 0; i < p; ++i) {
    scales.push_back(-gammas[i]);
    extras.push_back(make_double2(1.0, 0.0));
  }
  for (int i = 0; i < p; ++i) {
    scales.push_back(gammas[i]);
    extras.push_back(make_double2(1.0, 0.0));
  }
  QSB_TRY(prepare_luts(t, scales, extras, false));

  int esweep = -1;
  if (!skip_forward) QSB_TRY(forward_fused(R, ket, p, gammas, betas, QSB_FROM_PLUS, value ? &esweep : nullptr, 0));

  const int ns = (int)R.shapes.size();
  std::vector<std::vector<int>> xs_sweeps(p);
  std::vector<int> dg_sweep(p, -1);
  for (int i = p - 1; i >= 0; --i) {
    const Gate g = make_gate(2.0 * betas[i], false);
    for (int s = 0; s < ns; ++s) {
      uint32_t f = SF_XSUM;
      const double2* lut = nullptr;
      double pre_ang = 0.0;
      if (s == 0) {
        if (i == p - 1) {
          f |= SF_BRA_FROM_KET;
        } else {
          // close layer i+1: <bra|C|ket> then its inverse phase exp(+i g_{i+1} C)
          f |= SF_PRE_DINNER | SF_PRE_PHASE;
          pre_ang = gammas[i + 1];
          if (t->kind != 0) lut = t->d_lut + (size_t)(p + i + 1) * t->nvals;
        }
      }
      const bool last = (i == 0) && (s == ns - 1);
      if (last) f |= SF_POST_DINNER | SF_NO_STORE;
      int idx;
      QSB_TRY(R.sweep(2, R.shapes[s], ket, bra, g, f, lut, pre_ang, make_double2(1.0, 0.0), true, &idx));
      xs_sweeps[i].push_back(idx);
      if (s == 0 && i < p - 1) dg_sweep[i + 1] = idx;
      if (last) dg_sweep[0] = idx;
    }
  }
  std::vector<double> h;
  QSB_TRY(R.fetch(h));
  for (int i = 0; i < p; ++i) {
    double xs = 0.0;
    for (int sw : xs_sweeps[i]) xs += Runner::slot_sum(h, R.maxgrid, R.grids, sw, 2);
    d_betas[i] = -2.0 * xs;
    // layer 0's contraction comes from the last sweep's post op (slot 0), the
    // others from the next layer group's first sweep (slot 1)
    d_gammas[i] = 2.0 * Runner::slot_sum(h, R.maxgrid, R.grids, dg_sweep[i], i == 0 ? 0 : 1);
  }
  if (value) {
    if (esweep >= 0) *value = Runner::slot_sum(h, R.maxgrid, R.grids, esweep, 0);
    else *value = NAN;  // skip_forward: caller already has it
  }
  return QSB_OK;
}

}  // extern "C"
