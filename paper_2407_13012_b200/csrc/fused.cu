// Host orchestration of the fused hot path: sweep planning, simulate,
// expectation, value_and_grad (adjoint walk over exactly two vectors) and the
// Rx layer.  Reference: circuit.py:98-113, adjoint.py:37-77, backend.py:200-207.
#include <nvtx3/nvToolsExt.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <memory>

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
// small.cu: the whole circuit in one CTA for n <= 11
int small_run(qsb_ctx* ctx, qsb_table* t, double2* ket, int p, const double* gammas, const double* betas, int mode,
              double* value, double* dg, double* db);
}  // namespace qsb

extern "C" int qsb_table_phase(qsb_ctx* ctx, qsb_table* t, double* amps, double gamma);
extern "C" int qsb_state_mirror(qsb_ctx* ctx, double* amps, int n);
extern "C" int qsb_diag_scale(qsb_ctx* ctx, double* amps, const double* table, uint64_t len);

namespace qsb {
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
    QSB_CUDA(dev_malloc((void**)&t->d_lut, need * sizeof(double2), ctx->device));
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

}  // namespace qsb

namespace {

// angle LUT of an fp64 table for one phase angle (see TvF64 in sweep_impl.cuh): m entries
// e^{i ang (vmin + 256 k / S)}, then 256 entries e^{i ang j / S}
__global__ void k_build_flut(double2* out, int m, double ang, double vmin, double S) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double sn, cn;
  if (i < m) {
    sincos(ang * (vmin + 256.0 * (double)i / S), &sn, &cn);
    out[i] = make_double2(cn, sn);
  } else if (i < m + 256) {
    sincos(ang * ((double)(i - m) / S), &sn, &cn);
    out[i] = make_double2(cn, sn);
  }
}

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

// Plain single-vector B sweeps run as lock-stepped 2-CTA clusters (256-byte DRAM runs;
// +5% on those sweeps).  Merged and bra/ket sweeps, whose per-tile times vary more,
// measured slower paired and stay unpaired (re-measured with the relaxed cluster
// barrier: still slower).  QSB_PAIR=0 disables, =2 pairs every single-vector B sweep,
// =3 every B sweep (A/B tests).
int pair_mode() {
  const char* e = getenv("QSB_PAIR");
  return e ? atoi(e) : 1;
}

// register-bit family of the fast sweeps (measured per window kind, n=30 chain):
// single-vector plain sweeps 6 on A windows (two R=5 warp groups) and 4 on B windows
// (R=4, paired clusters); single-vector merged sweeps 4 on A, 6 on B (4 when an fp64
// table is staged); merged bra/ket sweeps 4 on A, 3 on B (16 warps); other bra/ket
// sweeps 4.
// Overrides QSB_SWEEP_R1 / QSB_SWEEP_R2 (plain sweeps, 3..6 / 3..4), QSB_SWEEP_R1M
// (merged single-vector sweeps, 4..6) and QSB_SWEEP_R2M (merged bra/ket: 3 or 4) apply
// to both window kinds.  6 = the R=5 shapes with two independent warp groups per CTA.
// ftab: a sweep whose fp64 table tiles are TMA-staged, which only one-group kernels do
// (sweep_impl.cuh TSTG): its single-vector sweeps stay on family 4.
int sweep_family(int nv, int mode, bool is_a, bool ftab = false) {
  const bool merged = mode != SM_PLAIN;
  if (mode == SM_BRIDGE) return 4;
  if (merged && nv == 2) {
    const char* e2 = getenv("QSB_SWEEP_R2M");
    if (!e2) return is_a ? 4 : 3;
    return atoi(e2) == 3 ? 3 : 4;
  }
  if (!merged && nv == 1 && is_a) {  // QSB_SWEEP_R1A: plain single-vector A windows only (A/B runs)
    const char* ea = getenv("QSB_SWEEP_R1A");
    if (ea) return atoi(ea) == 4 ? 4 : 6;
  }
  if (merged && !is_a) {  // QSB_SWEEP_R1MB: B windows only (A/B runs that keep the Z2 mirror A family)
    const char* eb = getenv("QSB_SWEEP_R1MB");
    if (eb) {
      const int r = atoi(eb);
      return (r == 5 || r == 6) ? r : 4;
    }
  }
  const char* e = getenv(merged ? "QSB_SWEEP_R1M" : (nv == 1 ? "QSB_SWEEP_R1" : "QSB_SWEEP_R2"));
  // (round 2, Z2-reduced chain: merged single-vector B sweeps on two R=5 warp groups,
  // 13.4 ms per C3 step vs 14.0 for R=4 and 16.5 for one R=5 group)
  if (!e) return nv == 2 ? 4 : merged ? (is_a || ftab ? 4 : 6) : (is_a && !ftab ? 6 : 4);
  int r = atoi(e);
  if (merged) return (r == 5 || r == 6) ? r : 4;
  if (nv == 2 && r >= 5) r = 4;  // two vectors of 32 amplitudes do not fit in registers
  if (r < 3 || r > 6) r = 4;
  return r;
}

// Fill the tile/phase part of SweepArgs for one sweep. Returns the number of gates.
// n: stored index bits of the arrays; vshift = 1 for a Z2-reduced half statevector,
// whose B windows sit one stored bit below their (virtual) qubits: qubits 0..10 are
// stored bits 0..10, qubit 11 is the top qubit n-1 (local bit 11 of the mirror A tile
// pair), qubits 12.. are stored bits 11.. (sh.lo / sh.hi / sh.glo: qubit numbering)
int build_shape(const SweepShape& sh, int n, int nv, bool exact, SweepArgs& a, int gates_before_phase[kMaxPhases],
                const int* pass2 = nullptr, int gates_before_phase2[kMaxPhases] = nullptr, int* gates2 = nullptr,
                int mode = SM_PLAIN, int vshift = 0, bool ftab = false) {
  int gl[kSweepT];
  for (int i = 0; i < kSweepT; ++i) gl[i] = sh.is_a ? i : (i < 3 ? i : sh.glo + i - 3);
  const int fam = exact ? 4 : sweep_family(nv, mode, sh.is_a, ftab);
  const int shape = pick_shape(exact, sh.is_a, fam);
  a.groups = fam == 6 ? 2 : 1;
  const int np = shape_np(shape);
  PhaseSpec ps[kMaxPhases];
  for (int p = 0; p < np; ++p) ps[p] = shape_phase(shape, p);
  a.shape = shape;
  const int glo_st = sh.is_a ? 3 : sh.glo - vshift;  // stored bit of B-tile local bit 3
  a.glo = glo_st;
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
  a.cshift = glo_st;
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
    add_run(3, glo_st - 3);
    add_run(glo_st + 9, n - glo_st - 9);
  }
  a.ntiles = 1ull << (n - kSweepT);
  // whole window targeted -> the kernel uses the compile-time masks (shape_apply)
  a.full = sh.is_a ? (sh.lo == 0 && sh.hi == kSweepT - 1) : (sh.lo == sh.glo && sh.hi == sh.glo + 8);
  if (a.full)
    for (int p = 0; p < np; ++p)
      if (a.ph[p].apply != shape_apply(shape, p)) return -1;  // planner and kernel must agree
  if (pass2) {
    // second pass of a merged sweep: qubits [pass2[0], pass2[1]], phases in reverse order
    bool applied2[kSweepT] = {false};
    int g2 = 0;
    bool full2 = true;
    for (int pp = 0; pp < np; ++pp) {
      const int p = np - 1 - pp;
      gates_before_phase2[p] = g2;
      uint8_t apply = 0;
      for (int b = 0; b < R; ++b) {
        const int loc = ps[p].reg_l + b;
        const int g = gl[loc];
        if (ps[p].allow && !applied2[loc] && g >= pass2[0] && g <= pass2[1]) {
          apply |= (uint8_t)(1u << b);
          applied2[loc] = true;
          ++g2;
        }
      }
      a.apply2[p] = apply;
      if (apply != shape_apply_rev(shape, p)) full2 = false;
    }
    *gates2 = g2;
    a.full = a.full && full2;
  }
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
  // Z2 reduction: the cost table is flip-symmetric (C(x) = C(~x), every MaxCut), so
  // |+>, the phases and the mixer keep psi(x) = psi(~x); the arrays then hold only
  // phi(x) = psi(x) for x < 2^(n-1) -- half the HBM bytes and FP64 work of every sweep.
  // The top qubit's X acts as the complement of all stored bits: the A window visits
  // tile pairs {T, ~T} (mirror mode), every contraction counts each amplitude twice.
  bool sym = false;
  int st() const { return sym ? n - 1 : n; }  // stored index bits
  const qsb_shard_visit* swap = nullptr;  // fused qubit-swap store (sharded walk)
  // Deferred gate scaling (window chain): the factored gates leave a real scale sigma^g
  // on every amplitude; instead of multiplying it out at the end of every sweep, the
  // chain carries it as `pend` (the vectors entering the next sweep are true/pend) and
  // folds it into the reduction weights; it is applied only where a state becomes
  // visible (the last sweep of a forward chain) or when it drifts towards the
  // exponent range's ends.  (bra and ket always carry the same pending scale.)
  bool defer = false;
  double pend = 1.0;
  bool apply_now = false;  // set by the chain for the sweep that must store true values
  // Forward checkpoints (spare HBM, value_and_grad): forward sweeps write their results to
  // ck[] out of place, so the backward sweeps read the ket from them and never store it.
  // in0 / out0: the v0 source / destination of the next sweep (nullptr: v0 in place).
  // angle LUTs of an fp64 table (fast mode), built lazily per angle into t->d_flut
  struct FLut {
    double ang, S;
    int m;
    uint64_t off;
  };
  std::vector<FLut> fluts;
  uint64_t flut_used = 0;

  const FLut* float_lut(double ang) {
    if (!t || t->kind != 0 || exact) return nullptr;
    const char* e = getenv("QSB_NO_FLUT");
    if (e && atoi(e)) return nullptr;
    for (const FLut& f : fluts)
      if (f.ang == ang) return &f;
    const double range = t->vmax - t->vmin;
    if (!(range >= 0.0) || !std::isfinite(range)) return nullptr;
    double S = 1.0;  // a power of two with |ang| / S <= 2^-9
    while (fabs(ang) / S > 1.0 / 512.0) S *= 2.0;
    const double mm = floor(range * S / 256.0) + 2.0;
    if (mm > 65536.0) return nullptr;
    const int m = (int)mm;
    const uint64_t need = flut_used + (uint64_t)m + 256;
    if (need > t->flut_cap) {  // grow, keeping this call's LUTs
      const uint64_t cap = std::max<uint64_t>(need, 2 * t->flut_cap);
      double2* nb = nullptr;
      if (dev_malloc((void**)&nb, cap * sizeof(double2), ctx->device) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      if (t->d_flut) {
        if (flut_used) cudaMemcpyAsync(nb, t->d_flut, flut_used * sizeof(double2), cudaMemcpyDeviceToDevice, ctx->stream);
        cudaStreamSynchronize(ctx->stream);
        cudaFree(t->d_flut);
      }
      t->d_flut = nb;
      t->flut_cap = cap;
    }
    const int total = m + 256;
    k_build_flut<<<(total + 255) / 256, 256, 0, ctx->stream>>>(t->d_flut + flut_used, m, ang, t->vmin, S);
    if (cudaGetLastError() != cudaSuccess) return nullptr;
    ctx->launches++;
    fluts.push_back({ang, S, m, flut_used});
    flut_used = need;
    return &fluts.back();
  }

  std::vector<double2*> ck;
  bool want_ck = false;  // run_chain asks the context for up to F checkpoints (spare HBM)
  double2* in0 = nullptr;
  double2* out0 = nullptr;

  int init(int total_sweeps_upper) {
    shapes = plan_sweeps(n);
    unsigned g1, g2;
    QSB_TRY(sweep_grid(ctx, 1, exact, 1ull << (st() - kSweepT), &g1));
    QSB_TRY(sweep_grid(ctx, 2, exact, 1ull << (st() - kSweepT), &g2));
    maxgrid = std::max(g1, g2);
    QSB_TRY(ensure_scratch(ctx, (uint64_t)total_sweeps_upper * kSlots * maxgrid * sizeof(double) + 64));
    partials = ctx->d_scratch;
    return QSB_OK;
  }

  // algorithmic HBM bytes of one sweep: every amplitude read/written once, plus
  // one read of the table (compact index or f64) when the sweep has table ops
  double alg_bytes(int nv, int mode, uint32_t flags) const {
    const double N = (double)(1ull << st());
    const double tb = t ? (t->kind == 1 ? 1.0 : t->kind == 2 ? 2.0 : 8.0) : 0.0;
    double b = 0.0;
    if (nv == 1) {
      if (!(flags & SF_PLUS)) b += 16.0 * N;
      if (!(flags & SF_NO_STORE)) b += 16.0 * N;
    } else {
      b += (mode == SM_BRIDGE || (flags & SF_BRA_FROM_KET)) ? 16.0 * N : 32.0 * N;
      if (!(flags & SF_NO_STORE)) b += (flags & SF_KEEP_V0) ? 16.0 * N : 32.0 * N;
    }
    if ((flags & kTableOps) || mode == SM_BRIDGE) b += tb * N;
    return b;
  }

  // live-profiler kind (qsb_prof_end): ((mode * 2 + nv - 1) * 2 + is_b), 12 kinds
  static int prof_kind(int nv, int mode, bool is_a) { return ((mode * 2 + nv - 1) * 2) + (is_a ? 0 : 1); }

  static constexpr uint32_t kTableOps = SF_PRE_PHASE | SF_BRA_FROM_KET | SF_PRE_DINNER | SF_POST_EXPECT |
                                        SF_POST_DINNER | SF_MID_PHASE | SF_MID_DINNER | SF_MID_EXPECT;

  // one plain sweep (one gate pass) over window `sh`, gates on [sh.lo, sh.hi]
  int sweep(int nv, const SweepShape& sh, double2* v0, double2* v1, const Gate& g, uint32_t flags,
            const double2* lut, double pre_ang, double2 pre_extra, bool want_partials, int* idx_out) {
    return sweep_any(nv, SM_PLAIN, sh, nullptr, v0, v1, g, g, flags, lut, pre_ang, pre_extra, want_partials, idx_out);
  }

  // general sweep: pass 1 gates g1 on [sh.lo, sh.hi]; merged / bridge sweeps add
  // mid ops and pass 2 gates g2 on [pass2[0], pass2[1]] (phases in reverse order)
  int sweep_any(int nv, int mode, const SweepShape& sh, const int* pass2, double2* v0, double2* v1, const Gate& g1,
                const Gate& g2, uint32_t flags, const double2* lut, double pre_ang, double2 pre_extra,
                bool want_partials, int* idx_out) {
    SweepArgs a;
    memset(&a, 0, sizeof(a));
    int gbp[kMaxPhases], gbp2[kMaxPhases] = {0, 0, 0, 0}, gates2 = 0;
    // merged / bridge sweeps over an fp64 table: TMA-stage each tile's table values for
    // the mid ops, single-vector plain sweeps for their pre / post ops (QSB_NO_FTAB=1:
    // read them from HBM per element)
    const bool ftab = t && t->kind == 0 && t->values && !exact && !getenv("QSB_NO_FTAB") &&
                      (mode != SM_PLAIN || (nv == 1 && (flags & (SF_PRE_PHASE | SF_POST_EXPECT))));
    const int gates = build_shape(sh, st(), nv, exact, a, gbp, mode != SM_PLAIN ? pass2 : nullptr, gbp2, &gates2, mode,
                                  sym ? 1 : 0, ftab);
    if (gates < 0) return invalid("internal: bad sweep layout");
    a.mode = mode;
    {
      const int pm = pair_mode();
      a.want_pair = ((nv == 1 && ((pm == 1 && mode == SM_PLAIN) || pm == 2)) || pm == 3) ? 1 : 0;
    }
    a.v0 = in0 ? in0 : v0;
    a.v1 = v1;
    a.o0 = out0;
    in0 = out0 = nullptr;  // one sweep only
    set_table(a, t);
    // (a bridge always reads the table: bra = C * ket between its passes)
    const bool table_ops = (flags & kTableOps) || mode == SM_BRIDGE;
    a.cmode = (t && t->kind != 0 && table_ops) ? ((!sh.is_a && t->kind == 1) ? 2 : 1) : 0;
    if (!sh.is_a) {  // TMA boxes for the strided B tiles
      QSB_TRY(encode_b_tile_map(&a.tm0, a.v0, st(), a.glo));
      if (nv == 2) QSB_TRY(encode_b_tile_map(&a.tm1, v1, st(), a.glo));
      if (a.cmode) QSB_TRY(encode_b_cidx_map(&a.tmc, t->cidx, t->kind == 1 ? 1 : 2, st(), a.glo));
    }
    if (ftab) {
      a.ftab = 1;
      if (!sh.is_a) QSB_TRY(encode_b_f64_map(&a.tmf, t->values, st(), a.glo));
    }
    a.mirror = (sym && sh.is_a) ? 1 : 0;
    a.tmask = sym ? (1ull << (st() - 11)) - 1ull : 0ull;
    a.lut = lut;
    a.pre_ang = pre_ang;
    a.pre_extra = pre_extra;
    if (t && t->kind == 0 && !exact && (flags & (SF_PRE_PHASE | SF_MID_PHASE))) {
      if (const FLut* fl = float_lut(pre_ang)) {
        a.flut = t->d_flut + fl->off;
        a.fl_S = fl->S;
        a.fl_xs = pre_ang / fl->S;
        a.fl_m = fl->m;
      }
    }
    a.form = g1.form;
    a.ga = g1.ga;
    a.gb = g1.gb;
    a.plus_amp = plus_amp > 0.0 ? plus_amp : 1.0 / sqrt((double)(1ull << n));
    const double s1 = g1.sigma * g1.sigma;
    // pending scale of the input vectors (deferred scaling; 1 otherwise) and its square,
    // the weight of every bra/ket or ket/ket contraction taken on raw values
    const double S = (defer && !exact) ? pend : 1.0, S2 = S * S;
    // xsum weights: the pending gate scale^2 where the kernel takes the xsum (fast: after
    // the phase's gates; exact: sigma = 1)
    auto after = [](const int* gb, const uint8_t* ap, int p) { return gb[p] + __builtin_popcount(ap[p]); };
    uint8_t ap1[kMaxPhases];
    for (int p = 0; p < kMaxPhases; ++p) ap1[p] = a.ph[p].apply;
    for (int p = 0; p < a.nphase; ++p) a.xs_w[p] = S2 * ipow(s1, exact ? gbp[p] : after(gbp, ap1, p));
    double G;  // this sweep's gate scale
    a.w0 = a.w1 = 1.0;
    if (mode != SM_PLAIN) {
      // pass-1 scale is still pending at the mid ops and throughout pass 2
      const double m = ipow(s1, gates);
      a.w0 = a.w1 = S2 * m;
      a.form2 = g2.form;
      a.ga2 = g2.ga;
      a.gb2 = g2.gb;
      for (int p = 0; p < a.nphase; ++p) a.xs_w2[p] = S2 * m * ipow(g2.sigma * g2.sigma, after(gbp2, a.apply2, p));
      G = ipow(g1.sigma, gates) * ipow(g2.sigma, gates2);
    } else {
      a.form2 = g1.form;
      G = exact ? 1.0 : ipow(g1.sigma, gates);
      a.w1 = S2;  // pre-op <bra|C|ket> on the raw input
    }
    // apply the scale (true values stored) or carry it to the next sweep
    const double out_scale = S * G;
    const bool carry = defer && !exact && !apply_now && fabs(out_scale) > 1e-150 && fabs(out_scale) < 1e150;
    if (carry) {
      a.post_scale = 1.0;
      if (mode == SM_PLAIN) a.w0 = out_scale * out_scale;  // post ops on raw values
    } else {
      a.post_scale = out_scale;
      if (!exact && out_scale != 1.0) flags |= SF_POST_SCALE;
    }
    a.flags = flags;
    if (swap && swap->swap_g) {
      a.sw_g = swap->swap_g;
      a.sw_rank = swap->swap_rank;
      a.sw_nl = n;
      for (int c = 0; c < (1 << swap->swap_g); ++c) {
        a.sw_out[0][c] = (double2*)swap->out0[c];
        a.sw_out[1][c] = (double2*)swap->out1[c];
      }
    }
    const int idx = nsweeps_launched++;
    a.partials = want_partials ? partials + (uint64_t)idx * kSlots * maxgrid : nullptr;
    unsigned grid = 0;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof) QSB_TRY(prof_mark(ctx, &e0));
    {
      // NVTX range per sweep (kind names as in bench.py's "kernels"), so an ncu / nsys run
      // can select sweeps by kind (ncu --nvtx --nvtx-include "braket_merged_A/"); a no-op
      // unless a tool is attached
      static const char* const kNames[12] = {"single_A", "single_B", "braket_A", "braket_B",
                                             "single_merged_A", "single_merged_B", "braket_merged_A",
                                             "braket_merged_B", "single_bridge_A", "single_bridge_B",
                                             "braket_bridge_A", "braket_bridge_B"};
      nvtxRangePushA(kNames[prof_kind(nv, mode, sh.is_a) % 12]);
      const int rc = launch_sweep(ctx, nv, exact, a, &grid);
      nvtxRangePop();
      QSB_TRY(rc);
    }
    if (ctx->prof) {
      QSB_TRY(prof_mark(ctx, &e1));
      ctx->prof_recs.push_back({e0, e1, prof_kind(nv, mode, sh.is_a), alg_bytes(nv, mode, flags)});
    }
    grids.push_back(grid);
    if (idx_out) *idx_out = idx;
    if (defer && !exact) pend = carry ? out_scale : 1.0;
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

// ------------------------------------------------------------------ the window chain
// Every layer (forward or backward) applies its Rx gates window by window.  Layer
// directions alternate (A, B1, .., Bk | Bk, .., B1, A | ...; backward layer i runs
// opposite to forward layer i), so consecutive layers meet on the same window and
// the two visits fuse into ONE merged sweep whose mid ops are the diagonal work
// between the layers: a layer of p forward + p backward costs 2p(K-1)+1 HBM passes
// instead of 2pK (K = windows per layer; n=30: K=3, 25 passes instead of 36).
struct Visit {
  bool bwd;
  int layer;
  int win;
  int lo, hi;
};

// slot contribution of a launched sweep: kind 0 = value, 1 = d_gamma[layer], 2 = d_beta[layer]
struct Contrib {
  int sweep, slot, kind, layer;
};

// QSB_NO_MERGE=1 runs every visit as its own sweep (A/B comparisons, tests)
bool merge_enabled() {
  const char* e = getenv("QSB_NO_MERGE");
  return !(e && atoi(e));
}

std::vector<Visit> chain_visits(int n, const std::vector<SweepShape>& wins, int p, bool fwd, bool bwd) {
  const int K = (int)wins.size();
  std::vector<Visit> out;
  auto gate_mask = [&](int w) -> uint64_t {
    const int lo = wins[w].is_a ? 0 : wins[w].glo;
    const int hi = wins[w].is_a ? std::min(kSweepT, n) - 1 : wins[w].glo + 8;
    return ((hi >= 63 ? ~0ull : ((1ull << (hi + 1)) - 1)) & ~((1ull << lo) - 1));
  };
  // forward layer i visits the windows ascending (i even) or descending (i odd), each
  // gating the qubits its predecessors in the layer have not; backward layer i visits
  // exactly forward layer i's (window, qubits) list in reverse, so every backward visit
  // undoes one forward visit -- with overlapping windows (n < 30: the top B window slides
  // down into the A window) a freshly computed descending partition would differ, and a
  // bridge could not keep the ket it leaves unchanged, nor a backward sweep read its ket
  // from a forward checkpoint
  auto layer = [&](bool b, int i) {
    const bool ascending = i % 2 == 0;
    uint64_t covered = 0;
    std::vector<Visit> fl;
    for (int k = 0; k < K; ++k) {
      const int w = ascending ? k : K - 1 - k;
      const uint64_t m = gate_mask(w) & ~covered;
      covered |= m;
      if (!m) continue;
      fl.push_back({b, i, w, __builtin_ctzll(m), 63 - __builtin_clzll(m)});
    }
    if (b) std::reverse(fl.begin(), fl.end());
    out.insert(out.end(), fl.begin(), fl.end());
  };
  if (fwd)
    for (int i = 0; i < p; ++i) layer(false, i);
  if (bwd)
    for (int i = p - 1; i >= 0; --i) layer(true, i);
  return out;
}

// Runs forward layers 0..p-1 (fwd) and/or the adjoint walk p-1..0 (bwd) as one chain
// of sweeps.  Contributions to <C> / d_gamma / d_beta are recorded in `contribs`.
// Window order of the chain's layers.  Merged sweeps (FP64 / shared-memory bound) land
// on the two END windows of the order, plain (HBM-bound) visits on the middle ones.
// QSB_WIN_ORDER=mid puts the A window second (B1, A, B2, ..): merged sweeps then run on
// 9-qubit B windows (less FP64 per amplitude than A's 12) and the plain visits on the
// contiguous A tiles (the fastest HBM pattern).  Default: A first (A, B1, B2, ..).
std::vector<SweepShape> chain_windows(const std::vector<SweepShape>& shapes) {
  std::vector<SweepShape> w = shapes;
  const char* e = getenv("QSB_WIN_ORDER");
  if (e && strcmp(e, "mid") == 0 && w.size() >= 3 && w[0].is_a) std::swap(w[0], w[1]);
  return w;
}

int run_chain(Runner& R, double2* ket, double2* bra, int p, const double* gammas, const double* betas, bool fwd,
              bool from_plus, bool want_value, bool bwd, std::vector<Contrib>& contribs) {
  const int n = R.n;
  const std::vector<SweepShape> wins = chain_windows(R.shapes);
  const std::vector<Visit> vis = chain_visits(n, wins, p, fwd, bwd);
  const int M = (int)vis.size();
  const bool merge = merge_enabled() && wins.size() >= 2;
  {
    const char* e = getenv("QSB_NO_DEFER");  // A/B: multiply the gate scale out in every sweep
    R.defer = !(e && atoi(e));
    R.pend = 1.0;
  }
  const double2 one = make_double2(1.0, 0.0);
  const uint64_t nvals = R.t->kind != 0 ? (uint64_t)R.t->nvals : 0;
  auto fwd_lut = [&](int i) { return R.t->kind != 0 ? R.t->d_lut + (size_t)i * nvals : nullptr; };
  auto inv_lut = [&](int i) { return R.t->kind != 0 ? R.t->d_lut + (size_t)(p + i) * nvals : nullptr; };
  auto gate_of = [&](const Visit& v) { return make_gate((v.bwd ? 2.0 : -2.0) * betas[v.layer], false); };
  auto win_of = [&](const Visit& v) {
    SweepShape sh = wins[v.win];
    sh.lo = v.lo;
    sh.hi = v.hi;
    return sh;
  };
  // boundary kinds between visit u and u+1: 0 none (same layer), 1 fwd->fwd, 2 fwd->bwd, 3 bwd->bwd
  auto boundary = [&](int u) {
    const Visit &a = vis[u], &b = vis[u + 1];
    if (a.bwd == b.bwd && a.layer == b.layer) return 0;
    if (!a.bwd && !b.bwd) return 1;
    if (!a.bwd && b.bwd) return 2;
    return 3;
  };

  // job kinds in launch order (0 forward, 1 bridge, 2 backward): the checkpoint wiring
  // needs F, the number of forward jobs, before the first launch
  auto is_pair = [&](int u) { return merge && u + 1 < M && vis[u + 1].win == vis[u].win && boundary(u) != 0; };
  int F = 0;
  for (int u = 0; u < M;) {
    const bool pr = is_pair(u);
    if (pr ? boundary(u) == 1 : !vis[u].bwd) ++F;
    u += pr ? 2 : 1;
  }
  // (merged chains only: there every layer boundary is a merged sweep, so forward and
  // backward jobs cover the same gates AND phases and backward job j starts exactly
  // where forward job F-1-j ended; an unmerged chain applies a backward layer's inverse
  // phase at the start of the next sweep instead)
  const bool ck_ok = R.want_ck && fwd && bwd && merge;
  if (ck_ok) QSB_TRY(ensure_checkpoints(R.ctx, 16ull << R.st(), F, R.ck));
  struct CkDone {  // every return path: the buffers may be released again once enqueued
    qsb_ctx* c;
    bool on;
    ~CkDone() {
      if (on) checkpoints_done(c);
    }
  } ck_done{R.ctx, ck_ok};
  const int K = ck_ok ? std::min<int>((int)R.ck.size(), F) : 0;
  if (K > 0) R.defer = false;  // checkpoints hold true values: no scale carried along the chain
  int fj = 0, bj = 0;  // forward / backward jobs launched so far
  // forward job k >= F-K writes checkpoint k-(F-K) (reading the previous one); the bridge
  // and backward job j < K read the ket from checkpoint K-1-j and do not store it
  auto wire = [&](int kind, uint32_t& f) {
    if (K == 0) return;
    if (kind == 0) {
      const int c = fj - (F - K);
      if (c >= 0) {
        R.out0 = R.ck[c];
        R.in0 = c > 0 ? R.ck[c - 1] : nullptr;
      }
    } else if (kind == 1) {
      R.in0 = R.ck[K - 1];
    } else if (bj < K) {
      R.in0 = R.ck[K - 1 - bj];
      f |= SF_KEEP_V0;
    }
  };

  for (int u = 0; u < M;) {
    const Visit& v = vis[u];
    const bool pair = is_pair(u);
    int idx = -1;
    if (pair) {
      const Visit& w = vis[u + 1];
      const int kind = boundary(u);
      const int pass2[2] = {w.lo, w.hi};
      uint32_t f = 0;
      int mode = SM_MERGED, nv = v.bwd ? 2 : 1;
      const double2* lut = nullptr;
      double ang = 0.0;
      if (kind == 1) {  // forward layer i -> i+1: phase exp(-i g_{i+1} C)
        f |= SF_MID_PHASE;
        lut = fwd_lut(w.layer);
        ang = -gammas[w.layer];
      } else if (kind == 2) {  // last forward layer -> first backward layer
        mode = SM_BRIDGE;
        nv = 2;
        if (want_value) f |= SF_MID_EXPECT;
        f |= SF_XSUM2;
        // the ket leaves the bridge as it came in (Rx(+2b) Rx(-2b) = 1): keep HBM's copy
        // instead of storing it -- when that copy carries no pending scale; the bra is then
        // stored with its scale applied so both vectors are true values afterwards
        if (R.pend == 1.0) f |= SF_KEEP_V0;
      } else {  // backward layer i -> i-1: <bra|C|ket>, then the inverse phase exp(+i g_i C)
        f |= SF_XSUM | SF_MID_DINNER | SF_MID_PHASE | SF_XSUM2;
        lut = inv_lut(v.layer);
        ang = gammas[v.layer];
      }
      R.apply_now = (!bwd && u + 2 >= M) || (f & SF_KEEP_V0);  // true values where the chain needs them
      const int jk = kind == 1 ? 0 : kind == 2 ? 1 : 2;
      wire(jk, f);
      QSB_TRY(R.sweep_any(nv, mode, win_of(v), pass2, ket, bra, gate_of(v), gate_of(w), f, lut, ang, one, true, &idx));
      if (jk == 0) ++fj;
      if (jk == 2) ++bj;
      if (kind == 2 && want_value) contribs.push_back({idx, 0, 0, 0});
      if (v.bwd) contribs.push_back({idx, 2, 2, v.layer});
      if (kind == 3) contribs.push_back({idx, 1, 1, v.layer});
      if (w.bwd) contribs.push_back({idx, 3, 2, w.layer});
      u += 2;
      continue;
    }
    // single visit: pre ops from the boundary before it, post ops from the one after
    uint32_t f = 0;
    const double2* lut = nullptr;
    double ang = 0.0;
    int dinner_pre = -1;
    const int before = u == 0 ? -1 : boundary(u - 1);
    if (u == 0) {
      if (fwd) {
        if (from_plus) f |= SF_PLUS;
        f |= SF_PRE_PHASE;
        lut = fwd_lut(0);
        ang = -gammas[0];
      } else {
        f |= SF_BRA_FROM_KET;
      }
    } else if (before == 1) {
      f |= SF_PRE_PHASE;
      lut = fwd_lut(v.layer);
      ang = -gammas[v.layer];
    } else if (before == 2) {
      f |= SF_BRA_FROM_KET;
    } else if (before == 3) {
      f |= SF_PRE_DINNER | SF_PRE_PHASE;
      dinner_pre = vis[u - 1].layer;
      lut = inv_lut(dinner_pre);
      ang = gammas[dinner_pre];
    }
    bool post_expect = false, post_dinner = false;
    if (u == M - 1) {
      if (v.bwd) post_dinner = true;
      else post_expect = want_value;
    } else if (boundary(u) == 2) {
      post_expect = want_value;
    }
    if (post_expect) f |= SF_POST_EXPECT;
    if (post_dinner) f |= SF_POST_DINNER | SF_NO_STORE;
    if (v.bwd) f |= SF_XSUM;
    R.apply_now = !bwd && u == M - 1;
    wire(v.bwd ? 2 : 0, f);
    QSB_TRY(R.sweep(v.bwd ? 2 : 1, win_of(v), ket, bra, gate_of(v), f, lut, ang, one, true, &idx));
    if (v.bwd) ++bj;
    else ++fj;
    if (post_expect) contribs.push_back({idx, 0, 0, 0});
    if (post_dinner) contribs.push_back({idx, 0, 1, v.layer});
    if (dinner_pre >= 0) contribs.push_back({idx, 1, 1, dinner_pre});
    if (v.bwd) contribs.push_back({idx, 2, 2, v.layer});
    ++u;
  }
  return QSB_OK;
}

// reduce the recorded contributions (fixed order) into value / d_gammas / d_betas
void collect(const Runner& R, const std::vector<double>& h, const std::vector<Contrib>& cs, double* value,
             double* dg, double* db, int p) {
  if (value) *value = 0.0;
  for (int i = 0; i < p && dg; ++i) dg[i] = 0.0;
  for (int i = 0; i < p && db; ++i) db[i] = 0.0;
  for (const Contrib& c : cs) {
    // a Z2-reduced sweep sums over half the amplitudes, each standing for two
    const double x = (R.sym ? 2.0 : 1.0) * Runner::slot_sum(h, R.maxgrid, R.grids, c.sweep, c.slot);
    if (c.kind == 0 && value) *value += x;
    else if (c.kind == 1 && dg) dg[c.layer] += 2.0 * x;
    else if (c.kind == 2 && db) db[c.layer] += -2.0 * x;
  }
}

int upper_sweeps(int n, int p) { return 2 * p * (int)plan_sweeps(n).size() + 4; }

// Z2 reduction applies to fast-mode chains over flip-symmetric tables with n >= 21 (every
// B window then lies above the A window's 12 qubits); QSB_NO_SYM=1 disables it
bool env_is(const char* name, const char* dflt) {
  const char* e = getenv(name);
  return !e || strcmp(e, dflt) == 0;
}

bool sym_ok(const qsb_table* t, int n, bool exact) {
  const char* e = getenv("QSB_NO_SYM");
  // the mirror A instantiations exist for the default register families (fused.cu
  // sweep_family) and the staggered bra/ket schedule; A/B experiment overrides of those
  // run the full vector
  const bool default_families = env_is("QSB_SWEEP_R1", "6") && env_is("QSB_SWEEP_R2", "4") &&
                                env_is("QSB_SWEEP_R1M", "4") && env_is("QSB_SWEEP_R2M", "4") && env_is("QSB_STAG", "1");
  return t && t->sym && !exact && n >= 21 && !(e && atoi(e)) && default_families;
}

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
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
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
  for (int k = 0; k < 3; ++k) {  // slot 3 (second-pass xsum) is unused by plain sweeps
    double acc = 0.0;
    for (int sw = 0; sw < ns; ++sw) acc += Runner::slot_sum(h, R.maxgrid, R.grids, sw, k);
    sums[k] = acc;
  }
  return QSB_OK;
}

int qsb_shard_visit_run(qsb_ctx* ctx, qsb_table* t, double* v0, double* v1, int n, int n_global,
                        const qsb_shard_visit* d, double* sums) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !t || !v0 || !d || !sums || (d->nv == 2 && !v1)) return invalid("qsb_shard_visit_run: null argument");
  if (d->nv != 1 && d->nv != 2) return invalid("qsb_shard_visit_run: nv must be 1 or 2");
  if (n < kSweepT || n > 62 || n != t->n) return invalid("qsb_shard_visit_run: n=%d (table n=%d, need >= 12)", n, t->n);
  if (n_global < n || n_global > 62) return invalid("qsb_shard_visit_run: n_global=%d < n=%d", n_global, n);
  if (d->mode < SM_PLAIN || d->mode > SM_BRIDGE || (d->mode == SM_BRIDGE && d->nv != 2))
    return invalid("qsb_shard_visit_run: bad mode %d", d->mode);
  SweepShape sh;
  if (d->window == 0) {
    sh = {true, d->lo1, d->hi1, 0};
  } else {
    if (d->window < 4 || d->window + 9 > n)
      return invalid("qsb_shard_visit_run: B window at %d does not fit n=%d", d->window, n);
    sh = {false, d->lo1, d->hi1, d->window};
  }
  const int wlo = sh.is_a ? 0 : sh.glo, whi = sh.is_a ? kSweepT - 1 : sh.glo + 8;
  if (d->lo1 < wlo || d->hi1 > whi || d->lo1 > d->hi1) return invalid("qsb_shard_visit_run: pass 1 outside the window");
  if (d->mode != SM_PLAIN && (d->lo2 < wlo || d->hi2 > whi || d->lo2 > d->hi2))
    return invalid("qsb_shard_visit_run: pass 2 outside the window");
  if (d->swap_g) {
    if (d->swap_g < 1 || d->swap_g > 3 || n - d->swap_g < whi + 1)
      return invalid("qsb_shard_visit_run: swap store needs the top %d bits outside the window", d->swap_g);
    for (int c = 0; c < (1 << d->swap_g); ++c)
      if (!d->out0[c] || (d->nv == 2 && !d->out1[c])) return invalid("qsb_shard_visit_run: missing swap target %d", c);
  }
  Runner R{ctx, t, n, false};
  R.plus_amp = 1.0 / sqrt((double)(1ull << n_global));
  R.maxgrid = (unsigned)std::min<uint64_t>(ctx->num_sms, 1ull << (n - kSweepT));
  QSB_TRY(ensure_scratch(ctx, (uint64_t)2 * kSlots * R.maxgrid * sizeof(double) + 64));
  R.partials = ctx->d_scratch;
  const double2* lut = nullptr;
  if ((d->flags & (QSB_SW_PRE_PHASE | QSB_SW_MID_PHASE)) && t->kind != 0) {
    QSB_TRY(prepare_luts(t, {d->phase_scale}, {make_double2(1.0, 0.0)}, false));
    lut = t->d_lut;
  }
  const Gate g1 = make_gate(d->theta1, false), g2 = make_gate(d->mode != SM_PLAIN ? d->theta2 : d->theta1, false);
  const int pass2[2] = {d->lo2, d->hi2};
  R.swap = d;
  int idx = -1;
  QSB_TRY(R.sweep_any(d->nv, d->mode, sh, d->mode != SM_PLAIN ? pass2 : nullptr, (double2*)v0, (double2*)v1, g1, g2,
                      d->flags & ~QSB_SW_EXACT, lut, d->phase_scale, make_double2(1.0, 0.0), true, &idx));
  std::vector<double> h;
  QSB_TRY(R.fetch(h));
  for (int k = 0; k < kSlots; ++k) sums[k] = Runner::slot_sum(h, R.maxgrid, R.grids, idx, k);
  return QSB_OK;
}

}  // extern "C"

namespace {
// one instance of qsb_value_and_grad_many in flight on its context's stream
struct Pending {
  std::unique_ptr<Runner> R;
  std::vector<Contrib> cs;
  double* out;
  int p;
};

int finish(Pending& q) {
  std::vector<double> h;
  QSB_TRY(q.R->fetch(h));
  collect(*q.R, h, q.cs, q.out, q.out + 1, q.out + 1 + q.p, q.p);
  q.R.reset();
  return QSB_OK;
}
}  // namespace

extern "C" int qsb_value_and_grad_many(int count, qsb_ctx* const* ctxs, qsb_table* const* tables, double* const* kets,
                                       double* const* bras, const int* ps, const double* gammas, const double* betas,
                                       double* out) {
  if (count < 0 || (count && (!ctxs || !tables || !kets || !bras || !ps || !gammas || !betas || !out)))
    return invalid("qsb_value_and_grad_many: null argument");
  std::vector<Pending> pend(count);
  size_t go = 0, oo = 0;
  for (int k = 0; k < count; ++k) {
    qsb_ctx* ctx = ctxs[k];
    qsb_table* t = tables[k];
    const int p = ps[k];
    if (!ctx || !t || !kets[k] || !bras[k]) return invalid("qsb_value_and_grad_many: null instance %d", k);
    if (p < 1) return invalid("gradient needs depth p >= 1 (instance %d)", k);
    if (t->n < kSweepT) return invalid("qsb_value_and_grad_many: instance %d has n=%d < 12 (qsb_small_batch)", k, t->n);
    QSB_CUDA(cudaSetDevice(ctx->device));
    // a context's partials scratch serves one Runner at a time: complete the previous
    // instance on the same context before issuing this one
    for (int j = k - 1; j >= 0; --j)
      if (ctxs[j] == ctx && pend[j].R) {
        QSB_TRY(finish(pend[j]));
        break;
      }
    const double* g = gammas + go;
    const double* b = betas + go;
    Pending& q = pend[k];
    q.R.reset(new Runner{ctx, t, t->n, false});
    q.R->sym = sym_ok(t, t->n, false);
    q.out = out + oo;
    q.p = p;
    QSB_TRY(q.R->init(upper_sweeps(t->n, p)));
    std::vector<double> scales;
    std::vector<double2> extras;
    for (int i = 0; i < p; ++i) scales.push_back(-g[i]);
    for (int i = 0; i < p; ++i) scales.push_back(g[i]);
    extras.assign(2 * p, make_double2(1.0, 0.0));
    QSB_TRY(prepare_luts(t, scales, extras, false));
    // launches are asynchronous: the next instance is issued while this one runs
    QSB_TRY(run_chain(*q.R, (double2*)kets[k], (double2*)bras[k], p, g, b, true, true, true, true, q.cs));
    go += p;
    oo += 1 + 2 * (size_t)p;
  }
  for (int k = 0; k < count; ++k)
    if (pend[k].R) QSB_TRY(finish(pend[k]));
  return QSB_OK;
}

extern "C" {

int qsb_rx_layer(qsb_ctx* ctx, double* amps, int n, double theta, unsigned flags) {
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
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
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !t || !amps) return invalid("qsb_simulate: null argument");
  if (p < 0 || (p > 0 && (!gammas || !betas))) return invalid("qsb_simulate: bad parameters");
  const bool exact = flags & QSB_EXACT;
  const int n = t->n;
  double2* a = (double2*)amps;
  if (n < kSweepT && p > 0 && (flags & QSB_FROM_PLUS) && p <= 1000)
    return small_run(ctx, t, a, p, gammas, betas, expect_out ? 1 : 0, expect_out, nullptr, nullptr);
  if (n < kSweepT || p == 0) {
    if (p == 0 && (flags & QSB_FROM_PLUS)) QSB_TRY(launch_fill_plus(ctx, a, t->len));
    else QSB_TRY(simulate_perop(ctx, t, a, p, gammas, betas, flags));
    if (expect_out) QSB_TRY(expectation_exact(ctx, t->values, a, t->len, expect_out));
    return QSB_OK;
  }
  Runner R{ctx, t, n, exact};
  R.sym = (flags & QSB_FROM_PLUS) && sym_ok(t, n, exact);
  ctx->last_half = 0;
  QSB_TRY(R.init(upper_sweeps(n, p)));
  std::vector<double> scales;
  std::vector<double2> extras;
  for (int i = 0; i < p; ++i) {
    scales.push_back(-gammas[i]);
    extras.push_back(make_double2(1.0, 0.0));
  }
  QSB_TRY(prepare_luts(t, scales, extras, exact));
  if (!exact) {
    std::vector<Contrib> cs;
    QSB_TRY(run_chain(R, a, nullptr, p, gammas, betas, true, flags & QSB_FROM_PLUS, expect_out != nullptr, false, cs));
    if (expect_out) {
      std::vector<double> h;
      QSB_TRY(R.fetch(h));
      collect(R, h, cs, expect_out, nullptr, nullptr, p);
    }
    if (R.sym) {  // the upper half: psi(2^(n-1) + y) = phi(2^(n-1) - 1 - y)
      if (flags & QSB_HALF_OUT) ctx->last_half = 1;
      else QSB_TRY(qsb_state_mirror(ctx, amps, n));
    }
    return QSB_OK;
  }
  QSB_TRY(forward_fused(R, a, p, gammas, betas, flags, nullptr, 0));
  if (expect_out) QSB_TRY(expectation_exact(ctx, t->values, a, t->len, expect_out));
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
    // Rx(+2 beta) layers: the exact fused sweeps (FMA-free, ascending qubit order:
    // bit-identical to n rx_qubit passes) for n >= 12, else the per-qubit kernel
    if (n >= kSweepT) {
      QSB_TRY(qsb_rx_layer(ctx, (double*)bra, n, 2.0 * betas[i], QSB_EXACT));
      QSB_TRY(qsb_rx_layer(ctx, (double*)ket, n, 2.0 * betas[i], QSB_EXACT));
    } else {
      QSB_TRY(rx_layer_perop(ctx, bra, n, 2.0 * betas[i]));
      QSB_TRY(rx_layer_perop(ctx, ket, n, 2.0 * betas[i]));
    }
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
  if (ctx) QSB_CUDA(cudaSetDevice(ctx->device));  // launches go to the context's GPU
  if (!ctx || !t || !ket_ || !bra_ || !d_gammas || !d_betas) return invalid("qsb_value_and_grad: null argument");
  if (p < 1) return invalid("gradient needs depth p >= 1");
  if (!gammas || !betas) return invalid("qsb_value_and_grad: null parameters");
  const bool exact = flags & QSB_EXACT;
  const int n = t->n;
  double2* ket = (double2*)ket_;
  double2* bra = (double2*)bra_;
  if (n < kSweepT && p <= 1000)
    return small_run(ctx, t, ket, p, gammas, betas, skip_forward ? 3 : 2, value, d_gammas, d_betas);
  if (exact || n < kSweepT)
    return value_and_grad_perop(ctx, t, ket, bra, p, gammas, betas, flags, skip_forward, value, d_gammas, d_betas);

  Runner R{ctx, t, n, false};
  R.sym = !skip_forward && sym_ok(t, n, false);
  R.want_ck = !skip_forward;
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

  std::vector<Contrib> cs;
  QSB_TRY(run_chain(R, ket, bra, p, gammas, betas, !skip_forward, true, value != nullptr && !skip_forward, true, cs));
  std::vector<double> h;
  QSB_TRY(R.fetch(h));
  collect(R, h, cs, value, d_gammas, d_betas, p);
  if (value && skip_forward) *value = NAN;  // caller already has it
  return QSB_OK;
}

}  // extern "C"
