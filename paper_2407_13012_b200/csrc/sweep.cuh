// Fused multi-qubit sweep: descriptor shared by the kernel (sweep.cu) and the
// host-side planner / orchestration (fused.cu).
#pragma once
#include "common.cuh"

namespace qsb {

constexpr int kSweepT = 12;        // tile = 2^12 amplitudes per vector
constexpr int kMaxPhases = 4;
constexpr int kSlots = 3;          // partial-sum slots: 0 expectation, 1 diag inner, 2 xsum

enum SweepFlags : uint32_t {
  SF_PLUS = 1u << 0,         // input is |+> (not loaded)
  SF_PRE_PHASE = 1u << 1,    // multiply by exp(i*ang*T) at load (all vectors)
  SF_BRA_FROM_KET = 1u << 2, // NV=2: bra = T * ket at load (bra not loaded)
  SF_PRE_DINNER = 1u << 3,   // NV=2: slot1 += T*Im(conj(bra) ket) at load, before the phase
  SF_XSUM = 1u << 4,         // NV=2: slot2 += w_phase * Im sum_pairs conj(b)X k, before each gate
  SF_POST_EXPECT = 1u << 5,  // NV=1: slot0 += T*|psi|^2 after gates and post scale
  SF_POST_DINNER = 1u << 6,  // NV=2: slot1 += T*Im(conj(bra) ket) after gates and post scale
  SF_NO_STORE = 1u << 7,
  SF_POST_SCALE = 1u << 8,   // multiply by the real post_scale after the gates
};

// gate forms: new0 = a*t - i*b*u, new1 = -i*b*t + a*u  (times an external real scale)
enum GateForm : int {
  GF_EXACT = 0,    // (a, b) = (c, s), FMA-free products (numba_impl.py:60-72)
  GF_FACT_C = 1,   // (a, b) = (1, s/c), true = c * computed
  GF_FACT_S = 2,   // (a, b) = (c/s, 1), true = s * computed
};

struct PhaseMap {
  uint8_t lane_l[5], lane_g[5];  // local / global bit of lane bit b
  uint8_t warp_l[4], warp_g[4];  // local / global bit of warp bit b
  uint8_t reg_l, reg_g;          // register bits: local reg_l.., global reg_g.. (consecutive)
  uint8_t apply;                 // register bits that receive the gate in this phase
  uint8_t pad;
};

struct SweepArgs {
  double2* v0;            // ket / the single vector
  double2* v1;            // bra (NV=2)
  const void* cidx;       // compact table index (kind 1: u8, 2: u16)
  const double* table;    // fp64 table (kind 0)
  const double2* lut;     // pre-phase LUT (kind 1/2), includes any extra scale
  double pre_ang;         // kind 0: factor = extra * (cos(pre_ang*T), sin(pre_ang*T))
  double2 pre_extra;      // kind 0 extra complex scale
  double vmin;            // compact: T = vmin + idx
  double post_scale;
  double ga, gb;          // gate coefficients (see GateForm)
  double plus_amp;        // 1/sqrt(N)
  double xs_w[kMaxPhases];
  double* partials;       // [kSlots][gridDim.x]
  uint64_t ntiles;
  uint32_t flags;
  int kind;
  int nlut;
  int form;
  int nphase;
  int nruns;
  uint8_t run_pos[4], run_len[4];
  PhaseMap ph[kMaxPhases];
};

// launch one sweep (picks the instantiation); grid chosen from occupancy
int launch_sweep(qsb_ctx* ctx, int nv, bool exact, SweepArgs& a, unsigned* grid_out);
int sweep_grid(qsb_ctx* ctx, int nv, bool exact, uint64_t ntiles, unsigned* grid_out);

}  // namespace qsb
