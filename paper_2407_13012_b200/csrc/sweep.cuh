// Fused multi-qubit sweep: descriptor shared by the kernel (sweep_impl.cuh) and the
// host-side planner / orchestration (fused.cu).
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime driver entry point)

#include "common.cuh"

namespace qsb {

constexpr int kSweepT = 12;        // tile = 2^12 amplitudes per vector
constexpr int kMaxPhases = 4;
// partial-sum slots: 0 expectation / post diag inner (mid expectation in a bridge),
// 1 pre (or mid) diag inner, 2 xsum of the first gate pass, 3 xsum of the second
constexpr int kSlots = 4;

enum SweepFlags : uint32_t {
  SF_PLUS = 1u << 0,         // input is |+> (not loaded)
  SF_PRE_PHASE = 1u << 1,    // multiply by exp(i*ang*T) at load (all vectors)
  SF_BRA_FROM_KET = 1u << 2, // NV=2: bra = T * ket at load (bra not loaded)
  SF_PRE_DINNER = 1u << 3,   // NV=2: slot1 += T*Im(conj(bra) ket) at load, before the phase
  SF_XSUM = 1u << 4,         // NV=2: slot2 += w_phase * Im sum_pairs conj(b)X k, before each gate
  SF_POST_EXPECT = 1u << 5,  // NV=1: slot0 += T*|psi|^2 after gates and post scale
  SF_POST_DINNER = 1u << 6,  // NV=2: slot0 += T*Im(conj(bra) ket) after gates and post scale
  SF_NO_STORE = 1u << 7,
  SF_POST_SCALE = 1u << 8,   // multiply by the real post_scale after the gates
  // merged sweeps (two gate passes over the same window, see SweepMode)
  SF_MID_PHASE = 1u << 9,    // between the passes: multiply by the phase (LUT / pre_ang)
  SF_MID_DINNER = 1u << 10,  // NV=2 merged: slot1 += T*Im(conj(bra) ket) between the passes
  SF_MID_EXPECT = 1u << 11,  // bridge: slot0 += T*|ket|^2 between the passes
  SF_XSUM2 = 1u << 12,       // NV=2: slot3 += xsum over the second pass's qubits
  SF_KEEP_V0 = 1u << 13,     // NV=2: v0 (the ket) is not stored -- the bridge's pass 2 undoes
                             // pass 1 (Rx(+2b) Rx(-2b) = 1), and a backward sweep whose ket
                             // result the next sweep reads from a forward checkpoint
};

// A merged sweep applies two layers' gates to one window per HBM pass.  The chain
// of windows visited by a layer alternates direction (A,B1,B2 | B2,B1,A | ...), so
// consecutive layers meet on the same window; the diagonal operators between them
// (phase, <bra|C|ket>, bra = C*ket, <C>) are elementwise and run between the passes.
enum SweepMode : int {
  SM_PLAIN = 0,   // one gate pass (+ pre / post ops)
  SM_MERGED = 1,  // pass 1 (layer i) -> mid ops -> pass 2 (layer i+-1), same vectors
  SM_BRIDGE = 2,  // NV=2: pass 1 on the ket only (last forward layer) -> <C>, bra = C*ket
                  // -> pass 2 on both (first backward layer)
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
  CUtensorMap tm0, tm1;   // B shapes: 5-D TMA boxes over v0 / v1 (one 64 KB tile per load)
  CUtensorMap tmc;        // B shapes with table ops: 5-D box over the compact index (cmode)
  CUtensorMap tmf;        // B shapes, staged fp64 table (ftab): 5-D box over the fp64 table
  double2* v0;            // ket / the single vector
  double2* v1;            // bra (NV=2)
  double2* o0;            // where v0's result goes (nullptr: in place; a forward checkpoint)
  double2* o1;            // where v1's result goes (nullptr: in place)
  const void* cidx;       // compact table index (kind 1: u8, 2: u16)
  const double* table;    // fp64 table (kind 0)
  const double2* lut;     // pre-phase LUT (kind 1/2), includes any extra scale
  double pre_ang;         // kind 0: factor = extra * (cos(pre_ang*T), sin(pre_ang*T))
  // kind 0, fast mode: angle LUT of pre_ang (nullptr: device sincos) -- fl_m entries
  // e^{i pre_ang (vmin + 256 k / fl_S)}, then 256 entries e^{i pre_ang j / fl_S}
  const double2* flut;
  double fl_S, fl_xs;     // scale S and pre_ang / S
  int fl_m;
  int ftab;               // merged / bridge sweep over an fp64 table: stage its tiles in smem
  double2 pre_extra;      // kind 0 extra complex scale
  double vmin;            // compact: T = vmin + idx
  double post_scale;
  double ga, gb;          // gate coefficients (see GateForm)
  double plus_amp;        // 1/sqrt(N)
  double xs_w[kMaxPhases];
  // merged sweeps: second pass gates (same form family as `form2`), its per-phase
  // xsum weights and gate masks, and end-of-sweep weights of slots 0 / 1
  double ga2, gb2;
  double xs_w2[kMaxPhases];
  double w0, w1;
  uint8_t apply2[kMaxPhases];
  int form2;
  int mode;
  int groups;             // warp groups per CTA (1, or 2 for the R=5 single-vector family "6")
  int want_pair;          // host: B sweeps may run as 2-CTA clusters (QSB_PAIR, fused.cu)
  // fused qubit-swap store (sharded walk): the tile goes to sw_out[q][c], c = the tile's
  // top sw_g local bits, at (local & (2^(sw_nl-sw_g)-1)) | (sw_rank << (sw_nl-sw_g))
  int sw_g, sw_rank, sw_nl;
  double2* sw_out[2][8];
  int pair;               // set at launch: this launch is paired (cluster barrier per tile)
  // Z2-reduced (flip-symmetric) state: the arrays hold the half statevector phi(x) =
  // psi(x), x < 2^(n-1); an A sweep works on tile pairs {T, T ^ tmask} of 2048
  // amplitudes with local bit 11 = the top qubit (see kMirBit in sweep_impl.cuh)
  int mirror;
  uint64_t tmask;
  double* partials;       // [kSlots][gridDim.x]
  uint64_t ntiles;
  uint32_t flags;
  int kind;
  int nlut;
  int form;
  int nphase;
  int nruns;
  uint8_t run_pos[4], run_len[4];
  int cshift;             // global bit of local bit 3 (cidx 8-entry chunk c -> base + (c << cshift))
  int shape;              // SweepShapeId
  int cmode;              // compact index tile in smem: 0 none, 1 natural order, 2 B-tile u8 (16-wide rows)
  int full;               // every window position is a target: gate masks are compile-time (shape_apply)
  int glo;                // B shapes: global bit of local bit 3
  PhaseMap ld;            // cp.async load mapping: lanes <-> local 0..4 (coalesced)
  PhaseMap ph[kMaxPhases];
};

// ---------------------------------------------------------------- sweep shapes
// A shape is the compile-time list of phase mappings of the 12 local bits onto
// (5 lane bits, W warp bits, R consecutive register bits).  Shapes 0-2 are the
// single-vector kernels (R=5, W=2), 3-5 the bra/ket kernels (R=4, W=3).
// "A" shapes: local bit i == global bit i (contiguous 4096-amplitude tiles).
// "B" shapes: local 0..2 -> global 0..2, local 3+i -> global glo+i.
// `allow` = false marks a load-only phase (exact mode keeps ascending order).
struct PhaseSpec {
  int lanes[5];
  int warps[4];
  int reg_l;
  bool allow;
};

// Families: R=5 (4 warps, shapes 0-2), R=4 (8 warps, 3-5), R=3 (16 warps, 6-7).
enum SweepShapeId : int {
  SH_A1 = 0, SH_A1X = 1, SH_B1 = 2, SH_A2 = 3, SH_A2X = 4, SH_B2 = 5, SH_A3 = 6, SH_B3 = 7
};

__host__ __device__ constexpr int shape_np(int sh) {
  return sh == SH_A1 ? 3 : sh == SH_A1X ? 4 : sh == SH_B1 ? 2 : sh == SH_A2 ? 3 : sh == SH_A2X ? 4
       : sh == SH_B2 ? 3 : sh == SH_A3 ? 4 : 3;
}
__host__ __device__ constexpr bool shape_is_a(int sh) { return sh != SH_B1 && sh != SH_B2 && sh != SH_B3; }
__host__ __device__ constexpr int shape_r(int sh) { return sh <= SH_B1 ? 5 : sh <= SH_B2 ? 4 : 3; }
__host__ __device__ constexpr int shape_w(int sh) { return sh <= SH_B1 ? 2 : sh <= SH_B2 ? 3 : 4; }

__host__ __device__ constexpr PhaseSpec shape_phase(int sh, int p) {
  // clang-format off
  return sh == SH_A1 ? (p == 0 ? PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 0, 0}, 7, true}
                      : p == 1 ? PhaseSpec{{5, 6, 7, 8, 9}, {10, 11, 0, 0}, 0, true}
                      :          PhaseSpec{{0, 1, 2, 3, 4}, {10, 11, 0, 0}, 5, true})
       : sh == SH_A1X ? (p == 0 ? PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 0, 0}, 7, false}
                      : p == 1 ? PhaseSpec{{5, 6, 7, 8, 9}, {10, 11, 0, 0}, 0, true}
                      : p == 2 ? PhaseSpec{{0, 1, 2, 3, 4}, {10, 11, 0, 0}, 5, true}
                      :          PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 0, 0}, 7, true})
       : sh == SH_B1 ? (p == 0 ? PhaseSpec{{0, 1, 2, 8, 9}, {10, 11, 0, 0}, 3, true}
                      :          PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 0, 0}, 7, true})
       : sh == SH_A2 ? (p == 0 ? PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 7, 0}, 8, true}
                      : p == 1 ? PhaseSpec{{4, 5, 6, 7, 8}, {9, 10, 11, 0}, 0, true}
                      :          PhaseSpec{{0, 1, 2, 3, 8}, {9, 10, 11, 0}, 4, true})
       : sh == SH_A2X ? (p == 0 ? PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 7, 0}, 8, false}
                      : p == 1 ? PhaseSpec{{4, 5, 6, 7, 8}, {9, 10, 11, 0}, 0, true}
                      : p == 2 ? PhaseSpec{{0, 1, 2, 3, 8}, {9, 10, 11, 0}, 4, true}
                      :          PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 7, 0}, 8, true})
       : sh == SH_B2 ? (p == 0 ? PhaseSpec{{0, 1, 2, 7, 8}, {9, 10, 11, 0}, 3, true}
                      : p == 1 ? PhaseSpec{{0, 1, 2, 3, 4}, {9, 10, 11, 0}, 5, true}
                      :          PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 7, 0}, 8, true})
       : sh == SH_A3 ? (p == 0 ? PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 7, 8}, 9, true}
                      : p == 1 ? PhaseSpec{{3, 4, 5, 6, 7}, {8, 9, 10, 11}, 0, true}
                      : p == 2 ? PhaseSpec{{0, 1, 2, 6, 7}, {8, 9, 10, 11}, 3, true}
                      :          PhaseSpec{{0, 1, 2, 3, 4}, {5, 9, 10, 11}, 6, true})
       :                (p == 0 ? PhaseSpec{{0, 1, 2, 6, 7}, {8, 9, 10, 11}, 3, true}
                      : p == 1 ? PhaseSpec{{0, 1, 2, 3, 4}, {5, 9, 10, 11}, 6, true}
                      :          PhaseSpec{{0, 1, 2, 3, 4}, {5, 6, 7, 8}, 9, true});
  // clang-format on
}

// Gate mask of phase p when the whole window is targeted: register bits that are a
// register bit for the first time (and the phase is allowed to apply gates).
// shape_apply_rev: the same for the reversed phase order (second pass of a merged
// sweep runs phases NP-1 .. 0).
__host__ __device__ constexpr uint32_t shape_apply(int sh, int p) {
  uint32_t m = 0;
  const PhaseSpec P = shape_phase(sh, p);
  if (!P.allow) return 0;
  for (int b = 0; b < shape_r(sh); ++b) {
    const int loc = P.reg_l + b;
    bool seen = false;
    for (int q = 0; q < p; ++q) {
      const PhaseSpec Q = shape_phase(sh, q);
      if (Q.allow && loc >= Q.reg_l && loc < Q.reg_l + shape_r(sh)) seen = true;
    }
    if (!seen) m |= 1u << b;
  }
  return m;
}

__host__ __device__ constexpr uint32_t shape_apply_rev(int sh, int p) {
  uint32_t m = 0;
  const PhaseSpec P = shape_phase(sh, p);
  if (!P.allow) return 0;
  for (int b = 0; b < shape_r(sh); ++b) {
    const int loc = P.reg_l + b;
    bool seen = false;
    for (int q = shape_np(sh) - 1; q > p; --q) {
      const PhaseSpec Q = shape_phase(sh, q);
      if (Q.allow && loc >= Q.reg_l && loc < Q.reg_l + shape_r(sh)) seen = true;
    }
    if (!seen) m |= 1u << b;
  }
  return m;
}

// family r in {6, 5, 4, 3} for fast mode (6 = the R=5 shapes run by two warp groups);
// exact mode always uses the R=4 shapes (ascending qubit order: A2X, B2)
__host__ __device__ constexpr int pick_shape(bool exact, bool is_a, int r) {
  return exact ? (is_a ? SH_A2X : SH_B2)
       : r >= 5 ? (is_a ? SH_A1 : SH_B1) : r == 4 ? (is_a ? SH_A2 : SH_B2) : (is_a ? SH_A3 : SH_B3);
}

// launch one sweep (picks the instantiation from a.shape / a.form / a.kind);
// B shapes need tm0 (and tm1 for NV=2) encoded with encode_b_tile_map()
int launch_sweep(qsb_ctx* ctx, int nv, bool exact, SweepArgs& a, unsigned* grid_out);
// 5-D box over a statevector for a B-shape tile with local bit 3 at global bit glo
int encode_b_tile_map(CUtensorMap* map, const double2* base, int n, int glo);
// 5-D box over the compact index (esz 1 or 2 bytes) for the same B tile
int encode_b_cidx_map(CUtensorMap* map, const void* base, int esz, int n, int glo);
// 5-D box over an fp64 table for the same B tile (4096 doubles in local-index order)
int encode_b_f64_map(CUtensorMap* map, const double* base, int n, int glo);
int sweep_grid(qsb_ctx* ctx, int nv, bool exact, uint64_t ntiles, unsigned* grid_out);
// the A/B experiment families (env knobs selecting non-default register families or the
// lock-step schedules) are compiled only with -DQSB_VARIANTS (tools/build_variant.py)
inline int variant_missing() {
  return invalid("this sweep family is an A/B experiment variant: build it with "
                 "`python tools/build_variant.py variants QSB_VARIANTS=1` and select it with QSB_LIB");
}

}  // namespace qsb
