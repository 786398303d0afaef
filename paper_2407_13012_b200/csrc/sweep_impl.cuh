// The fused sweep kernel — the hot path of every forward and backward layer.
// (Instantiated per family in sweep_nv*.cu / sweep_m_*.cu / sweep_bridge.cu /
// sweep_exact.cu; descriptor in sweep.cuh; dispatch in sweep_host.cu.)
//
// One launch streams the whole statevector (or the bra/ket pair) through HBM once.
// A CTA owns 2^12-amplitude tiles whose 12 "local" bits map to global index bits
// (shape "A": bits 0..11, contiguous; shape "B": bits 0..2 for 128-byte runs plus
// 9 higher bits glo..glo+8).  Each thread keeps 2^R amplitudes per vector in
// registers; a phase maps the 12 local bits onto (5 lane bits, W warp bits, R
// register bits), fixed at compile time by the shape, so shared-memory addresses
// are `thread_base (+|^) constant`.  Butterflies for register bits run in
// registers; between phases the tile is re-mapped through an XOR-swizzled
// shared-memory exchange (conflict-free 16-byte accesses: quarter-warp lanes
// always sit on three consecutive local bits, whose swizzle images are
// independent).
//
// Data movement is Blackwell-native: the kernel is persistent (one CTA per SM)
// and one elected thread streams vector-tiles into a ring of three 64 KB
// shared-memory slots with TMA — a single 1-D cp.async.bulk for a contiguous A
// tile, a single 5-D cp.async.bulk.tensor box for a strided B tile — completing
// on per-slot mbarriers (expect_tx).  While a tile is transformed in registers
// the next one or two vector-tiles are in flight (128 KB per SM).  The landed
// tile is read in the natural layout (every shape's first phase puts quarter-warp
// lanes on local bits 0..2: conflict-free), exchanges use the swizzled layout,
// and results go straight from registers to HBM with coalesced 16-byte stores
// (single-vector A tiles: back through the slot and out with one TMA bulk store).
// Bra/ket sweeps can run the two vectors half a stage apart (the staggered schedule,
// flag-mask bit kStagBit) so one vector's exchange overlaps the other's gates.
//
// Fused ops: the cost phase exp(-i*gamma*C) (compact index -> LUT, the index tile
// rides the A-tile TMA), bra = C*ket, <bra|C|ket>, sum_j <bra|X_j|ket> (before each
// phase's gates) and <psi|C|psi>.
#pragma once
#include <type_traits>
#include <utility>

#include "sweep.cuh"

namespace qsb {
namespace sweepk {

using namespace qsbd;

constexpr int kRing = 3;  // shared-memory slots (one vector-tile each)
constexpr uint32_t kTile = 1u << kSweepT;
constexpr uint32_t kSlotBytes = kTile * 16u;
constexpr uint32_t kCBytes = kTile * 2u;  // compact-index slot (u16 worst case)
// u8 phase LUT: up to kLutRep entries are stored 8 times interleaved (entry e, copy q at
// 8e + q) and lane q of each 8-lane quarter-warp reads copy q, so a 16-byte LUT load is
// conflict-free whatever the entries; larger LUTs (<= 256 entries) are stored once.
constexpr int kLutRep = 80;
constexpr uint32_t kLutBytes = kLutRep * 8 * 16;  // 10 KB (the 227 KB budget: ring + index ring + LUT + barriers)
constexpr size_t kSmemBytes = (size_t)kRing * kSlotBytes + (size_t)kRing * kCBytes + kLutBytes + 128;
// an fp64 table tile (4096 doubles) staged for the mid ops of merged / bridge sweeps: one
// slot over the compact-index ring and LUT area, which fp64 tables do not use
constexpr uint32_t kTabBytes = kTile * 8u;
static_assert(kTabBytes <= (size_t)kRing * kCBytes + kLutBytes, "fp64 table slot");
static_assert(kSmemBytes <= 232448, "dynamic shared memory per block on sm_100");
static_assert(256 * 16 <= kLutBytes, "a plain LUT of 256 entries must fit");

__host__ __device__ constexpr uint32_t swz(uint32_t x) {
  return x ^ (((x >> 3) ^ (x >> 6) ^ (x >> 9) ^ (x >> 12)) & 7u);
}

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ double2 lds(uint32_t addr) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts(uint32_t addr, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tma_5d(uint32_t dst, const CUtensorMap* map, int c1, int c4, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
      "%6}], [%7];" ::"r"(dst),
      "l"(map), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(c4), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// TMA stores (bulk groups of the issuing thread)
__device__ __forceinline__ void tma_store_1d(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, int c1, int c4, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(map),
               "r"(0), "r"(c1), "r"(0), "r"(0), "r"(c4), "r"(src)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint64_t tile_base(const SweepArgs& a, uint64_t tile) {
  uint64_t base = 0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if (r < a.nruns) {
      base |= (tile & ((1ull << a.run_len[r]) - 1ull)) << a.run_pos[r];
      tile >>= a.run_len[r];
    }
  }
  return base;
}

// global offset (in amplitudes) of local index l
template <bool IS_A>
__device__ __forceinline__ uint64_t gofs(uint32_t l, int glo) {
  if constexpr (IS_A) return l;
  else return (uint64_t)(l & 7u) | ((uint64_t)(l >> 3) << glo);
}

// local index of this thread's register-0 amplitude under phase map P
template <int W>
__device__ __forceinline__ uint32_t lbase(const PhaseSpec P, int lane, int warp) {
  uint32_t lb = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b) lb |= ((uint32_t)(lane >> b) & 1u) << P.lanes[b];
#pragma unroll
  for (int b = 0; b < W; ++b) lb |= ((uint32_t)(warp >> b) & 1u) << P.warps[b];
  return lb;
}

template <int FORM>
__device__ __forceinline__ void butterfly(double2& t, double2& u, double ga, double gb) {
  if constexpr (FORM == GF_EXACT) {  // numba_impl.py:60-72, products rounded separately
    const double c = ga, s = gb;
    const double2 n0 = make_double2(__dadd_rn(__dmul_rn(c, t.x), __dmul_rn(s, u.y)),
                                    __dadd_rn(__dmul_rn(c, t.y), -__dmul_rn(s, u.x)));
    const double2 n1 = make_double2(__dadd_rn(__dmul_rn(s, t.y), __dmul_rn(c, u.x)),
                                    __dadd_rn(__dmul_rn(c, u.y), -__dmul_rn(s, t.x)));
    t = n0;
    u = n1;
  } else if constexpr (FORM == GF_FACT_C) {  // (a, b) = (1, tau): 4 FMA per pair
    const double2 n0 = make_double2(fma(gb, u.y, t.x), fma(-gb, u.x, t.y));
    const double2 n1 = make_double2(fma(gb, t.y, u.x), fma(-gb, t.x, u.y));
    t = n0;
    u = n1;
  } else {  // (a, b) = (rho, 1)
    const double2 n0 = make_double2(fma(ga, t.x, u.y), fma(ga, t.y, -u.x));
    const double2 n1 = make_double2(fma(ga, u.x, t.y), fma(ga, u.y, -t.x));
    t = n0;
    u = n1;
  }
}

// gates on the register bits in `apply`, for the first NVA vectors
template <int FORM, int NVA, int NV, int NR, int R>
__device__ __forceinline__ void gate_bits(double2 (&v)[NV][NR], uint32_t apply, double ga, double gb) {
#pragma unroll
  for (int b = 0; b < R; ++b) {
    if (apply & (1u << b)) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j & (1 << b)) continue;
        const int k2 = j | (1 << b);
#pragma unroll
        for (int q = 0; q < NVA; ++q) butterfly<FORM>(v[q][j], v[q][k2], ga, gb);
      }
    }
  }
}

// gates on the register bits in `apply`, one vector
template <int FORM, int NR, int R>
__device__ __forceinline__ void gate_vec(double2 (&u)[NR], uint32_t apply, double ga, double gb) {
#pragma unroll
  for (int b = 0; b < R; ++b) {
    if (apply & (1u << b)) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j & (1 << b)) continue;
        butterfly<FORM>(u[j], u[j | (1 << b)], ga, gb);
      }
    }
  }
}

template <class F, int... I>
__device__ __forceinline__ void static_for_impl(F&& f, std::integer_sequence<int, I...>) {
  (f(std::integral_constant<int, I>{}), ...);
}
// f(integral_constant<int, 0>) ... f(integral_constant<int, N-1>), in order
template <int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  static_for_impl(f, std::make_integer_sequence<int, N>{});
}

// an exchange between phases p and q of shape sh keeps every amplitude in its warp
template <int W>
__host__ __device__ constexpr bool stag_local(int sh, int p, int q) {
  bool l = true;
  for (int b = 0; b < W; ++b) l = l && shape_phase(sh, p).warps[b] == shape_phase(sh, q).warps[b];
  return l;
}

// compile-time marker in a kernel's flag mask FM: run a merged bra/ket sweep with the
// staggered schedule (see the kernel); never set in SweepArgs::flags
constexpr uint32_t kStagBit = 1u << 30;
constexpr uint32_t kStagFlags = 0x5fffffffu;  // every flag, staggered (plain sweeps)
// compile-time marker: an A sweep over a flip-symmetric (Z2-reduced) half statevector.
// The unit of work is a PAIR of 2048-amplitude tiles {T, ~T} (contiguous 32 KB each):
// local bits 0..10 are qubits 0..10 within the tile, local bit 11 selects T / ~T and
// carries the top qubit, whose X acts as the complement of all stored bits -- element
// (1, l) holds phi(complement(T*2048 + l)), stored at position 2047 - l of tile ~T, so
// its natural smem position is L ^ 0x7FF.  See SweepArgs::mirror.
constexpr uint32_t kMirBit = 1u << 29;
static_assert((kStagFlags & kMirBit) == 0 && (kStagFlags & kStagBit) != 0, "flag-mask markers");
// the flag mask of a mirror instantiation of FM (0xffffffff = "every flag, no marker")
constexpr uint32_t mir_mask(uint32_t fm) { return fm == 0xffffffffu ? (0x1fffffffu | kMirBit) : (fm | kMirBit); }
#ifndef QSB_STAG_EARLY_STORE
#define QSB_STAG_EARLY_STORE 1  // staggered merged / bridge sweeps store the lead during the lag's last stage
#endif
#ifndef QSB_STAG_EARLY_STORE_PLAIN
#define QSB_STAG_EARLY_STORE_PLAIN 0  // the same for staggered plain sweeps (measured: 1.9 ms per C3 step slower)
#endif
#ifndef QSB_PAIR_SYNC
#define QSB_PAIR_SYNC 1  // paired B sweeps: 0 release/acquire lock-step, 1 relaxed lock-step, 2 one tile of slack
#endif
#ifndef QSB_TMA_STORE
#define QSB_TMA_STORE 1  // single-vector A sweeps (one warp group) store their tiles with TMA
#endif
#ifndef QSB_TMA_STORE_B
#define QSB_TMA_STORE_B 0  // 1: B tiles too (5-D tensor stores)
#endif
#ifndef QSB_LATE_KET
#define QSB_LATE_KET 1  // staggered plain bra/ket sweeps without pre ops land the ket after the bra's first gates
#endif
#ifndef QSB_STAG_ARRIVE_ALL
#define QSB_STAG_ARRIVE_ALL 1  // every thread arrives on the exchange mbarriers (0: one elected lane per warp after a __syncwarp -- same speed, but compute-sanitizer racecheck cannot follow it)
#endif
#ifndef QSB_EXCH_PRESYNC
#define QSB_EXCH_PRESYNC 0  // 1: a CTA barrier before every warp-crossing exchange (A/B builds)
#endif

// Im sum_{b in apply} <bra|X_b|ket> over this thread's register pairs (NV == 2)
template <int NR, int R>
__device__ __forceinline__ double xsum_bits(const double2 (&v)[2][NR], uint32_t apply) {
  double x0 = 0.0, x1 = 0.0, x2 = 0.0, x3 = 0.0;
#pragma unroll
  for (int b = 0; b < R; ++b) {
    if (apply & (1u << b)) {
#pragma unroll
      for (int j = 0; j < NR; ++j) {
        if (j & (1 << b)) continue;
        const int k2 = j | (1 << b);
        x0 = fma(v[1][j].x, v[0][k2].y, x0);
        x1 = fma(-v[1][j].y, v[0][k2].x, x1);
        x2 = fma(v[1][k2].x, v[0][j].y, x2);
        x3 = fma(-v[1][k2].y, v[0][j].x, x3);
      }
    }
  }
  return (x0 + x1) + (x2 + x3);
}

// ------------------------------------------------------------------ kernel
// SH: shape, NV: vectors (1 or 2), FORM: gate arithmetic, KSIN: f64 table +
// device sincos (else compact index + LUT), FULL: every window position is a
// target (gate masks fixed at compile time by the shape), MODE: SweepMode,
// FORM2: gate arithmetic of the second pass (merged / bridge sweeps), GR: warp
// groups per CTA.  With GR = 2 (single-vector sweeps) the CTA holds two independent
// groups of 2^W warps, each working through every other tile with its own named
// barrier, so one group's shared-memory exchanges overlap the other's FP64 gates.
// FM: the flags this instantiation may see (a compile-time mask; code for the others
// is dropped, which keeps the common sweeps lean in registers and instructions).
template <int SH, int NV, int FORM, bool KSIN, bool FULL, int MODE, int FORM2, int GR, uint32_t FM>
__global__ void __launch_bounds__(GR * (32 << shape_w(SH)), 1) k_sweep(const __grid_constant__ SweepArgs a) {
  constexpr int R = shape_r(SH), W = shape_w(SH), NP = shape_np(SH);
  constexpr bool IS_A = shape_is_a(SH);
  constexpr bool EXACT = FORM == GF_EXACT;
  constexpr int NT = 32 << W;
  constexpr int NR = 1 << R;
  constexpr int NVA = MODE == SM_BRIDGE ? 1 : NV;  // vectors of the pre ops and the first pass
  static_assert(5 + W + R == kSweepT, "tile size");
  static_assert(MODE == SM_PLAIN || !EXACT, "merged sweeps are fast-mode only");
  static_assert(MODE != SM_BRIDGE || NV == 2, "a bridge sweep produces the bra");
  static_assert(GR == 1 || (GR == 2 && NV == 1), "warp groups: single-vector sweeps only");
  // staggered merged bra/ket sweep: the two vectors run half a stage apart, so one
  // vector's shared-memory exchange is in flight while the other's gates run
  // (bridge sweeps: the second pass only -- the first runs on the ket alone; plain
  // sweeps: after the pre ops, which need both vectors at load)
  constexpr bool STAG = NV == 2 && GR == 1 && !EXACT && FM != 0xffffffffu && (FM & kStagBit) != 0;
  constexpr bool STAG1 = STAG && MODE == SM_MERGED;  // staggered from the first stage
  constexpr bool STAGP = STAG && MODE == SM_PLAIN;
  constexpr bool EARLY = STAGP ? QSB_STAG_EARLY_STORE_PLAIN != 0 : QSB_STAG_EARLY_STORE != 0;
  // staggered plain sweeps with no pre ops (the ket is not needed before stage 0): the
  // ket lands after the bra's first gates, which hide part of its load latency (its TMA
  // load is issued only when the previous tile releases both slots)
  const bool late_ket = STAGP && QSB_LATE_KET && !(a.flags & (SF_PRE_PHASE | SF_BRA_FROM_KET | SF_PRE_DINNER));
  // single-vector A tiles leave through shared memory and a 1-D TMA store (no per-thread
  // global stores holding registers); the slot is reloaded once the store has read it.
  // (B tiles measured slower with 5-D tensor stores of 128-byte runs.)
  constexpr bool TMAST = QSB_TMA_STORE && NV == 1 && GR == 1 && (IS_A || QSB_TMA_STORE_B);
  // the next load into a slot waits for the slot's store to be read: A tiles issue it
  // after the first phase, B tiles (slow strided loads) at the tile start
  constexpr bool LATE_ISSUE = TMAST && IS_A;
  constexpr bool MIR = IS_A && FM != 0xffffffffu && (FM & kMirBit) != 0;
  static_assert(!MIR || shape_phase(SH, 0).reg_l + R == kSweepT, "mirror: the landing map holds local bit 11 in registers");
  // natural smem position of local index L (the TMA landing / TMA store layout)
  auto nat = [](uint32_t L) -> uint32_t {
    if constexpr (MIR) return (L & 0x800u) ? (L ^ 0x7FFu) : L;
    else return L;
  };
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(smem_raw);
  const uint32_t cring_s = ring_s + kRing * kSlotBytes;
  uint8_t* cring = smem_raw + kRing * kSlotBytes;
  double2* slut = (double2*)(cring + kRing * kCBytes);
  const uint32_t bar_s = ring_s + kRing * kSlotBytes + kRing * kCBytes + kLutBytes;

  const int tid = threadIdx.x & (NT - 1), grp = GR == 1 ? 0 : (int)(threadIdx.x / NT);
  const int lane = tid & 31, warp = tid >> 5;  // within the group
  const uint32_t flags = a.flags & FM;
  const int glo = a.glo;
  // compact-index tiles ride the TMA of the tile's first vector (cmode, see sweep.cuh)
  const int cmode = KSIN ? 0 : a.cmode;
  const uint32_t cbytes = IS_A ? (a.kind == 2 ? 2u * kTile : kTile) : 2u * kTile;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < GR * kRing; ++s) mbar_init(bar_s + 8 * s, 1);
    mbar_init(bar_s + 8 * 8, 1);  // the staged fp64 table tile (merged / bridge sweeps)
    if constexpr (STAG) {  // exchange barriers of the two vectors: one arrival per warp
      mbar_init(bar_s + 8 * 6, QSB_STAG_ARRIVE_ALL ? NT : 1u << W);
      mbar_init(bar_s + 8 * 7, QSB_STAG_ARRIVE_ALL ? NT : 1u << W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!KSIN && a.kind == 1 && (flags & (SF_PRE_PHASE | SF_MID_PHASE))) {  // u8 LUT in smem
    if (a.nlut <= kLutRep) {
      for (int i = threadIdx.x; i < 8 * a.nlut; i += GR * NT) slut[i] = a.lut[i >> 3];
    } else {
      for (int i = threadIdx.x; i < a.nlut; i += GR * NT) slut[i] = a.lut[i];
    }
  }
  __syncthreads();

  const uint64_t my_tiles = a.ntiles > blockIdx.x ? (a.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint64_t nseq = my_tiles * NV;

  // Full barrier of sequence s: one per slot; with GR=2 one per (group, slot), so a
  // barrier only ever has one outstanding phase (tile s and s+6 are consumed by the
  // same group in order, and tile s+6 is issued only after tile s+3, hence s, is done).
  auto seq_bar = [&](uint64_t s) {
    const uint32_t b = (uint32_t)(s % kRing) + (GR == 2 ? 3u * (uint32_t)(s & 1) : 0u);
    return bar_s + 8u * b;
  };
  // producer (thread 0 of a group): sequence s -> slot s % 3.  NV=1: tile s; NV=2:
  // even = bra (v1) of tile s/2, odd = ket (v0).
  auto issue = [&](uint64_t s) {
    if (tid != 0 || s >= nseq) return;
    if constexpr (TMAST) bulk_wait_read0();  // the slot's previous tile has left
    const uint64_t k = s / NV;
    const int q = NV == 2 ? (int)((s & 1) ^ 1) : 0;
    const uint64_t tile = blockIdx.x + k * gridDim.x;
    const uint32_t slot = (uint32_t)(s % kRing);
    const uint32_t bar = seq_bar(s);
    const bool vec = !((q == 0 && (flags & SF_PLUS)) ||
                       (q == 1 && (MODE == SM_BRIDGE || (flags & SF_BRA_FROM_KET))));
    const bool cid = cmode != 0 && (s % NV) == 0;
    const uint32_t bytes = (vec ? kSlotBytes : 0u) + (cid ? cbytes : 0u);
    if (bytes == 0) {
      mbar_arrive(bar);
      return;
    }
    mbar_expect_tx(bar, bytes);
    if (vec) {
      if constexpr (MIR) {  // the pair {T, ~T}: two contiguous 32 KB tiles
        const double2* src = q == 0 ? a.v0 : a.v1;
        tma_1d(ring_s + slot * kSlotBytes, src + (tile << 11), kSlotBytes / 2, bar);
        tma_1d(ring_s + slot * kSlotBytes + kSlotBytes / 2, src + ((tile ^ a.tmask) << 11), kSlotBytes / 2, bar);
      } else if constexpr (IS_A) {
        const uint64_t base = tile << kSweepT;
        tma_1d(ring_s + slot * kSlotBytes, (q == 0 ? a.v0 : a.v1) + base, kSlotBytes, bar);
      } else {
        const int lowbits = glo - 3;
        const int c1 = (int)(tile & ((1ull << lowbits) - 1ull));
        const int c4 = (int)(tile >> lowbits);
        tma_5d(ring_s + slot * kSlotBytes, q == 0 ? &a.tm0 : &a.tm1, c1, c4, bar);
      }
    }
    if (cid) {
      const uint32_t cdst = cring_s + (uint32_t)(k % kRing) * kCBytes;
      if constexpr (MIR) {  // the pair's table entries, the same natural layout as its amplitudes
        const uint8_t* cx = (const uint8_t*)a.cidx;
        const uint32_t esz = cbytes / kTile;
        tma_1d(cdst, cx + (tile << 11) * esz, cbytes / 2, bar);
        tma_1d(cdst + cbytes / 2, cx + ((tile ^ a.tmask) << 11) * esz, cbytes / 2, bar);
      } else if constexpr (IS_A) {
        tma_1d(cdst, (const uint8_t*)a.cidx + (tile << kSweepT) * (cbytes / kTile), cbytes, bar);
      } else {
        const int lowbits = glo - 3;
        const int c1 = (int)(tile & ((1ull << lowbits) - 1ull));
        tma_5d(cdst, &a.tmc, cmode == 2 ? (c1 >> 1) : c1, (int)(tile >> lowbits), bar);
      }
    }
  };
  // group barrier
  auto gsync = [&]() {
    if constexpr (GR == 1) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"(NT) : "memory");
  };
  auto wait_seq = [&](uint64_t s) { mbar_wait(seq_bar(s), (uint32_t)((s / (GR * kRing)) & 1)); };
  // fp64 table tile of a merged / bridge sweep (a.ftab): loaded into one slot at the tile
  // start (every thread has passed the previous tile's table reads by then -- there is a
  // CTA barrier between), waited for just before the mid ops (plain single-vector sweeps:
  // the pre / post ops); the slot overlays the compact-index ring (fp64 tables have none)
  constexpr bool TSTG = GR == 1 && !EXACT && (MODE != SM_PLAIN ? !KSIN : NV == 1);
  const bool tstage = TSTG && a.ftab;
  const uint32_t tab_s = cring_s, tbar = bar_s + 8u * 8u;
  const double* tsm = (const double*)cring;
  auto issue_tab = [&](uint64_t tile) {
    if (!tstage || threadIdx.x != 0) return;
    fence_proxy_async();
    mbar_expect_tx(tbar, kTabBytes);
    if constexpr (MIR) {
      tma_1d(tab_s, a.table + (tile << 11), kTabBytes / 2, tbar);
      tma_1d(tab_s + kTabBytes / 2, a.table + ((tile ^ a.tmask) << 11), kTabBytes / 2, tbar);
    } else if constexpr (IS_A) {
      tma_1d(tab_s, a.table + (tile << kSweepT), kTabBytes, tbar);
    } else {
      const int lowbits = glo - 3;
      tma_5d(tab_s, &a.tmf, (int)(tile & ((1ull << lowbits) - 1ull)), (int)(tile >> lowbits), tbar);
    }
  };

  double acc0 = 0.0, acc0b = 0.0, acc1 = 0.0, acc1b = 0.0, acc2 = 0.0, acc3 = 0.0;
  uint32_t fph[2] = {0u, 0u};  // STAG: phase parity of the two exchange barriers
  double2 v[NV][NR];

  // NV=1: tile k lands in slot k % 3, two tiles in flight.  NV=2: bra / ket of tile k
  // in slots 2k % 3 / (2k+1) % 3, both used for the exchanges; after the tile's last
  // exchange they are refilled with the ket of tile k+1 and the bra of tile k+2
  // (the bra of tile k+1 is already in flight in the third slot).
  // GR=2: tile k in slot k % 3; the group finishing tile k refills its slot with tile
  // k+3 (the other group's next-but-one), so every tile is in flight for about one
  // group-tile time.
  if (grp == 0) {
    issue(0);
    issue(1);
    if constexpr (NV == 2 || GR == 2) issue(2);
  }
  // Paired launch (B windows): CTAs 2c, 2c+1 form a cluster and work on tiles that
  // differ only in global bit 3 -- the two 128-byte halves of the same 256-byte runs.
  // A cluster barrier per tile keeps them in step, so DRAM sees 256-byte requests
  // (measured 4.6 -> 6.2 TB/s for the bare B-tile stream, profiles/r1e_probe_stream.txt).
  // Both CTAs must pass the same number of barriers: iterate to the larger tile count.
  const uint64_t iters = a.pair ? (a.ntiles + gridDim.x - 1) / gridDim.x : my_tiles;
  for (uint64_t k = grp; k < iters; k += GR) {
   if (k < my_tiles) {
    const uint64_t tileT = blockIdx.x + k * gridDim.x;
    const uint64_t base = tile_base(a, tileT);
    issue_tab(tileT);
    const uint32_t tpar = (uint32_t)(((k - (uint64_t)grp) / GR) & 1u);  // this tile's phase of tbar
    // table views: position of local element l in the smem index tile (the natural
    // layout) and its stored index (mirror: element (1, l) is stored at 2047 - l of ~T)
    auto tl = [&](uint32_t l) -> uint32_t { return nat(l); };
    auto tgi = [&](uint32_t l) -> uint64_t {
      if constexpr (MIR) return (l & 0x800u) ? ((tileT ^ a.tmask) << 11) + (~l & 0x7FFu) : (tileT << 11) + l;
      else return base + gofs<IS_A>(l, glo);
    };
    const uint8_t* cs = cring + (uint32_t)(k % kRing) * kCBytes;
    const uint32_t tb8 = (uint32_t)((blockIdx.x + k * gridDim.x) & 1u) << 3;  // cmode 2: tile's half of each row
    constexpr PhaseSpec P0 = shape_phase(SH, 0);
    uint32_t lb = lbase<W>(P0, lane, warp);
    uint32_t xs_addr;      // byte address of the exchange slot for this tile (ket for NV=2)
    uint32_t xb_addr = 0;  // NV=2: the bra's slot

    // Loads are unconditional (a skipped TMA leaves stale data that is overwritten
    // below): no branch around the register tile, hence no phi-moves of it.
    if constexpr (NV == 1) {
      if constexpr (GR == 1 && !LATE_ISSUE) issue(k + 2);  // (LATE_ISSUE: after the first phase)
      wait_seq(k);
      xs_addr = ring_s + (uint32_t)(k % kRing) * kSlotBytes;
      const bool plus = flags & SF_PLUS;
#pragma unroll
      for (int j = 0; j < NR; ++j) {  // natural (TMA) layout
        const double2 x = lds(xs_addr + nat(lb | ((uint32_t)j << P0.reg_l)) * 16u);
        v[0][j] = make_double2(plus ? a.plus_amp : x.x, plus ? 0.0 : x.y);
      }
      if constexpr (MIR) gsync();  // the mirror half was read from other warps' chunks
    } else {
      xb_addr = ring_s + (uint32_t)((2 * k) % kRing) * kSlotBytes;
      xs_addr = ring_s + (uint32_t)((2 * k + 1) % kRing) * kSlotBytes;
      wait_seq(2 * k);
      if constexpr (MODE != SM_BRIDGE) {
#pragma unroll
        for (int j = 0; j < NR; ++j) v[1][j] = lds(xb_addr + nat(lb | ((uint32_t)j << P0.reg_l)) * 16u);
      }
      if constexpr (!STAG1) {  // staggered merged: the ket lands in stage 0
        if (!late_ket) {
          wait_seq(2 * k + 1);
#pragma unroll
          for (int j = 0; j < NR; ++j) v[0][j] = lds(xs_addr + nat(lb | ((uint32_t)j << P0.reg_l)) * 16u);
          if constexpr (MIR) gsync();
        }
      }
    }

    // ---------------------------------------------------------------- table views
    struct TvF64 {  // f64 table from HBM: device sincos, or (fast mode) the angle LUT
      const SweepArgs& a;
      __device__ double val(uint32_t, uint64_t g) const { return a.table[g]; }
      __device__ double2 phase(uint32_t, uint64_t g) const {
        double2 f;
        if (!EXACT && a.flut) {
          // e^{i ang T} = LUT1[k >> 8] * LUT2[k & 255] * e^{i x}: k = floor((T - vmin) S),
          // x = ang (T - vmin - k / S), |x| <= 2^-9 (S is chosen per angle), Taylor to
          // x^4 / x^5 (next terms < 2e-19): a few FMAs and two L1-cached loads instead of
          // a full double-precision sincos per amplitude
          const double u = (a.table[g] - a.vmin) * a.fl_S;
          const double fu = floor(u);
          const int k = (int)fu;
          const double x = a.fl_xs * (u - fu), x2 = x * x;
          const double c = fma(x2, fma(x2, 1.0 / 24.0, -0.5), 1.0);
          const double sn = x * fma(x2, fma(x2, 1.0 / 120.0, -1.0 / 6.0), 1.0);
          f = cmul_fast(cmul_fast(__ldg(&a.flut[k >> 8]), __ldg(&a.flut[a.fl_m + (k & 255)])), make_double2(c, sn));
        } else {
          double sn, cn;
          sincos(a.pre_ang * a.table[g], &sn, &cn);
          f = make_double2(cn, sn);
        }
        if constexpr (!EXACT) f = cmul_fast(f, a.pre_extra);
        return f;
      }
    };
    struct TvF64S {  // the staged fp64 tile (natural positions, tl-mapped by the caller)
      const SweepArgs& a;
      const double* tsm;
      __device__ double val(uint32_t l, uint64_t) const { return tsm[l]; }
      __device__ double2 phase(uint32_t l, uint64_t) const {
        double2 f;
        if (a.flut) {  // see TvF64
          const double u = (tsm[l] - a.vmin) * a.fl_S;
          const double fu = floor(u);
          const int k = (int)fu;
          const double x = a.fl_xs * (u - fu), x2 = x * x;
          const double c = fma(x2, fma(x2, 1.0 / 24.0, -0.5), 1.0);
          const double sn = x * fma(x2, fma(x2, 1.0 / 120.0, -1.0 / 6.0), 1.0);
          f = cmul_fast(cmul_fast(__ldg(&a.flut[k >> 8]), __ldg(&a.flut[a.fl_m + (k & 255)])), make_double2(c, sn));
        } else {
          double sn, cn;
          sincos(a.pre_ang * tsm[l], &sn, &cn);
          f = make_double2(cn, sn);
        }
        return cmul_fast(f, a.pre_extra);
      }
    };
    // LUT slot of entry c: replicated (8c + lane%8) or plain (c)
    const uint32_t lrep = a.nlut <= kLutRep ? 3u : 0u, lq = a.nlut <= kLutRep ? (uint32_t)(lane & 7) : 0u;
    struct TvU8 {  // u8 index tile in natural order, LUT in smem
      const SweepArgs& a;
      const uint8_t* cs;
      const double2* slut;
      uint32_t lrep, lq;
      __device__ double val(uint32_t l, uint64_t) const { return a.vmin + (double)cs[l]; }
      __device__ double2 phase(uint32_t l, uint64_t) const { return slut[((uint32_t)cs[l] << lrep) | lq]; }
    };
    struct TvU16 {  // u16 index tile, LUT in HBM (L1-cached)
      const SweepArgs& a;
      const uint16_t* cs;
      __device__ double val(uint32_t l, uint64_t) const { return a.vmin + (double)cs[l]; }
      __device__ double2 phase(uint32_t l, uint64_t) const { return __ldg(&a.lut[cs[l]]); }
    };
    struct TvU8Rows {  // u8 index of a B tile: 16-wide rows, this tile's half at tb8
      const SweepArgs& a;
      const uint8_t* cs;
      const double2* slut;
      uint32_t tb8, lrep, lq;
      __device__ uint32_t at(uint32_t l) const { return ((l >> 3) << 4) | tb8 | (l & 7u); }
      __device__ double val(uint32_t l, uint64_t) const { return a.vmin + (double)cs[at(l)]; }
      __device__ double2 phase(uint32_t l, uint64_t) const { return slut[((uint32_t)cs[at(l)] << lrep) | lq]; }
    };
    // table-kind dispatch hoisted out of the unrolled loops (tv: value / phase views)
    auto with_table = [&](auto&& fn) {
      if constexpr (KSIN) {
        if (tstage) fn(TvF64S{a, tsm});
        else fn(TvF64{a});
      } else {
        if (cmode == 2) fn(TvU8Rows{a, cs, slut, tb8, lrep, lq});
        else if (a.kind == 1) fn(TvU8{a, cs, slut, lrep, lq});
        else if (a.kind == 2) fn(TvU16{a, (const uint16_t*)cs});
        else if (tstage) fn(TvF64S{a, tsm});
        else fn(TvF64{a});
      }
    };

    // ---------------------------------------------------------------- pre ops
    if constexpr (MODE == SM_PLAIN) {
      auto pre_ops = [&](auto tv) {
        if constexpr (NV == 2) {
          if (flags & SF_BRA_FROM_KET) {
#pragma unroll
            for (int j = 0; j < NR; ++j) {
              const uint32_t l = lb | ((uint32_t)j << P0.reg_l);
              const double t = tv.val(tl(l), tgi(l));
              v[1][j] = make_double2(t * v[0][j].x, t * v[0][j].y);
            }
          }
          if (flags & SF_PRE_DINNER) {
#pragma unroll
            for (int j = 0; j < NR; ++j) {
              const uint32_t l = lb | ((uint32_t)j << P0.reg_l);
              const double t = tv.val(tl(l), tgi(l));
              const double d = v[1][j].x * v[0][j].y - v[1][j].y * v[0][j].x;
              if (j & 1) acc1b = fma(t, d, acc1b);
              else acc1 = fma(t, d, acc1);
            }
          }
        }
        if (flags & SF_PRE_PHASE) {
#pragma unroll
          for (int j = 0; j < NR; ++j) {
            const uint32_t l = lb | ((uint32_t)j << P0.reg_l);
            const double2 f = tv.phase(tl(l), tgi(l));
#pragma unroll
            for (int q = 0; q < NV; ++q) v[q][j] = cmul<EXACT>(v[q][j], f);
          }
        }
      };
      if (tstage) mbar_wait(tbar, tpar);  // the staged table tile serves the pre and post ops
      if (flags & (SF_PRE_PHASE | SF_BRA_FROM_KET | SF_PRE_DINNER)) with_table([&](auto tv) { pre_ops(tv); });
    }  // merged sweeps start and end mid-layer: no pre / post ops

    // exchange the register tile from phase map Q to phase map P through this tile's
    // slot(s) (swizzled): NV=1 through its one slot, NV=2 the ket and the bra through
    // their own slots at once.  When Q and P put the same local bits on the warp
    // index, every warp reads back only what it wrote (the swizzle keeps bits >= 3
    // fixed, and warp bits are >= 5): a warp barrier suffices.
    auto exchange = [&](const PhaseSpec Q, const PhaseSpec P, auto nvx) {
      bool local = true;
#pragma unroll
      for (int b = 0; b < W; ++b) local = local && Q.warps[b] == P.warps[b];
      const uint32_t nlb = lbase<W>(P, lane, warp);
      const uint32_t so = swz(lb) * 16u, sn = swz(nlb) * 16u;
      // no CTA barrier before the stores: each thread overwrites only the slots it read
      // under map Q (the landing read in the natural layout stays within the warp)
      // (kept for plain bra/ket B sweeps, where it measured faster: warps in step)
      constexpr bool PRESYNC = QSB_EXCH_PRESYNC || (NV == 2 && MODE == SM_PLAIN && !IS_A);
      if (PRESYNC && !local) gsync(); else __syncwarp();
#pragma unroll
      for (int q = 0; q < decltype(nvx)::value; ++q) {
        const uint32_t xa = q == 0 ? xs_addr : xb_addr;
#pragma unroll
        for (int j = 0; j < NR; ++j) sts(xa + (so ^ (swz((uint32_t)j << Q.reg_l) * 16u)), v[q][j]);
      }
      if (local) __syncwarp(); else gsync();
#pragma unroll
      for (int q = 0; q < decltype(nvx)::value; ++q) {
        const uint32_t xa = q == 0 ? xs_addr : xb_addr;
#pragma unroll
        for (int j = 0; j < NR; ++j) v[q][j] = lds(xa + (sn ^ (swz((uint32_t)j << P.reg_l) * 16u)));
      }
      lb = nlb;
    };
    // NV=2: after the tile's last exchange both slots are free -> refill them.  The
    // fence orders this tile's generic-proxy smem writes before the TMA writes.
    auto release = [&]() {
      if constexpr (NV == 2) {
        fence_proxy_async();
        __syncthreads();
        issue(2 * k + 3);
        issue(2 * k + 4);
      }
    };
    // sum_j <bra|X_j|ket> over this phase's gated qubits.  X_j commutes with every Rx,
    // so any point of the layer where both vectors carry the same gates gives the same
    // value: fast mode takes it after the phase's gates (xs_w = the pending scale^2
    // then), exact mode before them (the reference's order).
    auto xsum = [&](double& acc, double w, uint32_t apply) {
      if constexpr (NV == 2) acc = fma(w, xsum_bits<NR, R>(v, apply), acc);
    };

    // ---------------------------------------------------------------- pass 1
#pragma unroll
    for (int p = 0; p < ((STAG1 || STAGP) ? 0 : NP); ++p) {
      if (p > 0) exchange(shape_phase(SH, p - 1), shape_phase(SH, p), std::integral_constant<int, NVA>{});
      if (LATE_ISSUE && p == 1) issue(k + 2);  // tile k-1's store has long read its slot
      if (MODE == SM_PLAIN && p == NP - 1) release();
      // FULL: compile-time gate mask (no branches around the register tile)
      const uint32_t apply = FULL ? shape_apply(SH, p) : a.ph[p].apply;
      constexpr bool XS1 = NV == 2 && MODE != SM_BRIDGE;
      if constexpr (XS1 && EXACT) {
        if (flags & SF_XSUM) xsum(acc2, a.xs_w[p], apply);
      }
      gate_bits<FORM, NVA, NV, NR, R>(v, apply, a.ga, a.gb);
      if constexpr (XS1 && !EXACT) {
        if (flags & SF_XSUM) xsum(acc2, a.xs_w[p], apply);
      }
    }

    // ---------------------------------------------------------------- mid ops + pass 2
    // mid ops: the diagonal work between the passes, both vectors in the last map
    // (local base lbm)
    auto mid_ops = [&](uint32_t lbm) {
      constexpr int RM = shape_phase(SH, NP - 1).reg_l;
      if (tstage) mbar_wait(tbar, tpar);
      with_table([&](auto tv) {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const uint32_t lf = lbm | ((uint32_t)j << RM);
          const uint32_t l = tl(lf);
          const uint64_t g = tgi(lf);
          if constexpr (MODE == SM_BRIDGE) {
            const double t = tv.val(l, g);
            if (flags & SF_MID_EXPECT) {
              const double d = fma(v[0][j].x, v[0][j].x, v[0][j].y * v[0][j].y);
              if (j & 1) acc0b = fma(t, d, acc0b);
              else acc0 = fma(t, d, acc0);
            }
            v[1][j] = make_double2(t * v[0][j].x, t * v[0][j].y);
          } else {
            if constexpr (NV == 2) {
              if (flags & SF_MID_DINNER) {
                const double t = tv.val(l, g);
                const double d = v[1][j].x * v[0][j].y - v[1][j].y * v[0][j].x;
                if (j & 1) acc1b = fma(t, d, acc1b);
                else acc1 = fma(t, d, acc1);
              }
            }
            if (flags & SF_MID_PHASE) {
              const double2 f = tv.phase(l, g);
#pragma unroll
              for (int q = 0; q < NV; ++q) v[q][j] = cmul_fast(v[q][j], f);
            }
          }
        }
      });
    };
    if constexpr (MODE != SM_PLAIN && !STAG) {
      mid_ops(lb);
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) {
        const int p = NP - 1 - pp;
        if (pp > 0) exchange(shape_phase(SH, p + 1), shape_phase(SH, p), std::integral_constant<int, NV>{});
        if (pp == NP - 1) release();
        const uint32_t apply = FULL ? shape_apply_rev(SH, p) : a.apply2[p];
        gate_bits<FORM2, NV, NV, NR, R>(v, apply, a.ga2, a.gb2);
        if (flags & SF_XSUM2) xsum(acc3, a.xs_w2[p], apply);
      }
    }

    // ---------------------------------------------------------------- post helpers
    // the map the tile ends in: the last phase (plain) or the first (merged)
    constexpr int RL = shape_phase(SH, MODE == SM_PLAIN ? NP - 1 : 0).reg_l;
    // factored gates: one real scale per sweep (unless deferred)
    auto scale_vec = [&](int q) {
      const double sc = a.post_scale;
#pragma unroll
      for (int j = 0; j < NR; ++j) v[q][j] = make_double2(v[q][j].x * sc, v[q][j].y * sc);
    };
    auto store_vec = [&](int q) {
      double2* dst = q == 0 ? (a.o0 ? a.o0 : a.v0) : (a.o1 ? a.o1 : a.v1);  // out of place: a checkpoint
      if constexpr (MIR) {  // element (m, l): tile T at l, or tile ~T at 2047 - l
        const uint64_t t0 = tileT << 11, t1 = (tileT ^ a.tmask) << 11;
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const uint32_t L = lb | ((uint32_t)j << RL);
          st_stream(dst + ((L & 0x800u) ? t1 + (~L & 0x7FFu) : t0 + L), v[q][j]);
        }
        return;
      }
      uint64_t g1 = base + gofs<IS_A>(lb, glo);
      if (a.sw_g) {  // qubit swap fused into the store: the whole tile goes to shard c
        const int hb = a.sw_nl - a.sw_g;
        const uint64_t c = base >> hb;
        dst = a.sw_out[q][c];
        g1 = (g1 & ((1ull << hb) - 1ull)) | ((uint64_t)a.sw_rank << hb);
      }
      dst += g1;
#pragma unroll
      for (int j = 0; j < NR; ++j) st_stream(dst + gofs<IS_A>((uint32_t)j << RL, glo), v[q][j]);
    };

    // ------------------------------------------- staggered merged bra/ket sweep
    // Stages s = 0 .. 2NP-1 visit the maps P0 .. P(NP-1), P(NP-1) .. P0 (pass 1 gates,
    // mid ops after stage NP-1, pass 2 gates).  The lead vector (the bra: it lands
    // first) runs half a stage ahead of the lag (the ket): in every stage the lead is
    // gated while the lag's load from shared memory is in flight, and the lag is gated
    // while the lead's exchange is.  An exchange needs no barrier before its stores
    // (each thread writes the slots it alone read, under the map it leaves; the landing
    // read is per-warp, hence the __syncwarp) and one per-vector mbarrier (an arrival
    // per warp) before its loads when it moves warp bits -- no CTA-wide barrier until
    // the slots are released for the next tile.
    if constexpr (STAG) {
      using QLc = std::integral_constant<int, 1>;  // lead (bra)
      using QGc = std::integral_constant<int, 0>;  // lag (ket)
      auto xstore = [&](auto qc, const PhaseSpec Q, auto localc) {
        constexpr int q = decltype(qc)::value;
        const uint32_t xa = q == 0 ? xs_addr : xb_addr;
        const uint32_t so = swz(lbase<W>(Q, lane, warp)) * 16u;
        __syncwarp();
#pragma unroll
        for (int j = 0; j < NR; ++j) sts(xa + (so ^ (swz((uint32_t)j << Q.reg_l) * 16u)), v[q][j]);
        if constexpr (!decltype(localc)::value) {
          if constexpr (QSB_STAG_ARRIVE_ALL) {
            mbar_arrive(bar_s + 8u * (6u + (uint32_t)q));
          } else {
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_s + 8u * (6u + (uint32_t)q));
          }
        }
      };
      auto xload = [&](auto qc, const PhaseSpec P, auto localc) {
        constexpr int q = decltype(qc)::value;
        const uint32_t xa = q == 0 ? xs_addr : xb_addr;
        if constexpr (decltype(localc)::value) {
          __syncwarp();
        } else {
          mbar_wait(bar_s + 8u * (6u + (uint32_t)q), fph[q]);
          fph[q] ^= 1u;
        }
        const uint32_t sn = swz(lbase<W>(P, lane, warp)) * 16u;
#pragma unroll
        for (int j = 0; j < NR; ++j) v[q][j] = lds(xa + (sn ^ (swz((uint32_t)j << P.reg_l) * 16u)));
      };
      constexpr int NS = MODE == SM_PLAIN ? NP : 2 * NP;  // stages
      // the stage at which the lag is already in registers (no load): after the pre ops
      // (plain) or the mid ops (merged / bridge)
      constexpr int SREG = MODE == SM_PLAIN ? 0 : NP;
      static_for<NS>([&](auto sc) {
        constexpr int s = decltype(sc)::value;
        if constexpr (MODE == SM_BRIDGE && s < NP) {  // pass 1 ran in lock-step on the ket
          if constexpr (s == NP - 1) {
            mid_ops(lb);
            lb = lbase<W>(shape_phase(SH, 0), lane, warp);  // the tile ends in map P0 (stores)
          }
          return;
        }
        constexpr int p = s < NP ? s : 2 * NP - 1 - s;
        constexpr PhaseSpec M = shape_phase(SH, p);
        // an exchange follows this stage unless it ends pass 1 (same map) or the sweep
        constexpr bool exch = s != NP - 1 && s != NS - 1;
        constexpr int pn = s + 1 < NP ? s + 1 : 2 * NP - 2 - s;  // map of stage s+1
        constexpr bool loc = exch && stag_local<W>(SH, p, pn);
        const uint32_t apply = s < NP ? (FULL ? shape_apply(SH, p) : a.ph[p].apply)
                                      : (FULL ? shape_apply_rev(SH, p) : a.apply2[p]);
        auto gates = [&](auto qc) {
          constexpr int q = decltype(qc)::value;
          if constexpr (s < NP) gate_vec<FORM, NR, R>(v[q], apply, a.ga, a.gb);
          else gate_vec<FORM2, NR, R>(v[q], apply, a.ga2, a.gb2);
        };
        gates(QLc{});
        if constexpr (s == 0 && MODE == SM_PLAIN) {
          if (late_ket) {  // the lag lands (natural layout)
            wait_seq(2 * k + 1);
#pragma unroll
            for (int j = 0; j < NR; ++j) v[0][j] = lds(xs_addr + nat(lb | ((uint32_t)j << M.reg_l)) * 16u);
            if constexpr (MIR) gsync();
          }
        }
        if constexpr (s == 0 && MODE == SM_MERGED) {  // the lag lands (natural layout)
          wait_seq(2 * k + 1);
#pragma unroll
          for (int j = 0; j < NR; ++j) v[0][j] = lds(xs_addr + nat(lb | ((uint32_t)j << M.reg_l)) * 16u);
          if constexpr (MIR) gsync();  // before the first exchange stores into either slot
        } else if constexpr (s != SREG) {
          constexpr int pp = s - 1 < NP ? s - 1 : 2 * NP - s;  // map of stage s-1
          xload(QGc{}, M, std::integral_constant<bool, stag_local<W>(SH, pp, p)>{});
        }
        if constexpr (exch) xstore(QLc{}, M, std::integral_constant<bool, loc>{});
        if constexpr (s == NS - 1) {
          release();  // the lag's last read: refill both slots
          if constexpr (MODE == SM_PLAIN) lb = lbase<W>(M, lane, warp);  // the tile ends in this map
          // the lead is final: its stores drain while the lag is gated (scaled here, so
          // its last xsum weight is divided by the scale)
          if constexpr (EARLY) {
            if (!EXACT && (flags & SF_POST_SCALE)) scale_vec(1);
            if (!(flags & SF_NO_STORE)) store_vec(1);
          }
        }
        gates(QGc{});
        double w = s < NP ? a.xs_w[p] : a.xs_w2[p];
        if constexpr (s == NS - 1 && EARLY) {
          if (!EXACT && (flags & SF_POST_SCALE)) w /= a.post_scale;
        }
        if constexpr (s < NP) {
          if (flags & SF_XSUM) xsum(acc2, w, apply);
        } else {
          if (flags & SF_XSUM2) xsum(acc3, w, apply);
        }
        if constexpr (s == NP - 1 && MODE == SM_MERGED) mid_ops(lbase<W>(M, lane, warp));
        if constexpr (exch) {
          xload(QLc{}, shape_phase(SH, pn), std::integral_constant<bool, loc>{});
          xstore(QGc{}, M, std::integral_constant<bool, loc>{});
        }
      });
    }

    // ---------------------------------------------------------------- post
    // (STAG: the lead is scaled and stored in the last stage)
    constexpr int Q0 = 0, Q1 = STAG && EARLY ? 1 : NV;  // vectors scaled / stored here
    if (!EXACT && (flags & SF_POST_SCALE)) {
#pragma unroll
      for (int q = Q0; q < Q1; ++q) scale_vec(q);
    }
    if constexpr (MODE == SM_PLAIN) {
      // post ops: <psi|C|psi> (NV=1) or <bra|C|ket> (NV=2) after the gates, in the last map
      if (flags & (SF_POST_EXPECT | SF_POST_DINNER)) with_table([&](auto tv) {
#pragma unroll
        for (int j = 0; j < NR; ++j) {
          const uint32_t l = lb | ((uint32_t)j << RL);
          const double t = tv.val(tl(l), tgi(l));
          double d;
          if constexpr (NV == 1) d = fma(v[0][j].x, v[0][j].x, v[0][j].y * v[0][j].y);
          else d = v[1][j].x * v[0][j].y - v[1][j].y * v[0][j].x;  // slot 0: PRE_DINNER may use slot 1
          if (j & 1) acc0b = fma(t, d, acc0b);
          else acc0 = fma(t, d, acc0);
        }
      });
    }
    // NV=1: order this tile's generic-proxy smem writes (exchanges) before the TMA that
    // will refill the slot.  Fenced here, ahead of the global stores: the fence's
    // MEMBAR then does not wait for this tile's 64 KB of stores to drain.
    // (B tiles: the 5-D store map is the input's, so out-of-place sweeps -- forward
    // checkpoints -- store from registers)
    const bool tma_out = TMAST && a.sw_g == 0 && !(flags & SF_NO_STORE) && (IS_A || !a.o0);
    if (tma_out) {
      // natural layout (the final map puts quarter-warp lanes on local bits 0..2:
      // conflict-free, and each 8-amplitude chunk is the warp's own -- a warp barrier
      // orders it after the last exchange's reads)
      if constexpr (MIR) gsync();  // the mirror half lands in other warps' chunks
      else __syncwarp();
#pragma unroll
      for (int j = 0; j < NR; ++j) sts(xs_addr + nat(lb | ((uint32_t)j << RL)) * 16u, v[0][j]);
    }
    if constexpr (NV == 1) fence_proxy_async();
    if (!(flags & SF_NO_STORE) && !tma_out) {
#pragma unroll
      for (int q = Q0; q < Q1; ++q) {
        if (q == 0 && (flags & SF_KEEP_V0)) continue;  // the ket's result is not stored
        store_vec(q);
      }
    }
    if constexpr (NV == 1) {
      gsync();  // the slot may be refilled from here on (TMAST: once the store has read it)
      if constexpr (TMAST) {
        if (tma_out && tid == 0) {
          const uint64_t tile = blockIdx.x + k * gridDim.x;
          double2* ob = a.o0 ? a.o0 : a.v0;
          if constexpr (MIR) {
            tma_store_1d(ob + (tile << 11), xs_addr, kSlotBytes / 2);
            tma_store_1d(ob + ((tile ^ a.tmask) << 11), xs_addr + kSlotBytes / 2, kSlotBytes / 2);
          } else if constexpr (IS_A) {
            tma_store_1d(ob + (tile << kSweepT), xs_addr, kSlotBytes);
          } else {
            const int lowbits = glo - 3;
            tma_store_5d(&a.tm0, (int)(tile & ((1ull << lowbits) - 1ull)), (int)(tile >> lowbits), xs_addr);
          }
          bulk_commit();
        }
      }
      if constexpr (GR == 2) issue(k + 3);
    }
   }  // k < my_tiles
    if (a.pair) {  // no data crosses the pair: a relaxed arrive (no fence on this tile's stores)
      if constexpr (QSB_PAIR_SYNC == 0) {
        asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      } else if constexpr (QSB_PAIR_SYNC == 1) {
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
        asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
      } else {  // one tile of slack: wait for the partner's previous tile, then arrive
        if (k != (uint64_t)grp) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
        asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      }
    }
  }
  if constexpr (QSB_PAIR_SYNC == 2) {
    if (a.pair && iters > (uint64_t)grp) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }

  if constexpr (TMAST) {
    if (tid == 0) bulk_wait0();  // the tiles are in global memory before the kernel ends
  }

  // ------------------------------------------------------------ partial sums
  if (a.partials) {
    double* red = (double*)smem_raw;
    __syncthreads();
    acc0 = warp_sum(acc0 + acc0b);
    acc1 = warp_sum(acc1 + acc1b);
    acc2 = warp_sum(acc2);
    acc3 = warp_sum(acc3);
    constexpr int NW = GR << W;
    const int gw = threadIdx.x >> 5;
    if (lane == 0) {
      red[gw] = acc0;
      red[NW + gw] = acc1;
      red[2 * NW + gw] = acc2;
      red[3 * NW + gw] = acc3;
    }
    __syncthreads();
    if (threadIdx.x < kSlots) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) s += red[threadIdx.x * NW + w];
      // slots 0 / 1 of a merged sweep are taken before the final scale
      const double wt = threadIdx.x == 0 ? a.w0 : threadIdx.x == 1 ? a.w1 : 1.0;
      a.partials[threadIdx.x * gridDim.x + blockIdx.x] = s * wt;
    }
  }
}

template <int SH, int NV, int FORM, bool KSIN, bool FULL, int MODE = SM_PLAIN, int FORM2 = FORM, int GR = 1,
          uint32_t FM = 0xffffffffu>
struct SweepKernel {
  static constexpr int threads = GR * (32 << shape_w(SH));
  static int grid(qsb_ctx* ctx, uint64_t ntiles, unsigned* g) {
    // once per device (function attributes are per device; thread-safe)
    struct Init {
      cudaError_t err;
      int occ;
    };
    static PerDevice<Init> cache;
    const Init& init = cache.get(ctx->device, [&] {
      Init r{cudaSetDevice(ctx->device), 1};
      if (r.err == cudaSuccess)
        r.err = cudaFuncSetAttribute(k_sweep<SH, NV, FORM, KSIN, FULL, MODE, FORM2, GR, FM>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
      int o = 0;
      if (r.err == cudaSuccess)
        r.err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_sweep<SH, NV, FORM, KSIN, FULL, MODE, FORM2, GR, FM>,
                                                              threads, kSmemBytes);
      r.occ = o < 1 ? 1 : o;
      return r;
    });
    QSB_CUDA(init.err);
    const uint64_t want = (uint64_t)ctx->num_sms * init.occ;
    *g = (unsigned)(ntiles < want ? ntiles : want);
    return QSB_OK;
  }
  static int launch(qsb_ctx* ctx, SweepArgs& a, unsigned* gout) {
    unsigned g;
    QSB_TRY(grid(ctx, a.ntiles, &g));
    // B windows run as 2-CTA clusters (see the kernel) when the grid allows it
    a.pair = (!shape_is_a(SH) && GR == 1 && (g % 2) == 0 && a.want_pair) ? 1 : 0;
    if (a.pair) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(g);
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = kSmemBytes;
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      QSB_CUDA(cudaLaunchKernelEx(&cfg, k_sweep<SH, NV, FORM, KSIN, FULL, MODE, FORM2, GR, FM>, a));
    } else {
      k_sweep<SH, NV, FORM, KSIN, FULL, MODE, FORM2, GR, FM><<<g, threads, kSmemBytes, ctx->stream>>>(a);
    }
    QSB_CHECK_LAUNCH(ctx, "sweep");
    if (gout) *gout = g;
    return QSB_OK;
  }
};

// fast-mode instantiations of one register family (A shape SA, B shape SB, GR warp
// groups; FMX = kStagFlags: the staggered bra/ket schedule).  A sweeps always cover their whole 12-bit window; B windows may be partial.
template <int NV, int SA, int SB, int GR = 1, uint32_t FMX = 0xffffffffu, bool WM = false>
int launch_fast(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  auto L = [&](auto k) { return decltype(k)::launch(ctx, a, g); };
  const bool ksin = a.kind == 0;
  const bool c = a.form == GF_FACT_C;
  constexpr int C = GF_FACT_C, S = GF_FACT_S, P = SM_PLAIN;
  // lean instantiation: whole window, gates only -- the chain's mid-layer forward
  // sweeps (for bra/ket sweeps the lean variant measured slower: not used)
  constexpr uint32_t LEAN = SF_POST_SCALE;
  if (a.mirror && a.shape == SA) {  // Z2-reduced half statevector (whole A window only)
    if constexpr (WM) {
      if (!a.full) return invalid("internal: mirror A sweeps gate the whole window");
      constexpr uint32_t FM = mir_mask(FMX);
      if constexpr (NV == 1) {
        if ((a.flags & ~LEAN) == 0)
          return c ? L(SweepKernel<SA, NV, C, false, true, P, C, GR, LEAN | kMirBit>{})
                   : L(SweepKernel<SA, NV, S, false, true, P, S, GR, LEAN | kMirBit>{});
      }
      if (c) return ksin ? L(SweepKernel<SA, NV, C, true, true, P, C, GR, FM>{}) : L(SweepKernel<SA, NV, C, false, true, P, C, GR, FM>{});
      return ksin ? L(SweepKernel<SA, NV, S, true, true, P, S, GR, FM>{}) : L(SweepKernel<SA, NV, S, false, true, P, S, GR, FM>{});
    } else {
      return invalid("internal: this sweep family has no mirror (Z2-reduced) A instantiation");
    }
  }
  if constexpr (NV == 1) {
    if (a.full && (a.flags & ~LEAN) == 0) {
      if (a.shape == SA) return c ? L(SweepKernel<SA, NV, C, false, true, P, C, GR, LEAN>{})
                                  : L(SweepKernel<SA, NV, S, false, true, P, S, GR, LEAN>{});
      return c ? L(SweepKernel<SB, NV, C, false, true, P, C, GR, LEAN>{})
               : L(SweepKernel<SB, NV, S, false, true, P, S, GR, LEAN>{});
    }
  }
  if (a.shape == SA) {
    if (!a.full) {  // partial A windows (sharded tails below bit 12): runtime masks
      if (c) return ksin ? L(SweepKernel<SA, NV, C, true, false, P, C, GR, FMX>{}) : L(SweepKernel<SA, NV, C, false, false, P, C, GR, FMX>{});
      return ksin ? L(SweepKernel<SA, NV, S, true, false, P, S, GR, FMX>{}) : L(SweepKernel<SA, NV, S, false, false, P, S, GR, FMX>{});
    }
    if (c) return ksin ? L(SweepKernel<SA, NV, C, true, true, P, C, GR, FMX>{}) : L(SweepKernel<SA, NV, C, false, true, P, C, GR, FMX>{});
    return ksin ? L(SweepKernel<SA, NV, S, true, true, P, S, GR, FMX>{}) : L(SweepKernel<SA, NV, S, false, true, P, S, GR, FMX>{});
  }
  if (a.full) return c ? L(SweepKernel<SB, NV, C, false, true, P, C, GR, FMX>{}) : L(SweepKernel<SB, NV, S, false, true, P, S, GR, FMX>{});
  return c ? L(SweepKernel<SB, NV, C, false, false, P, C, GR, FMX>{}) : L(SweepKernel<SB, NV, S, false, false, P, S, GR, FMX>{});
}

// merged / bridge instantiations (fast mode; shapes SA / SB of one register family).  Table ops between
// the passes dispatch on the table kind at run time (KSIN = false).
template <int NV, int MODE, int F1, int SA = SH_A2, int SB = SH_B2, int GR = 1, bool STG = false, bool WM = false>
int launch_merged_f1(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  auto L = [&](auto k) { return decltype(k)::launch(ctx, a, g); };
  // every flag a merged / bridge sweep of this kind can carry (run_chain, fused.cu)
  constexpr uint32_t M0 = SF_POST_SCALE | (MODE == SM_BRIDGE ? (uint32_t)(SF_MID_EXPECT | SF_XSUM2 | SF_KEEP_V0)
                                          : NV == 1 ? (uint32_t)SF_MID_PHASE
                                                    : (uint32_t)(SF_XSUM | SF_MID_DINNER | SF_MID_PHASE | SF_XSUM2 |
                                                                 SF_KEEP_V0));
  static_assert(!STG || (NV == 2 && MODE != SM_PLAIN), "the staggered schedule is a merged / bridge bra/ket sweep");
  constexpr uint32_t M = M0 | (STG ? kStagBit : 0u);
  if ((a.flags & ~M0) != 0) return invalid("internal: unexpected flags 0x%x for a merged sweep", a.flags);
  const bool c2 = a.form2 == GF_FACT_C;
  if (a.mirror && a.shape == SA) {  // Z2-reduced half statevector (whole A window only)
    if constexpr (WM) {
      constexpr uint32_t MM = M | kMirBit;
      if (!a.full) return invalid("internal: mirror A sweeps gate the whole window");
      if constexpr (MODE == SM_BRIDGE) return L(SweepKernel<SA, NV, F1, false, true, MODE, F1, GR, MM>{});
      else return c2 ? L(SweepKernel<SA, NV, F1, false, true, MODE, GF_FACT_C, GR, MM>{})
                     : L(SweepKernel<SA, NV, F1, false, true, MODE, GF_FACT_S, GR, MM>{});
    } else {
      return invalid("internal: this sweep family has no mirror (Z2-reduced) A instantiation");
    }
  }
  if constexpr (MODE == SM_BRIDGE) {  // Rx(-2b) then Rx(+2b): the same form
    if (a.shape == SA) return a.full ? L(SweepKernel<SA, NV, F1, false, true, MODE, F1, GR, M>{})
                                        : L(SweepKernel<SA, NV, F1, false, false, MODE, F1, GR, M>{});
    return a.full ? L(SweepKernel<SB, NV, F1, false, true, MODE, F1, GR, M>{})
                  : L(SweepKernel<SB, NV, F1, false, false, MODE, F1, GR, M>{});
  } else {
    if (a.shape == SA) {
      if (a.full) return c2 ? L(SweepKernel<SA, NV, F1, false, true, MODE, GF_FACT_C, GR, M>{})
                            : L(SweepKernel<SA, NV, F1, false, true, MODE, GF_FACT_S, GR, M>{});
      return c2 ? L(SweepKernel<SA, NV, F1, false, false, MODE, GF_FACT_C, GR, M>{})
                : L(SweepKernel<SA, NV, F1, false, false, MODE, GF_FACT_S, GR, M>{});
    }
    if (a.full) return c2 ? L(SweepKernel<SB, NV, F1, false, true, MODE, GF_FACT_C, GR, M>{})
                          : L(SweepKernel<SB, NV, F1, false, true, MODE, GF_FACT_S, GR, M>{});
    return c2 ? L(SweepKernel<SB, NV, F1, false, false, MODE, GF_FACT_C, GR, M>{})
              : L(SweepKernel<SB, NV, F1, false, false, MODE, GF_FACT_S, GR, M>{});
  }
}

// exact-mode instantiations (ascending qubit order, FMA-free): shapes A2X / B2
template <int NV>
int launch_exact(qsb_ctx* ctx, SweepArgs& a, unsigned* g) {
  auto L = [&](auto k) { return decltype(k)::launch(ctx, a, g); };
  if (a.shape == SH_A2X) {
    if (!a.full)
      return a.kind == 0 ? L(SweepKernel<SH_A2X, NV, GF_EXACT, true, false>{})
                         : L(SweepKernel<SH_A2X, NV, GF_EXACT, false, false>{});
    return a.kind == 0 ? L(SweepKernel<SH_A2X, NV, GF_EXACT, true, true>{})
                       : L(SweepKernel<SH_A2X, NV, GF_EXACT, false, true>{});
  }
  return a.full ? L(SweepKernel<SH_B2, NV, GF_EXACT, false, true>{}) : L(SweepKernel<SH_B2, NV, GF_EXACT, false, false>{});
}

}  // namespace sweepk
}  // namespace qsb
