// Streaming-structure probe (not part of the library): how fast can a persistent
// one-CTA-per-SM kernel stream a 16 GiB complex128 array HBM -> smem -> registers ->
// HBM with the sweep kernel's data movement, without the gate arithmetic?
//   mode 0: TMA 1-D tile load (3-slot ring) -> LDS -> STG            (the sweep's I/O)
//   mode 1: mode 0 + 2 swizzled smem exchanges per tile               (+ sweep's smem)
//   mode 2: TMA load -> LDS -> STS back into the slot -> TMA 1-D store (bulk store)
//   mode 3: plain LDG.128 -> STG.128 grid-stride copy                 (no smem)
//   mode 5/6: B tile (global bits 0..2 + 9 bits at glo = 12 / 21) via a 5-D TMA box,
//           strided STG, no arithmetic                                (B-sweep I/O)
//   mode 4: the sweep's A-window work: 3 phase maps, 2 exchanges, 4 gate levels each
//           (factored Rx butterflies, 4 DFMA per pair), post scale     (= k_sweep NV=1)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe tools/probe_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

constexpr int kT = 12, kTile = 1 << kT, kSlot = kTile * 16, kRing = 3;

__device__ __forceinline__ double2 lds(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void stg(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__host__ __device__ constexpr uint32_t swz(uint32_t x) { return x ^ (((x >> 3) ^ (x >> 6) ^ (x >> 9) ^ (x >> 12)) & 7u); }

struct Map {
  int lanes[5], warps[3], reg;
};
__host__ __device__ constexpr Map map_of(int p) {
  return p == 0 ? Map{{0, 1, 2, 3, 4}, {5, 6, 7}, 8} : p == 1 ? Map{{4, 5, 6, 7, 8}, {9, 10, 11}, 0} : Map{{0, 1, 2, 3, 8}, {9, 10, 11}, 4};
}
__device__ __forceinline__ uint32_t mbase(const Map& m, int lane, int warp) {
  uint32_t l = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b) l |= (uint32_t)((lane >> b) & 1) << m.lanes[b];
#pragma unroll
  for (int b = 0; b < 3; ++b) l |= (uint32_t)((warp >> b) & 1) << m.warps[b];
  return l;
}
__device__ __forceinline__ void bfly(double2& t, double2& u, double gb) {
  const double2 n0 = make_double2(fma(gb, u.y, t.x), fma(-gb, u.x, t.y));
  const double2 n1 = make_double2(fma(gb, t.y, u.x), fma(-gb, t.x, u.y));
  t = n0;
  u = n1;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k_stream(const double2* __restrict__ src, double2* __restrict__ dst,
                                                    uint64_t ntiles, double scale) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bars = ring + kRing * kSlot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](uint64_t k) {
    if (tid != 0 || k >= mine) return;
    const uint64_t t = blockIdx.x + k * gridDim.x;
    const uint32_t slot = (uint32_t)(k % kRing), bar = bars + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlot) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ring + slot * kSlot),
                 "l"(src + (t << kT)), "r"(kSlot), "r"(bar)
                 : "memory");
  };
  issue(0);
  issue(1);
  for (uint64_t k = 0; k < mine; ++k) {
    const uint64_t t = blockIdx.x + k * gridDim.x;
    if (MODE != 2) issue(k + 2);
    mbar_wait(bars + 8 * (uint32_t)(k % kRing), (uint32_t)((k / kRing) & 1));
    const uint32_t slot = ring + (uint32_t)(k % kRing) * kSlot;
    // natural map: lanes = bits 0..4, warps = bits 5..7, registers = bits 8..11
    const uint32_t lb = (uint32_t)lane | ((uint32_t)warp << 5);
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = lds(slot + (lb | (j << 8)) * 16u);
    if (MODE == 1) {
      // two exchanges: regs <-> bits 0..3, then back (same traffic as the sweep's)
      const uint32_t lb1 = ((uint32_t)lane << 4) | ((uint32_t)(warp & 1) << 9) | ((uint32_t)(warp >> 1) << 10);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t a0 = e == 0 ? lb : lb1, a1 = e == 0 ? lb1 : lb;
        const int r0 = e == 0 ? 8 : 0, r1 = e == 0 ? 0 : 8;
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; ++j) sts(slot + swz(a0 | (j << r0)) * 16u, v[j]);
        __syncthreads();
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = lds(slot + swz(a1 | (j << r1)) * 16u);
      }
    }
    uint32_t lout = lb;
    int rout = 8;
    if (MODE == 4) {
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const Map P = map_of(p);
        if (p > 0) {
          const Map Q = map_of(p - 1);
          const uint32_t qb = mbase(Q, lane, warp), pb = mbase(P, lane, warp);
          __syncthreads();
#pragma unroll
          for (int j = 0; j < 16; ++j) sts(slot + swz(qb | (j << Q.reg)) * 16u, v[j]);
          __syncthreads();
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = lds(slot + swz(pb | (j << P.reg)) * 16u);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (!(j & (1 << b))) bfly(v[j], v[j | (1 << b)], scale * 0.25);
      }
      lout = mbase(map_of(2), lane, warp);
      rout = 4;
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = make_double2(v[j].x * scale, v[j].y * scale);
    if (MODE == 2) {
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) sts(slot + (lb | (j << 8)) * 16u, v[j]);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + (t << kT)), "r"(slot),
                     "r"(kSlot)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // the slot is refilled two tiles later: allow one store group in flight
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
      __syncthreads();
      issue(k + 2);  // into slot (k+2)%3 == (k-1)%3, whose store was waited for above
    } else {
      double2* d = dst + (t << kT);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) stg(d + (lout | (j << rout)), v[j]);
      __syncthreads();
    }
  }
  if (MODE == 2 && tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// B tile with L contiguous low bits (runs of 2^L amplitudes) and 12-L window bits at
// glo; SC: store contiguous (tile order) instead of back to the strided positions
template <int L, bool SC, int CL = 1>
__global__ void __launch_bounds__(256, 1) k_btile(const __grid_constant__ CUtensorMap tm, double2* __restrict__ dst,
                                                  uint64_t ntiles, int glo, double scale) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bars = ring + kRing * kSlot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int lowbits = glo - L;
  auto issue = [&](uint64_t k) {
    if (tid != 0 || k >= mine) return;
    const uint64_t t = blockIdx.x + k * gridDim.x;
    const uint32_t slot = (uint32_t)(k % kRing), bar = bars + 8 * slot;
    const int c1 = (int)(t & ((1ull << lowbits) - 1)), c4 = (int)(t >> lowbits);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlot) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(ring + slot * kSlot),
        "l"(&tm), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(c4), "r"(bar)
        : "memory");
  };
  issue(0);
  issue(1);
  for (uint64_t k = 0; k < mine; ++k) {
    const uint64_t t = blockIdx.x + k * gridDim.x;
    issue(k + 2);
    mbar_wait(bars + 8 * (uint32_t)(k % kRing), (uint32_t)((k / kRing) & 1));
    const uint32_t slot = ring + (uint32_t)(k % kRing) * kSlot;
    const uint32_t lb = (uint32_t)lane | ((uint32_t)warp << 5);
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = lds(slot + (lb | (j << 8)) * 16u);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = make_double2(v[j].x * scale, v[j].y * scale);
    const uint64_t base = (t & ((1ull << lowbits) - 1)) << L | (t >> lowbits) << (glo + 12 - L);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t l = lb | (j << 8);
      if (SC) stg(dst + ((t << kT) | l), v[j]);
      else stg(dst + (base | (l & ((1u << L) - 1)) | ((uint64_t)(l >> L) << glo)), v[j]);
    }
    __syncthreads();
    if (CL > 1) {  // keep the cluster's CTAs (adjacent 128 B runs) in lockstep
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
  }
}

// Generalised A-window probe: NV vectors (2: bra/ket with slots 2k%3 / (2k+1)%3 as in
// the library), MERGED = two gate passes (phases 0,1,2 then 2,1,0), XSUM = bra/ket
// contraction after each phase's gates.
template <int NV, bool MERGED, int XSUM, int MID = 0, bool STAG = false>
__global__ void __launch_bounds__(256, 1) k_probe(double2* __restrict__ v0g, double2* __restrict__ v1g, uint64_t ntiles,
                                                   double gb, double* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // MID: the diagonal between the passes as the library does it for a u8 table: index
  // byte from a 4 KB tile in smem, (cos, sin) from a 41-entry LUT in smem, <bra|C|ket>
  // accumulation, complex multiply of both vectors
  uint8_t* cidx = smem + kRing * kSlot + 64;
  double2* lut = (double2*)(cidx + kTile);
  for (int i = threadIdx.x; i < kTile; i += 256) cidx[i] = (uint8_t)((i * 2654435761u) >> 26) % 41;
  for (int i = threadIdx.x; i < 64; i += 256) lut[i] = make_double2(cos(0.1 * i), sin(0.1 * i));
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bars = ring + kRing * kSlot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const uint64_t nseq = mine * NV;
  auto issue = [&](uint64_t sq) {
    if (tid != 0 || sq >= nseq) return;
    const uint64_t k = sq / NV;
    const int q = NV == 2 ? (int)((sq & 1) ^ 1) : 0;
    const uint64_t t = blockIdx.x + k * gridDim.x;
    const uint32_t slot = (uint32_t)(sq % kRing), bar = bars + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlot) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ring + slot * kSlot),
                 "l"((q == 0 ? v0g : v1g) + (t << kT)), "r"(kSlot), "r"(bar)
                 : "memory");
  };
  auto wait = [&](uint64_t sq) { mbar_wait(bars + 8 * (uint32_t)(sq % kRing), (uint32_t)((sq / kRing) & 1)); };
  double acc = 0.0;
  issue(0);
  issue(1);
  if (NV == 2) issue(2);
  for (uint64_t k = 0; k < mine; ++k) {
    const uint64_t t = blockIdx.x + k * gridDim.x;
    uint32_t sk, sb = 0;
    double2 v[NV][16];
    const uint32_t lb0 = mbase(map_of(0), lane, warp);
    if (NV == 1) {
      issue(k + 2);
      wait(k);
      sk = ring + (uint32_t)(k % kRing) * kSlot;
    } else {
      sb = ring + (uint32_t)((2 * k) % kRing) * kSlot;
      sk = ring + (uint32_t)((2 * k + 1) % kRing) * kSlot;
      wait(2 * k);
#pragma unroll
      for (int j = 0; j < 16; ++j) v[NV - 1][j] = lds(sb + (lb0 | (j << 8)) * 16u);
      wait(2 * k + 1);
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) v[0][j] = lds(sk + (lb0 | (j << 8)) * 16u);
    uint32_t cpk[4] = {0, 0, 0, 0};
    if (MID == 2) {  // prefetch the mid-op index bytes now, packed 4 per register
      const uint32_t lm = mbase(map_of(2), lane, warp);
#pragma unroll
      for (int j = 0; j < 16; ++j) cpk[j >> 2] |= (uint32_t)cidx[lm | (j << map_of(2).reg)] << (8 * (j & 3));
    }
    auto exch = [&](int qi, int pi) {
      const Map Q = map_of(qi), P = map_of(pi);
      const uint32_t qb = mbase(Q, lane, warp), pb = mbase(P, lane, warp);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int j = 0; j < 16; ++j) sts((q == 0 ? sk : sb) + swz(qb | (j << Q.reg)) * 16u, v[q][j]);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int j = 0; j < 16; ++j) v[q][j] = lds((q == 0 ? sk : sb) + swz(pb | (j << P.reg)) * 16u);
    };
    auto gates = [&](int q0 = 0, int q1 = NV, bool xs = true) {
      double x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (!(j & (1 << b))) {
#pragma unroll
            for (int q = 0; q < NV; ++q)
              if (q >= q0 && q < q1) bfly(v[q][j], v[q][j | (1 << b)], gb);
          }
      if (XSUM && NV == 2 && xs) {  // after the gates (X_j commutes with the layer)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (!(j & (1 << b))) {
              const int k2 = j | (1 << b);
              const int sl = XSUM == 1 ? 0 : XSUM == 2 ? (j & 3) : ((j & ((1 << b) - 1)) | ((j >> (b + 1)) << b));
              x[sl] = fma(v[1][j].x, v[0][k2].y, x[sl]);
              x[sl] = fma(-v[1][j].y, v[0][k2].x, x[sl]);
              x[sl] = fma(v[1][k2].x, v[0][j].y, x[sl]);
              x[sl] = fma(-v[1][k2].y, v[0][j].x, x[sl]);
            }
#pragma unroll
        for (int i = 0; i < 8; ++i) acc += x[i];
      }
    };
    // staggered exchange (NV=2): the ket's loads and gates overlap the bra's stores
    auto xg = [&](int qi, int pi) {
      if (!STAG || NV != 2) {
        exch(qi, pi);
        gates();
        return;
      }
      const Map Q = map_of(qi), P = map_of(pi);
      const uint32_t qb = mbase(Q, lane, warp), pb = mbase(P, lane, warp);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) sts(sk + swz(qb | (j << Q.reg)) * 16u, v[0][j]);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[0][j] = lds(sk + swz(pb | (j << P.reg)) * 16u);
#pragma unroll
      for (int j = 0; j < 16; ++j) sts(sb + swz(qb | (j << Q.reg)) * 16u, v[NV - 1][j]);
      gates(0, 1, false);
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 16; ++j) v[NV - 1][j] = lds(sb + swz(pb | (j << P.reg)) * 16u);
      gates(1, 2, true);
    };
    gates();
    xg(0, 1);
    xg(1, 2);
    int last = 2;
    if (MERGED && MID) {
      const uint32_t lm = mbase(map_of(2), lane, warp);
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t l = lm | (j << map_of(2).reg);
        const int ci = MID == 2 ? (int)((cpk[j >> 2] >> (8 * (j & 3))) & 0xffu) : (int)cidx[l];
        const double tv = -40.0 + (double)ci;
        if (NV == 2) acc = fma(tv, v[1][j].x * v[0][j].y - v[1][j].y * v[0][j].x, acc);
        const double2 f = lut[ci];
#pragma unroll
        for (int q = 0; q < NV; ++q)
          v[q][j] = make_double2(fma(v[q][j].x, f.x, -v[q][j].y * f.y), fma(v[q][j].x, f.y, v[q][j].y * f.x));
      }
    }
    if (MERGED) {
      xg(2, 1);
      xg(1, 0);
      last = 0;
    }
    if (NV == 2) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      issue(2 * k + 3);
      issue(2 * k + 4);
    } else {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    const Map L = map_of(last);
    const uint32_t lo = mbase(L, lane, warp);
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double2* d = (q == 0 ? v0g : v1g) + (t << kT);
#pragma unroll
      for (int j = 0; j < 16; ++j) stg(d + (lo | (j << L.reg)), v[q][j]);
    }
    if (NV == 1) __syncthreads();
  }
  if (acc == 12345.0) out[0] = acc;
}

// B tile whose 9 window bits are two groups: glo..glo+4 and the top four bits n-4..n-1
__global__ void __launch_bounds__(256, 1) k_bsplit(const __grid_constant__ CUtensorMap tm, double2* __restrict__ dst,
                                                   uint64_t ntiles, int glo, int n, double scale) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t ring = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t bars = ring + kRing * kSlot;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kRing; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bars + 8 * s));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint64_t mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const int lowbits = glo - 3, midbits = n - 4 - (glo + 5);
  auto issue = [&](uint64_t k) {
    if (tid != 0 || k >= mine) return;
    const uint64_t t = blockIdx.x + k * gridDim.x;
    const uint32_t slot = (uint32_t)(k % kRing), bar = bars + 8 * slot;
    const int c1 = (int)(t & ((1ull << lowbits) - 1)), c3 = (int)(t >> lowbits);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlot) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, "
        "%6}], [%7];" ::"r"(ring + slot * kSlot),
        "l"(&tm), "r"(0), "r"(c1), "r"(0), "r"(c3), "r"(0), "r"(bar)
        : "memory");
  };
  issue(0);
  issue(1);
  for (uint64_t k = 0; k < mine; ++k) {
    const uint64_t t = blockIdx.x + k * gridDim.x;
    issue(k + 2);
    mbar_wait(bars + 8 * (uint32_t)(k % kRing), (uint32_t)((k / kRing) & 1));
    const uint32_t slot = ring + (uint32_t)(k % kRing) * kSlot;
    const uint32_t lb = (uint32_t)lane | ((uint32_t)warp << 5);
    double2 v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = lds(slot + (lb | (j << 8)) * 16u);
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = make_double2(v[j].x * scale, v[j].y * scale);
    const uint64_t base = ((t & ((1ull << lowbits) - 1)) << 3) | ((t >> lowbits) << (glo + 5));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t l = lb | (j << 8);
      const uint64_t gidx = base | (l & 7) | ((uint64_t)((l >> 3) & 31) << glo) | ((uint64_t)(l >> 8) << (n - 4));
      stg(dst + gidx, v[j]);
    }
    __syncthreads();
  }
  (void)midbits;
}

__global__ void k_ldg(const double2* __restrict__ src, double2* __restrict__ dst, uint64_t n, double scale) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(src + i);
    __stcs(dst + i, make_double2(v.x * scale, v.y * scale));
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap bmap(const double2* base, int n, int glo, int L,
                        CUtensorMapL2promotion promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap m;
  const int H = 12 - L;  // window bits: 5 + (H - 5)
  const cuuint64_t dims[5] = {2ull << L, 1ull << (glo - L), 32, 1ull << (H - 5), 1ull << (n - glo - H)};
  const cuuint64_t strides[4] = {(1ull << L) * 16, (1ull << glo) * 16, (1ull << (glo + 5)) * 16, (1ull << (glo + H)) * 16};
  const cuuint32_t box[5] = {2u << L, 1, 32, 1u << (H - 5), 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = ((EncodeFn)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d (L=%d glo=%d)\n", (int)r, L, glo);
  return m;
}

static CUtensorMap bmap_split(const double2* base, int n, int glo) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap m;
  // {bits 0-2 (16 doubles), tile-low glo-3 bits, 5 window bits, tile-mid bits, 4 top window bits}
  const int mid = n - 4 - (glo + 5);
  const cuuint64_t dims[5] = {16, 1ull << (glo - 3), 32, 1ull << mid, 16};
  const cuuint64_t strides[4] = {128, (1ull << glo) * 16, (1ull << (glo + 5)) * 16, (1ull << (n - 4)) * 16};
  const cuuint32_t box[5] = {16, 1, 32, 1, 16};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = ((EncodeFn)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("split encode failed %d\n", (int)r);
  return m;
}

int main() {
  const int n = 30;
  const uint64_t N = 1ull << n;
  double2 *a, *b;
  if (cudaMalloc(&a, N * 16) || cudaMalloc(&b, N * 16)) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 0x3f, N * 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = kRing * kSlot + 64 + kTile + 64 * 16;
  cudaFuncSetAttribute(k_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_stream<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_btile<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_btile<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_btile<4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_btile<5, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_btile<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const CUtensorMap m12 = bmap(a, n, 12, 3), m21 = bmap(a, n, 21, 3), m4 = bmap(a, n, 18, 4), m5 = bmap(a, n, 18, 5),
                    m2 = bmap(a, n, 18, 2);
  const CUtensorMap mp0 = bmap(a, n, 21, 3, CU_TENSOR_MAP_L2_PROMOTION_NONE),
                    mp1 = bmap(a, n, 21, 3, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const uint64_t ntiles = N >> kT;
  const char* names[] = {"tma1d+stg", "tma1d+2exch+stg", "tma1d+tma-store", "ldg/stg", "A-window full sweep work",
                         "B L=3 glo=12", "B L=3 glo=21", "B L=3 glo=21, contiguous store", "B L=4 glo=18",
                         "B L=5 glo=18", "B L=2 glo=18", "B L=3 glo=21 promo none", "B L=3 glo=21 promo 128",
                         "B L=3 glo=21 2x grid (2 CTA/SM? no)", "B L=3 glo=21 cluster-2 lockstep",
                         "B L=3 glo=21 cluster-4 lockstep", "B L=3 glo=12 cluster-2 lockstep"};
  double* dout;
  cudaMalloc(&dout, 64);
  auto setp = [&](auto k) { cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); };
  setp(k_probe<1, false, 0>);
  setp(k_probe<1, true, 0>);
  setp(k_probe<2, false, 0>);
  setp(k_probe<2, false, 1>);
  setp(k_probe<2, false, 2>);
  setp(k_probe<2, false, 3>);
  setp(k_probe<2, true, 0>);
  setp(k_probe<2, true, 3>);
  setp(k_probe<2, true, 3, 1>);
  setp(k_probe<1, true, 0, 1>);
  setp(k_probe<2, true, 3, 2>);
  setp(k_probe<1, true, 0, 2>);
  setp(k_probe<2, true, 3, 1, true>);
  setp(k_probe<2, false, 3, 0, true>);
  const char* pnames[] = {"probe A NV1 plain", "probe A NV1 merged", "probe A NV2 plain", "probe A NV2 plain+xsum(1 acc)",
                          "probe A NV2 plain+xsum(4 acc)", "probe A NV2 plain+xsum(8 acc)", "probe A NV2 merged",
                          "probe A NV2 merged+xsum(8 acc)", "probe A NV2 merged+xsum+mid", "probe A NV1 merged+mid", "probe A NV2 merged+xsum+mid(pf)", "probe A NV1 merged+mid(pf)",
                          "probe A NV2 merged+xsum+mid STAGGERED", "probe A NV2 plain+xsum STAGGERED"};
  const double pbytes[] = {32.0, 32.0, 64.0, 64.0, 64.0, 64.0, 64.0, 64.0, 64.0, 32.0, 64.0, 32.0, 64.0, 64.0};
  for (int m = 0; m < 14; ++m) {
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (m == 0) k_probe<1, false, 0><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 1) k_probe<1, true, 0><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 2) k_probe<2, false, 0><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 3) k_probe<2, false, 1><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 4) k_probe<2, false, 2><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 5) k_probe<2, false, 3><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 6) k_probe<2, true, 0><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 7) k_probe<2, true, 3><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 8) k_probe<2, true, 3, 1><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 9) k_probe<1, true, 0, 1><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 10) k_probe<2, true, 3, 2><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 11) k_probe<1, true, 0, 2><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 12) k_probe<2, true, 3, 1, true><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      if (m == 13) k_probe<2, false, 3, 0, true><<<sms, 256, smem>>>(a, b, ntiles, 0.3, dout);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-34s: %.3f ms  %.1f GB/s  (%s)\n", pnames[m], best, pbytes[m] * N / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  cudaFuncSetAttribute(k_btile<3, false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_btile<3, false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 16; ++mode) {
    if (mode == 12) continue;
    float best = 1e9f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k_stream<0><<<sms, 256, smem>>>(a, b, ntiles, 1.0);
      if (mode == 1) k_stream<1><<<sms, 256, smem>>>(a, b, ntiles, 1.0);
      if (mode == 2) k_stream<2><<<sms, 256, smem>>>(a, b, ntiles, 1.0);
      if (mode == 3) k_ldg<<<sms * 8, 256>>>(a, b, N, 1.0);
      if (mode == 4) k_stream<4><<<sms, 256, smem>>>(a, b, ntiles, 1.0);
      if (mode == 5) k_btile<3, false><<<sms, 256, smem>>>(m12, b, ntiles, 12, 1.0);
      if (mode == 6) k_btile<3, false><<<sms, 256, smem>>>(m21, b, ntiles, 21, 1.0);
      if (mode == 7) k_btile<3, true><<<sms, 256, smem>>>(m21, b, ntiles, 21, 1.0);
      if (mode == 8) k_btile<4, false><<<sms, 256, smem>>>(m4, b, ntiles, 18, 1.0);
      if (mode == 9) k_btile<5, false><<<sms, 256, smem>>>(m5, b, ntiles, 18, 1.0);
      if (mode == 10) k_btile<2, false><<<sms, 256, smem>>>(m2, b, ntiles, 18, 1.0);
      if (mode == 11) k_btile<3, false><<<sms, 256, smem>>>(mp0, b, ntiles, 21, 1.0);
      if (mode == 12) k_btile<3, false><<<sms, 256, smem>>>(mp1, b, ntiles, 21, 1.0);
      if (mode == 13 || mode == 14 || mode == 15) {
        const int cl = mode == 13 ? 2 : mode == 14 ? 4 : 2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(sms);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const CUtensorMap& mm = mode == 15 ? m12 : m21;
        const int gl = mode == 15 ? 12 : 21;
        if (cl == 2) cudaLaunchKernelEx(&cfg, k_btile<3, false, 2>, mm, b, ntiles, gl, 1.0);
        else cudaLaunchKernelEx(&cfg, k_btile<3, false, 4>, mm, b, ntiles, gl, 1.0);
      }
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("mode %d %-34s: %.3f ms  %.1f GB/s  (%s)\n", mode, names[mode], best, 32.0 * N / (best * 1e-3) / 1e9, cudaGetErrorString(err));
  }
  // ---- B tiles (L=3) with clusters of CL CTAs kept in lockstep, for several window positions
  cudaFuncSetAttribute(k_btile<3, false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_btile<3, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  // reference output (no cluster) for a correctness check
  double2* ref;
  cudaMalloc(&ref, N * 16);
  const int glos[] = {12, 16, 21};
  for (int gi = 0; gi < 3; ++gi) {
    const int gl = glos[gi];
    const CUtensorMap mm = bmap(a, n, gl, 3);
    k_btile<3, false, 1><<<sms, 256, smem>>>(mm, ref, ntiles, gl, 1.0);
    cudaDeviceSynchronize();
    for (int cl : {1, 2, 4, 8}) {
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl == 8 ? 144 : sms);
        cfg.blockDim = dim3(256);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaMemset(b, 0, N * 16);
        cudaEventRecord(e0);
        if (cl == 1) cudaLaunchKernelEx(&cfg, k_btile<3, false, 1>, mm, b, ntiles, gl, 1.0);
        if (cl == 2) cudaLaunchKernelEx(&cfg, k_btile<3, false, 2>, mm, b, ntiles, gl, 1.0);
        if (cl == 4) cudaLaunchKernelEx(&cfg, k_btile<3, false, 4>, mm, b, ntiles, gl, 1.0);
        if (cl == 8) cudaLaunchKernelEx(&cfg, k_btile<3, false, 8>, mm, b, ntiles, gl, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      // compare b with ref on a sample
      static double2 hb[4096], hr[4096];
      bool same = true;
      const uint64_t offs[3] = {0ull, N / 3, N - 4096};
      for (uint64_t off : offs) {
        cudaMemcpy(hb, b + off, sizeof(hb), cudaMemcpyDeviceToHost);
        cudaMemcpy(hr, ref + off, sizeof(hr), cudaMemcpyDeviceToHost);
        for (int q = 0; q < 4096; ++q) same = same && hb[q].x == hr[q].x && hb[q].y == hr[q].y;
      }
      printf("B L=3 glo=%2d cluster %d: %.3f ms  %.1f GB/s  same=%d (%s)\n", gl, cl, best, 32.0 * N / (best * 1e-3) / 1e9,
             (int)same, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // ---- TLB test at n=29: contiguous top window (bits 20..28: 512 distinct 2 MB pages per tile)
  // vs a split window (bits 12..16 + 25..28: 16 pages per tile), same bytes
  {
    const int n2 = 29;
    const uint64_t N2 = 1ull << n2, nt2 = N2 >> kT;
    cudaFuncSetAttribute(k_bsplit, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const CUtensorMap mc = bmap(a, n2, 20, 3), ms = bmap_split(a, n2, 12);
    for (int v = 0; v < 2; ++v) {
      float best = 1e9f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (v == 0) k_btile<3, false><<<sms, 256, smem>>>(mc, b, nt2, 20, 1.0);
        else k_bsplit<<<sms, 256, smem>>>(ms, b, nt2, 12, n2, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms_;
        cudaEventElapsedTime(&ms_, e0, e1);
        if (ms_ < best) best = ms_;
      }
      printf("n=29 B L=3 %s: %.3f ms  %.1f GB/s (%s)\n", v == 0 ? "window 20..28 (512 pages/tile)" : "window 12..16+25..28 (16 pages)",
             best, 32.0 * N2 / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
