// Bare-I/O ceiling of the checkpointed bra/ket sweep (not part of the library): per
// amplitude it reads the bra and the ket and writes the bra (48 B), with no arithmetic.
//   ldg2 : dst[i] = a[i] + c[i], grid-stride LDG/STG (the DRAM ceiling of a 2:1 read/write mix)
//   A    : 1-D TMA tiles of both vectors (the library's 3-slot ring, 2 slots per tile),
//          LDS both, STG the sum back into the bra          (braket A-window I/O)
//   B    : the same with 5-D TMA boxes (bits 0..2 + 9 bits at glo)  (braket B-window I/O)
// n = 29 (the C3 Z2-reduced statevector: 8 GiB per vector).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o probe_braket tools/probe_braket_io.cu -lcuda
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
__device__ __forceinline__ void stg(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__global__ void k_ldg2(const double2* __restrict__ a, const double2* __restrict__ c, double2* __restrict__ d, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const double2 x = __ldcs(a + i), y = __ldcs(c + i);
    __stcs(d + i, make_double2(x.x + y.x, x.y + y.y));
  }
}

// IS_A: contiguous 4096-amplitude tiles (1-D bulk copies); else 5-D boxes over (bits 0..2,
// bits glo..glo+8) with the tile index on the remaining bits
template <bool IS_A>
__global__ void __launch_bounds__(256, 1) k_braket(const __grid_constant__ CUtensorMap tb,
                                                   const __grid_constant__ CUtensorMap tk, double2* bra,
                                                   const double2* ket, uint64_t ntiles, int glo) {
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
  const uint64_t nseq = 2 * mine;
  const int lowbits = glo - 3;
  auto issue = [&](uint64_t s) {  // sequence s: tile s/2, even = bra, odd = ket
    if (tid != 0 || s >= nseq) return;
    const uint64_t t = blockIdx.x + (s / 2) * gridDim.x;
    const uint32_t slot = (uint32_t)(s % kRing), bar = bars + 8 * slot;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kSlot) : "memory");
    if constexpr (IS_A) {
      const double2* src = (s & 1) ? ket : bra;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       ring + slot * kSlot),
                   "l"(src + (t << kT)), "r"(kSlot), "r"(bar)
                   : "memory");
    } else {
      const int c1 = (int)(t & ((1ull << lowbits) - 1)), c4 = (int)(t >> lowbits);
      asm volatile(
          "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5, %6}], [%7];" ::"r"(ring + slot * kSlot),
          "l"((s & 1) ? &tk : &tb), "r"(0), "r"(c1), "r"(0), "r"(0), "r"(c4), "r"(bar)
          : "memory");
    }
  };
  issue(0);
  issue(1);
  issue(2);
  for (uint64_t k = 0; k < mine; ++k) {
    const uint64_t t = blockIdx.x + k * gridDim.x;
    const uint32_t sb = (uint32_t)((2 * k) % kRing), sk = (uint32_t)((2 * k + 1) % kRing);
    const uint32_t lb = (uint32_t)lane | ((uint32_t)warp << 5);
    double2 v[16];
    mbar_wait(bars + 8 * sb, (uint32_t)(((2 * k) / kRing) & 1));
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = lds(ring + sb * kSlot + (lb | (j << 8)) * 16u);
    mbar_wait(bars + 8 * sk, (uint32_t)(((2 * k + 1) / kRing) & 1));
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const double2 y = lds(ring + sk * kSlot + (lb | (j << 8)) * 16u);
      v[j] = make_double2(v[j].x + y.x, v[j].y + y.y);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    issue(2 * k + 3);
    issue(2 * k + 4);
    const uint64_t base = IS_A ? (t << kT) : ((t & ((1ull << lowbits) - 1)) << 3 | (t >> lowbits) << (glo + 9));
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t l = lb | (j << 8);
      stg(bra + (IS_A ? (base | l) : (base | (l & 7u) | ((uint64_t)(l >> 3) << glo))), v[j]);
    }
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
// 5-D view of a 2^n array of 16-byte amplitudes as the library's B tiles
// (sweep_host.cu encode_b_tile_map): {8 amplitudes of bits 0..2, bits 3..glo-1, 5 + 4
// window bits at glo, the bits above}; a box = one 4096-amplitude tile
static CUtensorMap bmap(const double2* base, int n, int glo) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  CUtensorMap m;
  const cuuint64_t dims[5] = {16, 1ull << (glo - 3), 32, 16, 1ull << (n - glo - 9)};
  const cuuint64_t strides[4] = {128, (1ull << glo) * 16, (1ull << (glo + 5)) * 16, (1ull << (glo + 9)) * 16};
  const cuuint32_t box[5] = {16, 1, 32, 16, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = ((EncodeFn)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("encode failed %d\n", (int)r);
  return m;
}

int main() {
  const int n = 29;
  const uint64_t N = 1ull << n, ntiles = N >> kT;
  double2 *a, *c, *d;
  if (cudaMalloc(&a, N * 16) || cudaMalloc(&c, N * 16) || cudaMalloc(&d, N * 16)) {
    printf("alloc failed\n");
    return 1;
  }
  cudaMemset(a, 0x3f, N * 16);
  cudaMemset(c, 0x3e, N * 16);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = kRing * kSlot + 64;
  cudaFuncSetAttribute(k_braket<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_braket<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int glos[] = {12, 20};
  CUtensorMap tb[2], tk[2];
  for (int i = 0; i < 2; ++i) {
    tb[i] = bmap(a, n, glos[i]);
    tk[i] = bmap(c, n, glos[i]);
  }
  const char* names[] = {"ldg2 (grid-stride, 8 CTAs/SM)", "A tiles, TMA 1-D ring", "B tiles glo=12, TMA 5-D ring",
                         "B tiles glo=20, TMA 5-D ring"};
  for (int mode = 0; mode < 4; ++mode) {
    float best = 1e9f;
    for (int rep = 0; rep < 7; ++rep) {
      cudaEventRecord(e0);
      if (mode == 0) k_ldg2<<<sms * 8, 256>>>(a, c, d, N);
      if (mode == 1) k_braket<true><<<sms, 256, smem>>>(tb[0], tk[0], a, c, ntiles, 12);
      if (mode >= 2) k_braket<false><<<sms, 256, smem>>>(tb[mode - 2], tk[mode - 2], a, c, ntiles, glos[mode - 2]);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("%-32s: %.3f ms  %.1f GB/s of 48 B/amp (%s)\n", names[mode], best, 48.0 * N / (best * 1e-3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
