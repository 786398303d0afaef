// Host side of the fused sweep: kernel dispatch and TMA descriptor encoding.
#include <stdlib.h>
#include <string.h>

#include "sweep.cuh"

namespace qsb {

int launch_sweep_nv1_r5(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_nv1_r4(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_nv1_r3(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_nv2_r4(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_nv2_r4t(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_nv2_r3t(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_nv2_r3(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_exact_nv1(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_exact_nv2(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv1_r4_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv1_r4_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv1_r5_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv1_r5_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv1_r5g_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv1_r5g_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_nv1_r5g(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_bridge(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_bridge_t(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_r3_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_r3_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_t_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_t_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_r3t_c(qsb_ctx* ctx, SweepArgs& a, unsigned* g);
int launch_sweep_m_nv2_r3t_s(qsb_ctx* ctx, SweepArgs& a, unsigned* g);

// plain bra/ket sweeps: staggered on A (bit 0) / B (bit 1) windows (QSB_STAGP; default
// both -- round 2, with the ket read from forward checkpoints and not stored, the
// staggered B sweeps measured 3% faster than lock-step)
static int stagp_mask() {
  const char* e = getenv("QSB_STAGP");
  return e ? atoi(e) : 3;
}
// merged bra/ket sweeps: staggered schedule (default; QSB_STAG=0: lock-step)
static bool stag_enabled() {
  const char* e = getenv("QSB_STAG");
  return e ? atoi(e) != 0 : true;
}

int launch_sweep(qsb_ctx* ctx, int nv, bool exact, SweepArgs& a, unsigned* gout) {
  if (a.mode != SM_PLAIN) {
    const int r = shape_r(a.shape);
    if (exact || a.form == GF_EXACT || a.shape != pick_shape(false, shape_is_a(a.shape), r) ||
        (nv == 1 && r == 3) || (nv == 2 && r == 5) || (a.mode == SM_BRIDGE && r != 4))
      return invalid("internal: merged sweeps are fast-mode; R=4 or R=5 (NV=1) / R=3 (NV=2) shapes");
    if (a.mode == SM_BRIDGE) {
      if (nv != 2) return invalid("internal: bridge needs nv=2");
      return stag_enabled() ? launch_sweep_bridge_t(ctx, a, gout) : launch_sweep_bridge(ctx, a, gout);
    }
    const bool c = a.form == GF_FACT_C;
    if (nv == 1) {
      if (r == 5 && a.groups == 2) return c ? launch_sweep_m_nv1_r5g_c(ctx, a, gout) : launch_sweep_m_nv1_r5g_s(ctx, a, gout);
      if (r == 5) return c ? launch_sweep_m_nv1_r5_c(ctx, a, gout) : launch_sweep_m_nv1_r5_s(ctx, a, gout);
      return c ? launch_sweep_m_nv1_r4_c(ctx, a, gout) : launch_sweep_m_nv1_r4_s(ctx, a, gout);
    }
    if (r == 3) {
      if (stag_enabled()) return c ? launch_sweep_m_nv2_r3t_c(ctx, a, gout) : launch_sweep_m_nv2_r3t_s(ctx, a, gout);
      return c ? launch_sweep_m_nv2_r3_c(ctx, a, gout) : launch_sweep_m_nv2_r3_s(ctx, a, gout);
    }
    if (stag_enabled()) return c ? launch_sweep_m_nv2_t_c(ctx, a, gout) : launch_sweep_m_nv2_t_s(ctx, a, gout);
    return c ? launch_sweep_m_nv2_c(ctx, a, gout) : launch_sweep_m_nv2_s(ctx, a, gout);
  }
  if (exact || a.form == GF_EXACT) return nv == 1 ? launch_sweep_exact_nv1(ctx, a, gout) : launch_sweep_exact_nv2(ctx, a, gout);
  const int r = shape_r(a.shape);
  if (nv == 1 && r == 5 && a.groups == 2) return launch_sweep_nv1_r5g(ctx, a, gout);
  if (nv == 1) return r == 5 ? launch_sweep_nv1_r5(ctx, a, gout) : r == 4 ? launch_sweep_nv1_r4(ctx, a, gout)
                                                                           : launch_sweep_nv1_r3(ctx, a, gout);
  if (r == 5) return invalid("internal: no R=5 bra/ket sweep");
  if (stagp_mask() & (shape_is_a(a.shape) ? 1 : 2)) return r == 4 ? launch_sweep_nv2_r4t(ctx, a, gout) : launch_sweep_nv2_r3t(ctx, a, gout);
  return r == 4 ? launch_sweep_nv2_r4(ctx, a, gout) : launch_sweep_nv2_r3(ctx, a, gout);
}

}  // namespace qsb

extern "C" int qsb_has_variants(void) {
#ifdef QSB_VARIANTS
  return 1;
#else
  return 0;
#endif
}

namespace qsb {

int sweep_grid(qsb_ctx* ctx, int nv, bool exact, uint64_t ntiles, unsigned* g) {
  // every shape runs one persistent CTA per SM (the ring takes ~220 KB of smem)
  (void)nv;
  (void)exact;
  *g = (unsigned)(ntiles < (uint64_t)ctx->num_sms ? ntiles : (uint64_t)ctx->num_sms);
  return QSB_OK;
}

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static const EncodeTiledFn fn = [] {  // thread-safe one-time lookup
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return (EncodeTiledFn)p;
    return (EncodeTiledFn) nullptr;
  }();
  return fn;
}
}  // namespace

// B tile: local bits 0..2 -> global 0..2 (8 amplitudes = 16 doubles, 128 B), local
// 3..7 -> glo..glo+4, local 8..11 -> glo+5..glo+8.  As a 5-D tensor of doubles
// (innermost first): {16, 2^(glo-3), 32, 16, 2^(n-glo-9)}; box {16, 1, 32, 16, 1}
// lands one 64 KB tile in local-index order.
int encode_b_tile_map(CUtensorMap* map, const double2* base, int n, int glo) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return invalid("cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (glo < 3 || n - glo - 9 < 0) return invalid("internal: bad B tile geometry n=%d glo=%d", n, glo);
  const cuuint64_t dims[5] = {16, 1ull << (glo - 3), 32, 16, 1ull << (n - glo - 9)};
  const cuuint64_t strides[4] = {128, (1ull << glo) * 16, (1ull << (glo + 5)) * 16, (1ull << (glo + 9)) * 16};
  const cuuint32_t box[5] = {16, 1, 32, 16, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return invalid("cuTensorMapEncodeTiled failed (%d) for n=%d glo=%d", (int)r, n, glo);
  return QSB_OK;
}

// Compact index of the same B tile.  u16: inner 8 entries (16 B) = local bits 0..2,
// natural local order in smem.  u8: the inner box must be 16 B, so it covers global
// bits 0..3 — bit 3 is the lowest tile-index bit (glo >= 4 for every B sweep); the
// tile's 8 entries sit at ((l >> 3) << 4) + 8 * (tile & 1) + (l & 7) in smem.
int encode_b_cidx_map(CUtensorMap* map, const void* base, int esz, int n, int glo) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return invalid("cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (glo < 4 || n - glo - 9 < 0) return invalid("internal: bad B index geometry n=%d glo=%d", n, glo);
  CUresult r;
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  if (esz == 2) {
    const cuuint64_t dims[5] = {8, 1ull << (glo - 3), 32, 16, 1ull << (n - glo - 9)};
    const cuuint64_t strides[4] = {16, (1ull << glo) * 2, (1ull << (glo + 5)) * 2, (1ull << (glo + 9)) * 2};
    const cuuint32_t box[5] = {8, 1, 32, 16, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT16, 5, (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[5] = {16, 1ull << (glo - 4), 32, 16, 1ull << (n - glo - 9)};
    const cuuint64_t strides[4] = {16, 1ull << glo, 1ull << (glo + 5), 1ull << (glo + 9)};
    const cuuint32_t box[5] = {16, 1, 32, 16, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 5, (void*)base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return invalid("cuTensorMapEncodeTiled (index) failed (%d) n=%d glo=%d", (int)r, n, glo);
  return QSB_OK;
}

int encode_b_f64_map(CUtensorMap* map, const double* base, int n, int glo) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return invalid("cuTensorMapEncodeTiled unavailable (driver too old?)");
  if (glo < 3 || n - glo - 9 < 0) return invalid("internal: bad B table geometry n=%d glo=%d", n, glo);
  const cuuint64_t dims[5] = {8, 1ull << (glo - 3), 32, 16, 1ull << (n - glo - 9)};
  const cuuint64_t strides[4] = {64, (1ull << glo) * 8, (1ull << (glo + 5)) * 8, (1ull << (glo + 9)) * 8};
  const cuuint32_t box[5] = {8, 1, 32, 16, 1};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, (void*)base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return invalid("cuTensorMapEncodeTiled (fp64 table) failed (%d) n=%d glo=%d", (int)r, n, glo);
  return QSB_OK;
}

}  // namespace qsb
