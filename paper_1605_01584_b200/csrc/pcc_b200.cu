// pcc_b200.cu -- C ABI (include/pcc_b200.h) over the sm_100a kernels.
//
// Host-side argument checking mirrors the reference's errors: anything the
// reference rejects with ValueError (bad ranges, sizes) returns PCC_EINVAL
// with a message; CUDA failures return PCC_ECUDA.  Nothing here falls back
// to a CPU path.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/pcc_b200.h"
#include "normalize.cuh"
#include "exact.cuh"
#include "split.cuh"
#include "syrk.cuh"
#include "verify.cuh"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char *what) {
  return fail(PCC_ECUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define PCC_CUDA(call, what)                      \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

struct DeviceConfig {
  bool ready = false;
  int sm_count = 0;
  int cc_major = 0, cc_minor = 0;
  int max_smem_optin = 0;
  int syrk_ctas_per_sm = 0;  // production contraction, grouped order
  int syrk_id_ctas = 0;      // the same kernel in bijection id order (PCC_SYRK_ORDER=id)
  int quad_ctas = 0;
  int exact_ctas = 0;
  int split_ctas = 0;
  int norm_regs[3] = {0, 0, 0};  // registers of normalize_rows_smem_kernel<256, MODE>
#ifdef PCC_TUNING_VARIANTS
  int variant_ctas[16] = {0};
#endif
  size_t total_mem = 0;
};

constexpr int kMaxDevices = 64;
DeviceConfig g_dev[kMaxDevices];
std::mutex g_dev_mu;

// Production contraction shape: TMA + mbarrier ring, 8 warps 64x32, BK 16 x 6
// stages, stage-level fragments, grouped tile order.  The measured
// alternatives of DESIGN.md's tuning table are compiled only into the tools
// build (tools/Makefile: -DPCC_TUNING_VARIANTS -> tools/libpcc_tune.so).
using V0 = pcc::SyrkCfg<2, 4, 8, 4, 16, 6>;
// Tail kernel: 64 x 64 quadrants of the GPU tiles of the last partial wave,
// 4 warps (32 x 32 each), two CTAs per SM -- same per-cell arithmetic.
using VQ = pcc::SyrkCfg<2, 2, 4, 4, 16, 6>;
#ifdef PCC_TUNING_VARIANTS
struct DeviceConfig;
int configure_tuning_variants(DeviceConfig &c);
#endif

template <class C, int LAYOUT, bool GROUPED = false>
int configure_tma_one(int *ctas) {
  using TL = pcc::TmaLayout<C>;
  PCC_CUDA(cudaFuncSetAttribute(pcc::syrk_tma_kernel<C, LAYOUT, GROUPED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                TL::kSmemBytes),
           "cudaFuncSetAttribute(syrk_tma smem)");
  PCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas, pcc::syrk_tma_kernel<C, LAYOUT, GROUPED>, TL::kThreads,
                                                         TL::kSmemBytes),
           "cudaOccupancyMaxActiveBlocksPerMultiprocessor(tma)");
  return PCC_OK;
}

template <class C, bool GROUPED = false>
int configure_tma_variant(int *ctas) {
  int c0 = 0, c1 = 0, c2 = 0;
  int rc = configure_tma_one<C, pcc::kLayoutPacked, GROUPED>(&c0);
  if (rc == PCC_OK) rc = configure_tma_one<C, pcc::kLayoutDense, GROUPED>(&c1);
  if (rc == PCC_OK) rc = configure_tma_one<C, pcc::kLayoutTiles, GROUPED>(&c2);
  *ctas = c0 < c1 ? (c0 < c2 ? c0 : c2) : (c1 < c2 ? c1 : c2);
  return rc;
}

template <int LAYOUT>
int configure_exact_one(int *ctas) {
  using C = pcc::ExactCfg;
  PCC_CUDA(cudaFuncSetAttribute(pcc::syrk_exact_kernel<LAYOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::kSmemBytes),
           "cudaFuncSetAttribute(syrk_exact smem)");
  PCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas, pcc::syrk_exact_kernel<LAYOUT>, C::kThreads,
                                                         C::kSmemBytes),
           "cudaOccupancyMaxActiveBlocksPerMultiprocessor(exact)");
  return PCC_OK;
}

int configure_exact(int *ctas) {
  int c0 = 0, c1 = 0, c2 = 0;
  int rc = configure_exact_one<pcc::kLayoutPacked>(&c0);
  if (rc == PCC_OK) rc = configure_exact_one<pcc::kLayoutDense>(&c1);
  if (rc == PCC_OK) rc = configure_exact_one<pcc::kLayoutTiles>(&c2);
  *ctas = c0 < c1 ? (c0 < c2 ? c0 : c2) : (c1 < c2 ? c1 : c2);
  return rc;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  static cudaError_t once_err = cudaSuccess;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    once_err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (once_err == cudaSuccess && q == cudaDriverEntryPointSuccess) fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (fn == nullptr) fail(PCC_ECUDA, "cuTensorMapEncodeTiled unavailable (%s)", cudaGetErrorString(once_err));
  return fn;
}

int encode_umap(const double *u, int64_t ldu, int64_t rows, CUtensorMap *map, int box_rows = pcc::kTile) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return PCC_ECUDA;
  const cuuint64_t dims[2] = {(cuuint64_t)ldu, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ldu * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)pcc::kSlab, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(u), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PCC_ECUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return PCC_OK;
}

// Split-mode digit planes int8 [KB][7][rows][32] as a 3-D tensor {32 B, rows,
// 7 KB}; a box {32, 128, box_slices} is `box_slices` K-major operand tiles
// of one K step, written with the 32-byte swizzle the UMMA descriptors use.
int encode_slice_map(const int8_t *slices, int64_t rows, int64_t k_blocks, int box_slices, CUtensorMap *map) {
  EncodeTiledFn fn = encode_fn();
  if (fn == nullptr) return PCC_ECUDA;
  constexpr int W = pcc::SplitCfg::kRowBytes;
  const cuuint64_t dims[3] = {W, (cuuint64_t)rows, (cuuint64_t)(pcc::SplitCfg::kSlices * k_blocks)};
  const cuuint64_t strides[2] = {W, (cuuint64_t)rows * W};
  const cuuint32_t box[3] = {W, (cuuint32_t)pcc::kTile, (cuuint32_t)box_slices};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t *>(slices), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(PCC_ECUDA, "cuTensorMapEncodeTiled(slices) failed (CUresult %d)", (int)r);
  return PCC_OK;
}

template <int LAYOUT>
int configure_split_one(int *ctas) {
  using C = pcc::SplitCfg;
  PCC_CUDA(cudaFuncSetAttribute(pcc::syrk_split_kernel<LAYOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                C::kSmemBytes),
           "cudaFuncSetAttribute(split smem)");
  PCC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(ctas, pcc::syrk_split_kernel<LAYOUT>, C::kThreads,
                                                         C::kSmemBytes),
           "cudaOccupancyMaxActiveBlocksPerMultiprocessor(split)");
  return PCC_OK;
}

int configure_split(int *ctas) {
  int c0 = 0, c1 = 0, c2 = 0;
  int rc = configure_split_one<pcc::kLayoutPacked>(&c0);
  if (rc == PCC_OK) rc = configure_split_one<pcc::kLayoutDense>(&c1);
  if (rc == PCC_OK) rc = configure_split_one<pcc::kLayoutTiles>(&c2);
  *ctas = c0 < c1 ? (c0 < c2 ? c0 : c2) : (c1 < c2 ? c1 : c2);
  return rc;
}

// K1 staged kernels: shared-memory opt-in (per device -- function attributes
// belong to the device's context) and the register count the launch uses to
// pick its CTA width.
constexpr int kNormSmemPerSm = 224 * 1024;
template <int MODE>
int configure_normalize(int *regs) {
  const void *fns[] = {(const void *)pcc::normalize_rows_smem_kernel<64, MODE>,
                       (const void *)pcc::normalize_rows_smem_kernel<128, MODE>,
                       (const void *)pcc::normalize_rows_smem_kernel<256, MODE>};
  for (const void *f : fns)
    PCC_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kNormSmemPerSm),
             "cudaFuncSetAttribute(normalize smem)");
  cudaFuncAttributes fa;
  PCC_CUDA(cudaFuncGetAttributes(&fa, pcc::normalize_rows_smem_kernel<256, MODE>), "cudaFuncGetAttributes(normalize)");
  *regs = fa.numRegs;
  PCC_CUDA(cudaFuncSetAttribute(pcc::normalize_rows_chunked_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                kNormSmemPerSm),
           "cudaFuncSetAttribute(normalize chunked smem)");
  return PCC_OK;
}

// Per-device one-time setup (smem opt-in, occupancy); returns the config of
// the calling thread's current device.
int device_config(const DeviceConfig **out, int device = -1) {
  if (device < 0) {
    PCC_CUDA(cudaGetDevice(&device), "cudaGetDevice");
    // A fresh host thread has no current driver context until a runtime call
    // binds the device's primary context; the driver entry points used below
    // (cuTensorMapEncodeTiled) need one.  cudaSetDevice binds it (once per
    // thread and device).
    static thread_local int bound = -1;
    if (bound != device) {
      PCC_CUDA(cudaSetDevice(device), "cudaSetDevice");
      bound = device;
    }
  }
  if (device >= kMaxDevices) return fail(PCC_EINVAL, "device %d out of range", device);
  std::lock_guard<std::mutex> lock(g_dev_mu);
  DeviceConfig &c = g_dev[device];
  if (!c.ready) {
    int prev = 0;
    PCC_CUDA(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != device) PCC_CUDA(cudaSetDevice(device), "cudaSetDevice");
    cudaDeviceProp p;
    PCC_CUDA(cudaGetDeviceProperties(&p, device), "cudaGetDeviceProperties");
    c.sm_count = p.multiProcessorCount;
    c.cc_major = p.major;
    c.cc_minor = p.minor;
    c.max_smem_optin = (int)p.sharedMemPerBlockOptin;
    c.total_mem = p.totalGlobalMem;
    if (p.major != 10) {
      if (prev != device) cudaSetDevice(prev);
      return fail(PCC_ECUDA, "device %d is sm_%d%d; this library is built for sm_100a (B200) only", device,
                  p.major, p.minor);
    }
    int rc = configure_tma_variant<V0, true>(&c.syrk_ctas_per_sm);
    if (rc == PCC_OK) rc = configure_tma_variant<V0, false>(&c.syrk_id_ctas);
    if (rc == PCC_OK) rc = configure_tma_variant<VQ>(&c.quad_ctas);
    if (rc == PCC_OK) rc = configure_exact(&c.exact_ctas);
    if (rc == PCC_OK) rc = configure_split(&c.split_ctas);
    if (rc == PCC_OK) rc = configure_normalize<pcc::kNormLocal>(&c.norm_regs[pcc::kNormLocal]);
    if (rc == PCC_OK) rc = configure_normalize<pcc::kNormBcast>(&c.norm_regs[pcc::kNormBcast]);
    if (rc == PCC_OK) rc = configure_normalize<pcc::kNormDigits>(&c.norm_regs[pcc::kNormDigits]);
#ifdef PCC_TUNING_VARIANTS
    if (rc == PCC_OK) rc = configure_tuning_variants(c);
#endif
    if (prev != device) cudaSetDevice(prev);
    if (rc != PCC_OK) return rc;
    if (c.syrk_ctas_per_sm < 1 || c.syrk_id_ctas < 1 || c.quad_ctas < 1)
      return fail(PCC_ECUDA, "the FP64 contraction cannot be resident on device %d", device);
    if (c.exact_ctas < 1) return fail(PCC_ECUDA, "exact contraction cannot be resident on device %d", device);
    if (c.split_ctas < 1) return fail(PCC_ECUDA, "split contraction cannot be resident on device %d", device);
    c.ready = true;
  }
  *out = &c;
  return PCC_OK;
}

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }



int check_u(const double *u, int64_t n, int64_t l, int64_t ldu) {
  if (n < 1 || (uint64_t)n > 0xFFFFFFFFull) return fail(PCC_EINVAL, "n must be in [1, 2^32-1], got %lld", (long long)n);
  if (l < 1) return fail(PCC_EINVAL, "l must be >= 1, got %lld", (long long)l);
  if (ldu < pcc_ldu(l) || (ldu & 1))
    return fail(PCC_EINVAL, "ldu %lld must be even and >= pcc_ldu(l) = %lld", (long long)ldu, (long long)pcc_ldu(l));
  if (u == nullptr || (reinterpret_cast<uintptr_t>(u) & 15))
    return fail(PCC_EINVAL, "u must be a non-null 16-byte aligned device pointer");
  return PCC_OK;
}

// Tiles of a launch that go to the quadrant tail kernel (see launch_tma_cfg).
uint64_t quad_tail(uint64_t tiles, uint64_t resident, int sm_count, int quad_ctas_per_sm) {
  uint64_t tail = quad_ctas_per_sm > 0 ? tiles % resident : 0;
  if (tail > 0 && 4 * tail > (uint64_t)sm_count * (uint64_t)quad_ctas_per_sm) tail = 0;
  return tail;
}

template <class C, int LAYOUT, bool GROUPED = false, bool SKEW = false, bool STAGE_FRAGS = (C::kSlabs <= 2)>
int launch_tma_cfg(const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tb, uint64_t te,
                   const pcc::Epilogue &ep, cudaStream_t stream, int ctas_per_sm, int sm_count,
                   int quad_ctas_per_sm = 0) {
  using TL = pcc::TmaLayout<C>;
  CUtensorMap map;
  int rc = encode_umap(u, ldu, pcc_rows_padded(n), &map);
  if (rc) return rc;
  const uint64_t m_g = ceil_div((uint64_t)n, pcc::kTile);
  const int k_tiles = (int)ceil_div((uint64_t)l, C::BK);
  const uint64_t resident = (uint64_t)sm_count * (uint64_t)ctas_per_sm;
  // Tail split: a last partial wave (tiles % resident) small enough to fit
  // one round of the tail kernel (64 x 64 quadrants, quad_ctas_per_sm CTAs
  // per SM) finishes in quad_ctas_per_sm / 4 of a tile time instead of a
  // whole one.  Larger remainders gain nothing and stay in the main kernel.
  const uint64_t tail = quad_tail(te - tb, resident, sm_count, quad_ctas_per_sm);
  const uint64_t main_end = te - tail;
  if (main_end > tb) {
    const uint64_t mt = main_end - tb;
    const unsigned grid = (unsigned)(mt < resident ? mt : resident);
    // Row-group height of the (optional) grouped order: ~sqrt(wave) rows.
    uint32_t group = 1;
    while ((group + 1) * (group + 1) <= grid) ++group;
    const pcc::TileOrder order = GROUPED ? pcc::make_tile_order(m_g, tb, main_end, group)
                                         : pcc::TileOrder{tb, main_end, 0, 0, 0, main_end, main_end, mt, 1};
    pcc::syrk_tma_kernel<C, LAYOUT, GROUPED, SKEW, STAGE_FRAGS>
        <<<grid, TL::kThreads, TL::kSmemBytes, stream>>>(map, n, k_tiles, m_g, order, ep);
    PCC_CUDA(cudaGetLastError(), "syrk_tma_kernel launch");
  }
  if (tail > 0) {
    using TQ = pcc::TmaLayout<VQ>;
    CUtensorMap qmap;
    rc = encode_umap(u, ldu, pcc_rows_padded(n), &qmap, VQ::kEdge);
    if (rc) return rc;
    const uint64_t jobs = 4 * tail;
    const uint64_t qres = (uint64_t)sm_count * (uint64_t)quad_ctas_per_sm;
    const unsigned grid = (unsigned)(jobs < qres ? jobs : qres);
    const pcc::TileOrder order{main_end, te, 0, 0, 0, te, te, jobs, 1};
    pcc::syrk_tma_kernel<VQ, LAYOUT><<<grid, TQ::kThreads, TQ::kSmemBytes, stream>>>(
        qmap, n, (int)ceil_div((uint64_t)l, VQ::BK), m_g, order, ep);
    PCC_CUDA(cudaGetLastError(), "syrk_tma_kernel<quadrants> launch");
  }
  return PCC_OK;
}

template <int LAYOUT>
int launch_exact(const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tb, uint64_t te,
                 const pcc::Epilogue &ep, cudaStream_t stream, const DeviceConfig *dc) {
  using C = pcc::ExactCfg;
  const uint64_t m_g = ceil_div((uint64_t)n, pcc::kTile);
  const uint64_t units = (te - tb) * C::kSubPerTile;
  const uint64_t resident = (uint64_t)dc->sm_count * (uint64_t)dc->exact_ctas;
  const unsigned grid = (unsigned)(units < resident ? units : resident);
  const int k_chunks = (int)ceil_div((uint64_t)l, (uint64_t)C::BK);
  uint32_t group = 1;  // ~sqrt(tiles in flight): a wave of units covers grid / 8 tiles
  while ((uint64_t)(group + 1) * (group + 1) * C::kSubPerTile <= grid) ++group;
  const pcc::TileOrder order = pcc::make_tile_order(m_g, tb, te, group);
  pcc::syrk_exact_kernel<LAYOUT><<<grid, C::kThreads, C::kSmemBytes, stream>>>(u, n, ldu, k_chunks, m_g, order, ep);
  PCC_CUDA(cudaGetLastError(), "syrk_exact_kernel launch");
  return PCC_OK;
}

static const int split_dbg = [] {  // experiment knob (wrong results): 1 = no TMA loads, 2 = no MMAs,
                                   // 3 = no TMA loads and no epilogue, 4 = no MMAs and no epilogue
  const char *e = getenv("PCC_SPLIT_DEBUG");
  return e ? atoi(e) : 0;
}();

template <int LAYOUT>
int launch_split(const int8_t *slices, const double *scale, int64_t n, int64_t l, uint64_t tb, uint64_t te,
                 const pcc::Epilogue &ep, cudaStream_t stream) {
  using C = pcc::SplitCfg;
  if (te <= tb) return PCC_OK;
  const DeviceConfig *dc = nullptr;
  int rc = device_config(&dc);
  if (rc) return rc;
  const int64_t rows = pcc_rows_padded(n), k_blocks = (int64_t)ceil_div((uint64_t)l, (uint64_t)C::kRowBytes);
  CUtensorMap map1;
  rc = encode_slice_map(slices, rows, k_blocks, 1, &map1);
  if (rc) return rc;
  const uint64_t m_g = ceil_div((uint64_t)n, pcc::kTile);
  const uint64_t resident = (uint64_t)dc->sm_count * (uint64_t)(dc->split_ctas > 0 ? dc->split_ctas : 1);
  const uint64_t tiles = te - tb;
  const unsigned grid = (unsigned)(tiles < resident ? tiles : resident);
  uint32_t group = 1;
  while ((uint64_t)(group + 1) * (group + 1) <= grid) ++group;
  const pcc::TileOrder order = pcc::make_tile_order(m_g, tb, te, group);
  pcc::syrk_split_kernel<LAYOUT><<<grid, C::kThreads, C::kSmemBytes, stream>>>(map1, scale, n, l,
                                                                               (int)k_blocks, m_g, order, ep, split_dbg);
  PCC_CUDA(cudaGetLastError(), "syrk_split_kernel launch");
  return PCC_OK;
}

#ifdef PCC_TUNING_VARIANTS
#include "../../tools/syrk_variants.inc"
#endif

template <int LAYOUT>
int launch_syrk(const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tb, uint64_t te,
                const pcc::Epilogue &ep, cudaStream_t stream, int variant = 0) {
  if (te <= tb) return PCC_OK;
  const DeviceConfig *dc = nullptr;
  int rc = device_config(&dc);
  if (rc) return rc;
  if (variant == PCC_VARIANT_EXACT) return launch_exact<LAYOUT>(u, n, l, ldu, tb, te, ep, stream, dc);
  if (variant == 0) {
    static const bool id_order = [] {  // A/B knob for the tile order, read once
      const char *e = getenv("PCC_SYRK_ORDER");
      return e != nullptr && strcmp(e, "id") == 0;
    }();
    if (id_order)
      return launch_tma_cfg<V0, LAYOUT, false>(u, n, l, ldu, tb, te, ep, stream, dc->syrk_id_ctas, dc->sm_count,
                                               dc->quad_ctas);
    return launch_tma_cfg<V0, LAYOUT, true>(u, n, l, ldu, tb, te, ep, stream, dc->syrk_ctas_per_sm, dc->sm_count,
                                            dc->quad_ctas);
  }
#ifdef PCC_TUNING_VARIANTS
  return launch_tuning_variant<LAYOUT>(variant, u, n, l, ldu, tb, te, ep, stream, dc);
#else
  return fail(PCC_EINVAL, "unknown contraction variant %d (0 or PCC_VARIANT_EXACT; the measured tuning shapes are "
              "built into tools/libpcc_tune.so only)", variant);
#endif
}

// Shared-memory-staged K1 launch (the default whenever a row fits), single
// destination or broadcast to dests; kNotStaged if the row is too long.
constexpr int kNotStaged = -1;
// Chunked K1 (normalize_rows_chunked_kernel) for long rows: eligible when
// every row starts 16-byte aligned and l is even (bulk copies), chosen from
// kChunkMinL samples on (measured, DESIGN.md §3 K1).  Rows in flight per SM =
// what ~60 MB of L2 holds (each row is read three times: HBM, then L2 twice),
// set through the CTA's shared-memory footprint.  Knobs: PCC_K1_CHUNK = 0
// (never) / 1 (whenever eligible); PCC_K1_CHUNK_CTAS = rows in flight per SM.
constexpr int64_t kChunkMinL = 8192;
template <int MODE>
int launch_normalize_chunked(const double *x, int64_t ldx, double *u, int64_t ldu, uint8_t *zero_variance, int64_t l,
                             int64_t row_lo, int64_t row_hi, const pcc::NormDests &dests, cudaStream_t stream,
                             const DeviceConfig *dc) {
  static const int knob = [] {
    const char *e = getenv("PCC_K1_CHUNK");
    return e ? atoi(e) : -1;
  }();
  static const int ctas_knob = [] {
    const char *e = getenv("PCC_K1_CHUNK_CTAS");
    return e ? atoi(e) : 0;
  }();
  const bool aligned_rows = (((reinterpret_cast<uintptr_t>(x) | (uintptr_t)(ldx * 8)) & 15) == 0) && (l % 2 == 0);
  if (!aligned_rows || knob == 0 || (knob < 0 && l < kChunkMinL)) return kNotStaged;
  if (MODE != pcc::kNormDigits && (ldu & 1)) return kNotStaged;
  const uint64_t rows = (uint64_t)(row_hi - row_lo);
  if (rows > 0x7FFFFFFFull) return fail(PCC_EINVAL, "too many rows");
  int k = (int)(60.0e6 / ((double)dc->sm_count * (double)l * 8.0));
  k = k < 3 ? 3 : (k > 16 ? 16 : k);
  if (ctas_knob > 0) k = ctas_knob;
  const int budget = kNormSmemPerSm / k - 1024;  // shared memory per CTA for k CTAs per SM
  int ch = 2048;
  while (ch > 256 && 2 * ch * (int)sizeof(double) > budget) ch /= 2;
  const size_t smem = (size_t)(budget > 2 * ch * (int)sizeof(double) ? budget : 2 * ch * (int)sizeof(double));
  pcc::normalize_rows_chunked_kernel<MODE><<<(unsigned)rows, pcc::kChunkThreads, smem, stream>>>(
      x, ldx, u, ldu, zero_variance, l, row_lo, ch, dests);
  PCC_CUDA(cudaGetLastError(), "normalize_rows_chunked_kernel launch");
  return PCC_OK;
}

template <int MODE>
int launch_normalize_staged(const double *x, int64_t ldx, double *u, int64_t ldu, uint8_t *zero_variance, int64_t l,
                            int64_t row_lo, int64_t row_hi, const pcc::NormDests &dests, cudaStream_t stream) {
  const uint64_t rows = (uint64_t)(row_hi - row_lo);
  // shared-memory row stride: l when every row starts 16-byte aligned and l
  // is even, else room for the 8-byte shift of a misaligned row
  const bool aligned_rows = (((reinterpret_cast<uintptr_t>(x) | (uintptr_t)(ldx * 8)) & 15) == 0) && (l % 2 == 0);
  const int64_t lds = aligned_rows ? l : ((l + 3) & ~(int64_t)1);
  const int64_t row_bytes = lds * (int64_t)sizeof(double);
  constexpr int64_t kSmPerSmem = kNormSmemPerSm;
  const DeviceConfig *dc = nullptr;
  const int cfg_rc = device_config(&dc);  // smem opt-in + register count of this device
  if (cfg_rc) return cfg_rc;
  {
    const int crc = launch_normalize_chunked<MODE>(x, ldx, u, ldu, zero_variance, l, row_lo, row_hi, dests, stream, dc);
    if (crc != kNotStaged) return crc;
  }
  // Shared-memory staging in natural order: as many CTAs per SM as rows allow
  // (4, 3, 2, then 1 CTA/SM), up to 8 rows per CTA.
  int per_cta = 0;
  size_t smem = 0;
  // Measured (round 1, profiles/r01_normalize.log): staging beats the
  // 3-pass kernel at every BASELINE row size (c4, 64 KB rows: 1.41 vs 1.82 ms).
  constexpr int64_t kMaxStagedRow = 110 * 1024;
  for (int ctas = 4; ctas >= 1 && per_cta == 0 && row_bytes <= kMaxStagedRow; --ctas) {
    const int64_t budget = kSmPerSmem / ctas - 1024;
    if (row_bytes <= budget) {
      per_cta = (int)(budget / row_bytes < pcc::kNormSmemMaxRows ? budget / row_bytes : pcc::kNormSmemMaxRows);
      smem = (size_t)per_cta * (size_t)row_bytes;
    }
  }
  if (per_cta < 1) return kNotStaged;
  static const int rows_knob = [] {  // tuning knob: PCC_NORMALIZE_ROWS = rows staged per CTA
    const char *e = getenv("PCC_NORMALIZE_ROWS");
    return e ? atoi(e) : 0;
  }();
  if (rows_knob > 0 && rows_knob <= pcc::kNormSmemMaxRows && rows_knob * row_bytes <= kSmPerSmem - 1024) {
    per_cta = rows_knob;
    smem = (size_t)per_cta * (size_t)row_bytes;
  }
  static const int width = [] {  // tuning knob: PCC_NORMALIZE_THREADS = 64 | 128 | 256
    const char *e = getenv("PCC_NORMALIZE_THREADS");
    return e ? atoi(e) : 0;
  }();
  // Widest CTA whose register footprint still lets every smem-resident CTA
  // run (measured, profiles/r01_normalize.log: c2 -> 128, c4 -> 256).
  const int regs = dc->norm_regs[MODE] > 0 ? dc->norm_regs[MODE] : 72;
  const int64_t occ_smem = (228 * 1024) / ((int64_t)smem + 1024);
  int threads = 64;
  for (int t : {256, 128})
    if (occ_smem * t * regs <= 65536) {
      threads = t;
      break;
    }
  if (width) threads = width;
  const uint64_t grid = ceil_div(rows, (uint64_t)per_cta);
  if (grid > 0x7FFFFFFFull) return fail(PCC_EINVAL, "too many rows");
  if (threads == 256)
    pcc::normalize_rows_smem_kernel<256, MODE><<<(unsigned)grid, 256, smem, stream>>>(
        x, ldx, u, ldu, zero_variance, l, row_lo, row_hi, per_cta, lds, dests);
  else if (threads == 128)
    pcc::normalize_rows_smem_kernel<128, MODE><<<(unsigned)grid, 128, smem, stream>>>(
        x, ldx, u, ldu, zero_variance, l, row_lo, row_hi, per_cta, lds, dests);
  else
    pcc::normalize_rows_smem_kernel<64, MODE><<<(unsigned)grid, 64, smem, stream>>>(
        x, ldx, u, ldu, zero_variance, l, row_lo, row_hi, per_cta, lds, dests);
  PCC_CUDA(cudaGetLastError(), "normalize_rows_smem_kernel launch");
  return PCC_OK;
}

}  // namespace

extern "C" {

const char *pcc_last_error(void) { return g_err; }

int pcc_version(void) { return 100; }

int64_t pcc_rows_padded(int64_t n) { return n <= 0 ? 0 : (int64_t)ceil_div((uint64_t)n, pcc::kTile) * pcc::kTile; }

int64_t pcc_ldu(int64_t l) { return l <= 0 ? 0 : (int64_t)ceil_div((uint64_t)l, PCC_K_ALIGN) * PCC_K_ALIGN; }

uint64_t pcc_gpu_tile_count(int64_t n) {
  if (n <= 0) return 0;
  const uint64_t m = ceil_div((uint64_t)n, pcc::kTile);
  return m * (m + 1) / 2;
}

int pcc_device_info(int device, pcc_device_info_t *info) {
  if (info == nullptr) return fail(PCC_EINVAL, "info is NULL");
  if (device < 0) return fail(PCC_EINVAL, "device must be >= 0");
  int count = 0;
  PCC_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (device >= count) return fail(PCC_EINVAL, "device %d >= device count %d", device, count);
  const DeviceConfig *dc = nullptr;
  int rc = device_config(&dc, device);
  if (rc) return rc;
  info->device = device;
  info->sm_count = dc->sm_count;
  info->cc_major = dc->cc_major;
  info->cc_minor = dc->cc_minor;
  info->max_smem_optin = dc->max_smem_optin;
  info->syrk_ctas_per_sm = dc->syrk_ctas_per_sm;
  info->syrk_smem_bytes = pcc::TmaLayout<V0>::kSmemBytes;
  info->gpu_tile = pcc::kTile;
  info->total_mem = dc->total_mem;
  return PCC_OK;
}

int pcc_normalize_rows_f64(const double *x, int64_t ldx, double *u, int64_t ldu, uint8_t *zero_variance,
                           int64_t l, int64_t row_lo, int64_t row_hi, void *stream) {
  if (l < 2) return fail(PCC_EINVAL, "need at least 2 samples per variable, got %lld", (long long)l);
  if (ldx < l || ldu < l) return fail(PCC_EINVAL, "ldx (%lld) and ldu (%lld) must be >= l (%lld)", (long long)ldx,
                                      (long long)ldu, (long long)l);
  if (row_lo < 0 || row_hi < row_lo)
    return fail(PCC_EINVAL, "bad row range [%lld, %lld)", (long long)row_lo, (long long)row_hi);
  if (row_hi == row_lo) return PCC_OK;
  if (!x || !u || !zero_variance) return fail(PCC_EINVAL, "null pointer");
  const uint64_t rows = (uint64_t)(row_hi - row_lo);
  static const int mode = [] {
    // tuning knob: PCC_NORMALIZE_KERNEL = global forces the 3-pass kernel
    const char *e = getenv("PCC_NORMALIZE_KERNEL");
    return (e && strcmp(e, "global") == 0) ? 0 : 1;
  }();
  if (mode == 1) {
    const pcc::NormDests none{};
    const int rc = launch_normalize_staged<pcc::kNormLocal>(x, ldx, u, ldu, zero_variance, l, row_lo, row_hi, none,
                                                  (cudaStream_t)stream);
    if (rc != kNotStaged) return rc;
  }
  // rows longer than the shared-memory budget: three streaming passes from global memory
  const uint64_t grid = ceil_div(rows, pcc::kNormRowsPerCta);
  if (grid > 0x7FFFFFFFull) return fail(PCC_EINVAL, "too many rows");
  pcc::normalize_rows_kernel<<<(unsigned)grid, pcc::kNormThreads, 0, (cudaStream_t)stream>>>(
      x, ldx, u, ldu, zero_variance, l, row_lo, row_hi);
  PCC_CUDA(cudaGetLastError(), "normalize_rows_kernel launch");
  return PCC_OK;
}

int pcc_normalize_rows_bcast_f64(const double *x, int64_t ldx, double *const *u, uint8_t *const *zero_variance,
                                 int32_t n_dest, int64_t ldu, int64_t l, int64_t row_lo, int64_t row_hi,
                                 void *stream) {
  if (l < 2) return fail(PCC_EINVAL, "need at least 2 samples per variable, got %lld", (long long)l);
  if (ldx < l || ldu < l) return fail(PCC_EINVAL, "ldx (%lld) and ldu (%lld) must be >= l (%lld)", (long long)ldx,
                                      (long long)ldu, (long long)l);
  if (row_lo < 0 || row_hi < row_lo)
    return fail(PCC_EINVAL, "bad row range [%lld, %lld)", (long long)row_lo, (long long)row_hi);
  if (n_dest < 1 || n_dest > pcc::kMaxNormDests)
    return fail(PCC_EINVAL, "destination count %d outside [1, %d]", n_dest, pcc::kMaxNormDests);
  if (!x || !u || !zero_variance) return fail(PCC_EINVAL, "null pointer");
  pcc::NormDests d{};
  d.n = n_dest;
  for (int i = 0; i < n_dest; ++i) {
    if (!u[i] || !zero_variance[i]) return fail(PCC_EINVAL, "null destination %d", i);
    d.u[i] = u[i];
    d.flags[i] = zero_variance[i];
  }
  if (row_hi == row_lo) return PCC_OK;
  const int rc = launch_normalize_staged<pcc::kNormBcast>(x, ldx, nullptr, ldu, nullptr, l, row_lo, row_hi, d,
                                                (cudaStream_t)stream);
  if (rc == kNotStaged)
    return fail(PCC_EINVAL, "rows of %lld samples are too long for the broadcast normaliser (unless 16-byte aligned "
                "with even l)", (long long)l);
  return rc;
}

int pcc_normalize_split_rows_f64(const double *x, int64_t ldx, int64_t n, int64_t l, uint8_t *zero_variance,
                                 int64_t row_lo, int64_t row_hi, int8_t *slices, double *scale, void *stream) {
  if (l < 2) return fail(PCC_EINVAL, "need at least 2 samples per variable, got %lld", (long long)l);
  if (l > pcc::SplitCfg::kMaxL)
    return fail(PCC_EINVAL, "split mode is bounded to l <= %lld (got %lld)", (long long)pcc::SplitCfg::kMaxL,
                (long long)l);
  if (ldx < l) return fail(PCC_EINVAL, "ldx (%lld) must be >= l (%lld)", (long long)ldx, (long long)l);
  if (n < 1 || row_lo < 0 || row_hi < row_lo || row_hi > n)
    return fail(PCC_EINVAL, "bad row range [%lld, %lld) for n = %lld", (long long)row_lo, (long long)row_hi,
                (long long)n);
  if (!x || !zero_variance || !slices || !scale) return fail(PCC_EINVAL, "null pointer");
  if (reinterpret_cast<uintptr_t>(slices) % 16 != 0) return fail(PCC_EINVAL, "slices must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t rows_total = pcc_rows_padded(n);
  constexpr int64_t W = pcc::SplitCfg::kRowBytes;
  if (row_hi == n && rows_total > n) {  // the range ends at the last row: pad rows get zero digits and scale 0
    const int64_t kb = (l + W - 1) / W;
    PCC_CUDA(cudaMemset2DAsync(slices + n * W, (size_t)(rows_total * W), 0, (size_t)((rows_total - n) * W),
                               (size_t)(kb * pcc::SplitCfg::kSlices), s),
             "cudaMemset2DAsync(pad digit rows)");
    PCC_CUDA(cudaMemsetAsync(scale + n, 0, (size_t)(rows_total - n) * sizeof(double), s), "cudaMemsetAsync(pad scales)");
  }
  if (row_hi == row_lo) return PCC_OK;
  pcc::NormDests d{};
  d.slices = slices;
  d.scale = scale;
  d.rows_total = rows_total;
  const int rc = launch_normalize_staged<pcc::kNormDigits>(x, ldx, nullptr, 0, zero_variance, l, row_lo, row_hi, d, s);
  if (rc == kNotStaged)
    return fail(PCC_EINVAL, "rows of %lld samples are too long for the fused normaliser", (long long)l);
  return rc;
}

int pcc_device_alloc(size_t bytes, void **ptr) {
  if (!ptr) return fail(PCC_EINVAL, "ptr is NULL");
  *ptr = nullptr;
  PCC_CUDA(cudaMalloc(ptr, bytes ? bytes : 1), "cudaMalloc");
  return PCC_OK;
}

int pcc_device_free(void *ptr) {
  if (ptr) PCC_CUDA(cudaFree(ptr), "cudaFree");
  return PCC_OK;
}

int pcc_ipc_get_handle(const void *ptr, unsigned char *handle) {
  if (!ptr || !handle) return fail(PCC_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  PCC_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)), "cudaIpcGetMemHandle");
  memcpy(handle, &h, sizeof(h));
  return PCC_OK;
}

int pcc_ipc_open_handle(const unsigned char *handle, void **ptr) {
  if (!ptr || !handle) return fail(PCC_EINVAL, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  *ptr = nullptr;
  PCC_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  return PCC_OK;
}

int pcc_ipc_close_handle(void *ptr) {
  if (ptr) PCC_CUDA(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
  return PCC_OK;
}

int pcc_enable_peer_access(int device, int peer) {
  int count = 0;
  PCC_CUDA(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
  if (device < 0 || peer < 0 || device >= count || peer >= count)
    return fail(PCC_EINVAL, "devices (%d, %d) outside [0, %d)", device, peer, count);
  if (device == peer) return PCC_OK;
  int can = 0;
  PCC_CUDA(cudaDeviceCanAccessPeer(&can, device, peer), "cudaDeviceCanAccessPeer");
  if (!can) return fail(PCC_ECUDA, "device %d cannot access device %d's memory (no peer path)", device, peer);
  int prev = 0;
  PCC_CUDA(cudaGetDevice(&prev), "cudaGetDevice");
  PCC_CUDA(cudaSetDevice(device), "cudaSetDevice");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  cudaSetDevice(prev);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();  // clear the sticky-free "already enabled" status
    return PCC_OK;
  }
  if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
  return PCC_OK;
}

int pcc_zero_rows_f64(double *u, int64_t ldu, int64_t row_lo, int64_t row_hi, void *stream) {
  if (row_lo < 0 || row_hi < row_lo || ldu < 0) return fail(PCC_EINVAL, "bad row range");
  if (row_hi == row_lo || ldu == 0) return PCC_OK;
  PCC_CUDA(cudaMemsetAsync(u + row_lo * ldu, 0, (size_t)(row_hi - row_lo) * (size_t)ldu * sizeof(double),
                           (cudaStream_t)stream),
           "cudaMemsetAsync(pad rows)");
  return PCC_OK;
}

int pcc_syrk_f64(const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tile_begin, uint64_t tile_end,
                 int32_t layout, double *out, int64_t ld_out, uint64_t out_base, int32_t ref_t, uint64_t ref_begin,
                 uint64_t ref_end, void *stream) {
  return pcc_syrk_f64_variant(0, u, n, l, ldu, tile_begin, tile_end, layout, out, ld_out, out_base, ref_t, ref_begin,
                              ref_end, stream);
}

int pcc_syrk_f64_variant(int32_t variant, const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tile_begin,
                         uint64_t tile_end, int32_t layout, double *out, int64_t ld_out, uint64_t out_base,
                         int32_t ref_t, uint64_t ref_begin, uint64_t ref_end, void *stream) {
  int rc = check_u(u, n, l, ldu);
  if (rc) return rc;
  const uint64_t total = pcc_gpu_tile_count(n);
  if (tile_begin > tile_end || tile_end > total)
    return fail(PCC_EINVAL, "tile range [%llu, %llu) invalid for %llu tiles", (unsigned long long)tile_begin,
                (unsigned long long)tile_end, (unsigned long long)total);
  if (out == nullptr) return fail(PCC_EINVAL, "out is NULL");
  pcc::Epilogue ep{out, ld_out, out_base, ref_t, 0, ref_begin, ref_end};
  cudaStream_t s = (cudaStream_t)stream;
  switch (layout) {
    case PCC_LAYOUT_PACKED:
      return launch_syrk<pcc::kLayoutPacked>(u, n, l, ldu, tile_begin, tile_end, ep, s, variant);
    case PCC_LAYOUT_DENSE:
      if (ld_out < n) return fail(PCC_EINVAL, "dense ld_out %lld < n %lld", (long long)ld_out, (long long)n);
      return launch_syrk<pcc::kLayoutDense>(u, n, l, ldu, tile_begin, tile_end, ep, s, variant);
    case PCC_LAYOUT_TILES: {
      if (ref_t < 1) return fail(PCC_EINVAL, "tile size must be >= 1, got %d", ref_t);
      ep.ref_m = ceil_div((uint64_t)n, (uint64_t)ref_t);
      const uint64_t ref_total = ep.ref_m * (ep.ref_m + 1) / 2;
      if (ref_begin > ref_end || ref_end > ref_total)
        return fail(PCC_EINVAL, "tile range [%llu, %llu) invalid for %llu tiles", (unsigned long long)ref_begin,
                    (unsigned long long)ref_end, (unsigned long long)ref_total);
      return launch_syrk<pcc::kLayoutTiles>(u, n, l, ldu, tile_begin, tile_end, ep, s, variant);
    }
    default:
      return fail(PCC_EINVAL, "unknown layout %d", layout);
  }
}

int pcc_syrk_exact_f64(const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tile_begin, uint64_t tile_end,
                       int32_t layout, double *out, int64_t ld_out, uint64_t out_base, int32_t ref_t,
                       uint64_t ref_begin, uint64_t ref_end, void *stream) {
  return pcc_syrk_f64_variant(PCC_VARIANT_EXACT, u, n, l, ldu, tile_begin, tile_end, layout, out, ld_out, out_base,
                              ref_t, ref_begin, ref_end, stream);
}

uint64_t pcc_split_slice_bytes(int64_t n, int64_t l) {
  if (n < 1 || l < 1) return 0;
  return (uint64_t)pcc::SplitCfg::kSlices * (uint64_t)pcc_rows_padded(n) *
         ceil_div((uint64_t)l, (uint64_t)pcc::SplitCfg::kRowBytes) * pcc::SplitCfg::kRowBytes;
}

int pcc_split_rows_f64(const double *u, int64_t n, int64_t l, int64_t ldu, int64_t row_lo, int64_t row_hi,
                       int8_t *slices, double *scale, void *stream) {
  int rc = check_u(u, n, l, ldu);
  if (rc) return rc;
  const int64_t rows = pcc_rows_padded(n);
  if (row_lo < 0 || row_lo > row_hi || row_hi > rows)
    return fail(PCC_EINVAL, "row range [%lld, %lld) invalid for %lld padded rows", (long long)row_lo,
                (long long)row_hi, (long long)rows);
  if (slices == nullptr || scale == nullptr) return fail(PCC_EINVAL, "slices / scale is NULL");
  if (reinterpret_cast<uintptr_t>(slices) % 16 != 0) return fail(PCC_EINVAL, "slices must be 16-byte aligned");
  if (row_hi == row_lo) return PCC_OK;
  const int64_t rows_per_block = 8;
  const unsigned grid = (unsigned)ceil_div((uint64_t)(row_hi - row_lo), (uint64_t)rows_per_block);
  pcc::split_rows_kernel<<<grid, 32 * rows_per_block, 0, (cudaStream_t)stream>>>(u, ldu, l, row_lo, row_hi, rows,
                                                                                 slices, scale);
  PCC_CUDA(cudaGetLastError(), "split_rows_kernel launch");
  return PCC_OK;
}

int pcc_syrk_split_f64(const int8_t *slices, const double *scale, int64_t n, int64_t l, uint64_t tile_begin,
                       uint64_t tile_end, int32_t layout, double *out, int64_t ld_out, uint64_t out_base,
                       int32_t ref_t, uint64_t ref_begin, uint64_t ref_end, void *stream) {
  if (n < 1 || l < 2) return fail(PCC_EINVAL, "need n >= 1 and l >= 2 (got n=%lld, l=%lld)", (long long)n, (long long)l);
  if (l > pcc::SplitCfg::kMaxL)
    return fail(PCC_EINVAL, "split mode is bounded to l <= %lld (got %lld); use pcc_syrk_f64",
                (long long)pcc::SplitCfg::kMaxL, (long long)l);
  if (slices == nullptr || scale == nullptr) return fail(PCC_EINVAL, "slices / scale is NULL");
  if (reinterpret_cast<uintptr_t>(slices) % 16 != 0) return fail(PCC_EINVAL, "slices must be 16-byte aligned");
  const uint64_t total = pcc_gpu_tile_count(n);
  if (tile_begin > tile_end || tile_end > total)
    return fail(PCC_EINVAL, "tile range [%llu, %llu) invalid for %llu tiles", (unsigned long long)tile_begin,
                (unsigned long long)tile_end, (unsigned long long)total);
  if (out == nullptr) return fail(PCC_EINVAL, "out is NULL");
  pcc::Epilogue ep{out, ld_out, out_base, ref_t, 0, ref_begin, ref_end};
  cudaStream_t s = (cudaStream_t)stream;
  switch (layout) {
    case PCC_LAYOUT_PACKED:
      return launch_split<pcc::kLayoutPacked>(slices, scale, n, l, tile_begin, tile_end, ep, s);
    case PCC_LAYOUT_DENSE:
      if (ld_out < n) return fail(PCC_EINVAL, "dense ld_out %lld < n %lld", (long long)ld_out, (long long)n);
      return launch_split<pcc::kLayoutDense>(slices, scale, n, l, tile_begin, tile_end, ep, s);
    case PCC_LAYOUT_TILES: {
      if (ref_t < 1) return fail(PCC_EINVAL, "tile size must be >= 1, got %d", ref_t);
      ep.ref_m = ceil_div((uint64_t)n, (uint64_t)ref_t);
      const uint64_t ref_total = ep.ref_m * (ep.ref_m + 1) / 2;
      if (ref_begin > ref_end || ref_end > ref_total)
        return fail(PCC_EINVAL, "tile range [%llu, %llu) invalid for %llu tiles", (unsigned long long)ref_begin,
                    (unsigned long long)ref_end, (unsigned long long)ref_total);
      return launch_split<pcc::kLayoutTiles>(slices, scale, n, l, tile_begin, tile_end, ep, s);
    }
    default:
      return fail(PCC_EINVAL, "unknown layout %d", layout);
  }
}

// Reference pass (tiles [j_lo, j_hi) of tile size t, _kernels.py:351-373):
// validate, zero the pass buffer (cells outside y <= x < n stay 0.0,
// _kernels.py:370-373) and find the GPU tiles [*tb, *te) covering those
// reference tile rows; the caller then runs the contraction with the TILES
// epilogue over them (an empty pass gives *tb == *te).
static int compute_pass_prepare(int64_t n, int64_t t, uint64_t j_lo, uint64_t j_hi, double *out, void *stream,
                                uint64_t *tb, uint64_t *te) {
  *tb = *te = 0;
  if (t < 1) return fail(PCC_EINVAL, "tile size must be >= 1, got %lld", (long long)t);
  const uint64_t m = ceil_div((uint64_t)n, (uint64_t)t);
  const uint64_t total = m * (m + 1) / 2;
  if (j_lo > j_hi || j_hi > total)
    return fail(PCC_EINVAL, "tile range [%llu, %llu) invalid for %llu tiles", (unsigned long long)j_lo,
                (unsigned long long)j_hi, (unsigned long long)total);
  if (j_hi == j_lo) return PCC_OK;
  if (out == nullptr) return fail(PCC_EINVAL, "out is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  PCC_CUDA(cudaMemsetAsync(out, 0, (size_t)(j_hi - j_lo) * (size_t)t * (size_t)t * sizeof(double), s),
           "cudaMemsetAsync(pass buffer)");
  const uint64_t yt_a = pcc::tile_row(m, j_lo), yt_b = pcc::tile_row(m, j_hi - 1);
  const uint64_t y_a = yt_a * (uint64_t)t;
  uint64_t y_b = (yt_b + 1) * (uint64_t)t;
  if (y_b > (uint64_t)n) y_b = (uint64_t)n;
  const uint64_t m_g = ceil_div((uint64_t)n, pcc::kTile);
  const uint64_t Ya = y_a / pcc::kTile, Yb = (y_b - 1) / pcc::kTile;
  *tb = pcc::row_prefix(m_g, Ya);
  *te = pcc::row_prefix(m_g, Yb + 1);
  return PCC_OK;
}

static int compute_pass_impl(int32_t variant, const double *u, int64_t n, int64_t l, int64_t ldu, int64_t t,
                             uint64_t j_lo, uint64_t j_hi, double *out, void *stream) {
  int rc = check_u(u, n, l, ldu);
  if (rc) return rc;
  uint64_t tb, te;
  rc = compute_pass_prepare(n, t, j_lo, j_hi, out, stream, &tb, &te);
  if (rc || tb == te) return rc;
  return pcc_syrk_f64_variant(variant, u, n, l, ldu, tb, te, PCC_LAYOUT_TILES, out, 0, 0, (int32_t)t, j_lo, j_hi,
                              stream);
}

int pcc_compute_pass_split_f64(const int8_t *slices, const double *scale, int64_t n, int64_t l, int64_t t,
                               uint64_t j_lo, uint64_t j_hi, double *out, void *stream) {
  if (n < 1 || l < 2) return fail(PCC_EINVAL, "need n >= 1 and l >= 2 (got n=%lld, l=%lld)", (long long)n, (long long)l);
  uint64_t tb, te;
  int rc = compute_pass_prepare(n, t, j_lo, j_hi, out, stream, &tb, &te);
  if (rc || tb == te) return rc;
  return pcc_syrk_split_f64(slices, scale, n, l, tb, te, PCC_LAYOUT_TILES, out, 0, 0, (int32_t)t, j_lo, j_hi, stream);
}

int pcc_compute_pass_f64(const double *u, int64_t n, int64_t l, int64_t ldu, int64_t t, uint64_t j_lo,
                         uint64_t j_hi, double *out, void *stream) {
  return compute_pass_impl(0, u, n, l, ldu, t, j_lo, j_hi, out, stream);
}

int pcc_compute_pass_exact_f64(const double *u, int64_t n, int64_t l, int64_t ldu, int64_t t, uint64_t j_lo,
                               uint64_t j_hi, double *out, void *stream) {
  return compute_pass_impl(PCC_VARIANT_EXACT, u, n, l, ldu, t, j_lo, j_hi, out, stream);
}

int pcc_scatter_range_f64(double *packed, const double *values, uint64_t first_tile, uint64_t count, int64_t t,
                          int64_t n, void *stream) {
  if (t < 1 || n < 1) return fail(PCC_EINVAL, "bad geometry n=%lld t=%lld", (long long)n, (long long)t);
  const uint64_t m = ceil_div((uint64_t)n, (uint64_t)t);
  if (first_tile + count > m * (m + 1) / 2) return fail(PCC_EINVAL, "tile range outside the tile matrix");
  if (count == 0) return PCC_OK;
  if (!packed || !values) return fail(PCC_EINVAL, "null pointer");
  const uint64_t cells = count * (uint64_t)t * (uint64_t)t;
  uint64_t grid = ceil_div(cells, 256);
  if (grid > 148ull * 64) grid = 148ull * 64;
  pcc::scatter_range_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(packed, values, first_tile, count, t,
                                                                              n, m);
  PCC_CUDA(cudaGetLastError(), "scatter_range_kernel launch");
  return PCC_OK;
}

int pcc_allpairs_f64(const double *x, int64_t n, int64_t l, int64_t ldx, double *u, int64_t ldu,
                     uint8_t *zero_variance, uint64_t tile_begin, uint64_t tile_end, int32_t layout, double *out,
                     int64_t ld_out, uint64_t out_base, void *stream) {
  int rc = check_u(u, n, l, ldu);
  if (rc) return rc;
  if (tile_end == UINT64_MAX) tile_end = pcc_gpu_tile_count(n);
  rc = pcc_normalize_rows_f64(x, ldx, u, ldu, zero_variance, l, 0, n, stream);
  if (rc) return rc;
  rc = pcc_zero_rows_f64(u, ldu, n, pcc_rows_padded(n), stream);
  if (rc) return rc;
  return pcc_syrk_f64(u, n, l, ldu, tile_begin, tile_end, layout, out, ld_out, out_base, 0, 0, 0, stream);
}

int pcc_row_stats_f64(const double *x, int64_t ldx, int64_t n, int64_t l, double *mean, double *ssd,
                      uint8_t *constant, void *stream) {
  if (n < 1 || l < 1 || ldx < l) return fail(PCC_EINVAL, "bad shape n=%lld l=%lld ldx=%lld", (long long)n,
                                              (long long)l, (long long)ldx);
  if (!x || !mean || !ssd || !constant) return fail(PCC_EINVAL, "null pointer");
  pcc::row_stats_kernel<<<(unsigned)ceil_div((uint64_t)n, 32), 256, 0, (cudaStream_t)stream>>>(x, ldx, l, n, mean, ssd,
                                                                                               constant);
  PCC_CUDA(cudaGetLastError(), "row_stats_kernel launch");
  return PCC_OK;
}

int pcc_naive_pairs_f64(const double *x, int64_t ldx, int64_t n, int64_t l, const double *mean, const double *ssd,
                        const uint8_t *constant, uint64_t id_lo, uint64_t id_hi, double *out, void *stream) {
  if (n < 1 || l < 1 || ldx < l) return fail(PCC_EINVAL, "bad shape");
  const uint64_t total = (uint64_t)n * ((uint64_t)n + 1) / 2;
  if (id_lo > id_hi || id_hi > total) return fail(PCC_EINVAL, "job id range [%llu, %llu) outside [0, %llu)",
                                                  (unsigned long long)id_lo, (unsigned long long)id_hi,
                                                  (unsigned long long)total);
  if (id_hi == id_lo) return PCC_OK;
  if (!x || !mean || !ssd || !constant || !out) return fail(PCC_EINVAL, "null pointer");
  const DeviceConfig *dc = nullptr;
  int rc = device_config(&dc);
  if (rc) return rc;
  uint64_t grid = ceil_div(id_hi - id_lo, 32);  // 8 warps x 4 pairs per CTA
  const uint64_t cap = (uint64_t)dc->sm_count * 8;
  if (grid > cap) grid = cap;
  pcc::naive_pairs_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(x, ldx, l, n, mean, ssd, constant, id_lo,
                                                                           id_hi, out);
  PCC_CUDA(cudaGetLastError(), "naive_pairs_kernel launch");
  return PCC_OK;
}

int pcc_tile_schedule(int64_t n, uint64_t tile_begin, uint64_t tile_end, uint32_t group, uint64_t *ys,
                      uint64_t *xs) {
  if (n < 1) return fail(PCC_EINVAL, "n must be >= 1");
  const uint64_t total = pcc_gpu_tile_count(n);
  if (tile_begin > tile_end || tile_end > total) return fail(PCC_EINVAL, "tile range outside the tile matrix");
  if (!ys || !xs) return fail(PCC_EINVAL, "null output");
  const uint64_t m = ceil_div((uint64_t)n, pcc::kTile);
  const pcc::TileOrder o = pcc::make_tile_order(m, tile_begin, tile_end, group);
  for (uint64_t s = 0; s < o.total; ++s) pcc::tile_at(o, m, s, ys[s], xs[s]);
  return PCC_OK;
}

int pcc_syrk_launches(int64_t n, uint64_t tile_begin, uint64_t tile_end, int32_t *launches) {
  if (!launches) return fail(PCC_EINVAL, "launches is NULL");
  if (n < 1) return fail(PCC_EINVAL, "n must be >= 1");
  if (tile_begin > tile_end || tile_end > pcc_gpu_tile_count(n))
    return fail(PCC_EINVAL, "tile range outside the tile matrix");
  const DeviceConfig *dc = nullptr;
  int rc = device_config(&dc);
  if (rc) return rc;
  const uint64_t tiles = tile_end - tile_begin;
  const uint64_t resident = (uint64_t)dc->sm_count * (uint64_t)dc->syrk_ctas_per_sm;
  const uint64_t tail = quad_tail(tiles, resident, dc->sm_count, dc->quad_ctas);
  *launches = (tiles > tail ? 1 : 0) + (tail > 0 ? 1 : 0);
  return PCC_OK;
}

int pcc_probe_fp64_peak(double *tflops) {
  if (!tflops) return fail(PCC_EINVAL, "tflops is NULL");
  const DeviceConfig *dc = nullptr;
  int rc = device_config(&dc);
  if (rc) return rc;
  double *scratch = nullptr;
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  // every resource is released on every path (the probe can run many times)
  auto release = [&] {
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    if (s) cudaStreamDestroy(s);
    if (scratch) cudaFree(scratch);
  };
  auto bail = [&](cudaError_t e, const char *what) {
    release();
    return cuda_fail(e, what);
  };
  cudaError_t e;
  if ((e = cudaMalloc(&scratch, sizeof(double))) != cudaSuccess) return bail(e, "cudaMalloc");
  if ((e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)) != cudaSuccess) return bail(e, "cudaStreamCreate");
  if ((e = cudaEventCreate(&e0)) != cudaSuccess) return bail(e, "cudaEventCreate");
  if ((e = cudaEventCreate(&e1)) != cudaSuccess) return bail(e, "cudaEventCreate");
  const int threads = 512, iters = 4000;
  const int grid = dc->sm_count * 2;
  pcc::dmma_probe_kernel<<<grid, threads, 0, s>>>(scratch, 200);  // warm-up
  if ((e = cudaGetLastError()) != cudaSuccess) return bail(e, "dmma_probe_kernel launch");
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, s);
    pcc::dmma_probe_kernel<<<grid, threads, 0, s>>>(scratch, iters);
    cudaEventRecord(e1, s);
    if ((e = cudaEventSynchronize(e1)) != cudaSuccess) return bail(e, "dmma_probe_kernel");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 256.0 * 8.0 * iters * (double)(threads / 32) * grid;
  *tflops = flops / ((double)best * 1e-3) / 1e12;
  release();
  return PCC_OK;
}

}  // extern "C"
