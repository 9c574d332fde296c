/*
 * pcc_b200.h -- C ABI of the B200-native all-pairs Pearson correlation engine.
 *
 * This is the drop-in boundary for the reference package `paircorr`'s hot
 * path (LightPCC, arXiv:1605.01584).  The reference has no C ABI: its de-facto
 * FFI is the set of numba kernels that its Python layers call with flat
 * C-contiguous arrays plus integers, released from the GIL
 * (/root/reference/pkg/src/paircorr/_kernels.py).  Each entry point below
 * names the reference function it replaces.  A host binding (ctypes) is shown
 * in INTEGRATION.md; the in-tree Python host layer is paper_1605_01584_b200/.
 *
 * Conventions (all entry points):
 *   - pointers named x, u, out, packed, values, zero_variance are DEVICE
 *     pointers (cudaMalloc / torch CUDA tensors); the caller owns all memory;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream); every call is asynchronous on it;
 *   - return 0 on success, PCC_EINVAL for a rejected argument (the reference
 *     raises ValueError), PCC_ECUDA for a CUDA failure; the message is in
 *     pcc_last_error() (thread-local).  No C++ exception crosses the ABI;
 *   - stateless and re-entrant; one host thread per device is the intended
 *     multi-GPU model (the calling thread's current device is used).
 */
#ifndef PCC_B200_H
#define PCC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCC_OK 0
#define PCC_EINVAL 1
#define PCC_ECUDA 2

/* Edge of the square GPU tile the contraction schedules (rows x cols).  The
 * GPU tile matrix has m_g = ceil(n / PCC_GPU_TILE) tiles per side and
 * m_g(m_g+1)/2 upper-triangle tile jobs, numbered by the same bijection as
 * the reference's jobs and t x t tiles (indexing.py:55-109, tiles.py:47-71). */
#define PCC_GPU_TILE 128
/* U's row padding: ldu must be >= pcc_ldu(l) (multiple of PCC_K_ALIGN) and
 * U must have pcc_rows_padded(n) rows, the pad rows/columns zero. */
#define PCC_K_ALIGN 32

/* Output layouts of pcc_syrk_f64. */
#define PCC_LAYOUT_PACKED 0 /* upper triangle in job-id order: out[F(y)+x-y - out_base] (tiles.py:93-99) */
#define PCC_LAYOUT_DENSE 1  /* full symmetric n x n, row stride ld_out (tiles.py:107-116 to_dense) */
#define PCC_LAYOUT_TILES 2  /* reference pass buffer: t x t tiles [ref_begin, ref_end) at
                               (J - ref_begin) * t * t, row-major inside a tile (tiles.py:1-18) */

typedef struct {
  int device;
  int sm_count;
  int cc_major;
  int cc_minor;
  int max_smem_optin;        /* bytes per block */
  int syrk_ctas_per_sm;      /* resident contraction CTAs per SM */
  int syrk_smem_bytes;       /* dynamic shared memory per contraction CTA */
  int gpu_tile;              /* == PCC_GPU_TILE */
  size_t total_mem;          /* bytes of device memory */
} pcc_device_info_t;

/* Last error message of the calling thread ("" if none). */
const char *pcc_last_error(void);

/* ABI version (major * 100 + minor). */
int pcc_version(void);

/* Device / kernel-configuration query for `device` (>= 0). */
int pcc_device_info(int device, pcc_device_info_t *info);

/* Helpers for sizing U: rows rounded up to the GPU tile, K rounded up to
 * PCC_K_ALIGN.  Pure functions of their arguments. */
int64_t pcc_rows_padded(int64_t n);
int64_t pcc_ldu(int64_t l);
/* Tiles of the GPU tile matrix: m_g(m_g+1)/2 with m_g = ceil(n/PCC_GPU_TILE). */
uint64_t pcc_gpu_tile_count(int64_t n);

/* Replaces _kernels.normalize_rows(x, u, zero_variance, row_lo, row_hi)
 * (_kernels.py:226-252), as driven by transform.normalize (transform.py:99-124).
 *
 * For rows i in [row_lo, row_hi) of x (row stride ldx doubles, l samples):
 * constant row (every sample equals the first, _kernels.py:209-223) or
 * computed ssd == 0.0  ->  u row all zeros, zero_variance[i] = 1;
 * else u[i][k] = (x[i][k] - mean) / sqrt(ssd), zero_variance[i] = 0, with
 * mean = sum8(x_i)/l and ssd = ssd8(x_i, mean) in the reference's fixed
 * 8-lane order without FMA -- bit-identical to the reference.
 * Also writes u[i][k] = 0 for l <= k < ldu.  Requires l >= 2 (the reference
 * Dataset's rule, transform.py:66-67), ldx >= l, ldu >= l. */
int pcc_normalize_rows_f64(const double *x, int64_t ldx, double *u, int64_t ldu,
                           uint8_t *zero_variance, int64_t l, int64_t row_lo, int64_t row_hi,
                           void *stream);

/* pcc_normalize_rows_f64 writing every U row and zero-variance flag to
 * n_dest (<= 16) buffers at once: u[d] / zero_variance[d] are device
 * pointers (host array), typically peer GPUs' U over NVLink opened with
 * pcc_ipc_open_handle -- normalisation fused with the all-gather of U in
 * the multi-GPU exchange (distributed.exchange_normalize, mode "p2p").
 * Replaces normalize_rows (_kernels.py:226-252) + the worker model's
 * per-worker normalisation (worker.py:68-80).  Rows up to 110 KB, or of any
 * length when 16-byte aligned with even l (the chunked kernel). */
int pcc_normalize_rows_bcast_f64(const double *x, int64_t ldx, double *const *u, uint8_t *const *zero_variance,
                                 int32_t n_dest, int64_t ldu, int64_t l, int64_t row_lo, int64_t row_hi,
                                 void *stream);

/* Plain device allocation (cudaMalloc) so an IPC handle covers exactly the
 * buffer; CUDA IPC of such buffers between the ranks of one node. */
int pcc_device_alloc(size_t bytes, void **ptr);
int pcc_device_free(void *ptr);
int pcc_ipc_get_handle(const void *ptr, unsigned char *handle /* 64 bytes */);
int pcc_ipc_open_handle(const unsigned char *handle /* 64 bytes */, void **ptr);
int pcc_ipc_close_handle(void *ptr);

/* Let kernels running on `device` load/store `peer`'s memory (in-process
 * multi-GPU exchange: the broadcast normaliser writes U rows into every
 * device's buffer over NVLink).  OK if device == peer or already enabled;
 * PCC_ECUDA if the two GPUs have no peer path. */
int pcc_enable_peer_access(int device, int peer);

/* Zero rows [row_lo, row_hi) of U (the pad rows up to pcc_rows_padded(n)). */
int pcc_zero_rows_f64(double *u, int64_t ldu, int64_t row_lo, int64_t row_hi, void *stream);

/* Replaces _kernels.compute_tile_range + _kernels.scatter_range
 * (_kernels.py:322-373) as driven by tiles.compute_pass / scatter_pass
 * (tiles.py:133-242) and engine.allpairs (engine.py:23-56).
 *
 * Symmetric tiled contraction C = U U^T over the GPU tile jobs
 * [tile_begin, tile_end) of the m_g x m_g GPU tile matrix.  Every cell
 * (y, x) with y <= x < n of those tiles gets C[y][x] = sum_k U[y][k] U[x][k]
 * (FP64, fixed per-cell K order: bitwise independent of the tile range, the
 * grid and the device count) and is written per `layout`:
 *   PCC_LAYOUT_PACKED: out[y(2n-y+1)/2 + x - y - out_base]
 *   PCC_LAYOUT_DENSE:  out[y*ld_out + x] and out[x*ld_out + y]
 *   PCC_LAYOUT_TILES:  reference t x t tile J = (y/t, x/t) if
 *                      ref_begin <= J < ref_end, at
 *                      out[(J - ref_begin)*t*t + (y%t)*t + (x%t)]
 *                      (cells outside y <= x < n are NOT written; see
 *                      pcc_compute_pass_f64 for the zero-filled variant).
 * U: device, pcc_rows_padded(n) rows of stride ldu (>= pcc_ldu(l), even),
 * 16-byte aligned, pad rows/columns zero. */
int pcc_syrk_f64(const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tile_begin,
                 uint64_t tile_end, int32_t layout, double *out, int64_t ld_out, uint64_t out_base,
                 int32_t ref_t, uint64_t ref_begin, uint64_t ref_end, void *stream);

/* The contraction in the reference's own arithmetic, bit-identical to
 * _kernels.dot8 (_kernels.py:30-68) for every cell: eight lane sums of
 * separately rounded products, k = j (mod 8) in increasing k, then the fixed
 * tree.  Runs on the FP64 CUDA cores (about half the tensor path's speed);
 * same arguments, layouts and errors as pcc_syrk_f64.  Same as
 * pcc_syrk_f64_variant(PCC_VARIANT_EXACT, ...). */
#define PCC_VARIANT_EXACT 100
int pcc_syrk_exact_f64(const double *u, int64_t n, int64_t l, int64_t ldu, uint64_t tile_begin,
                       uint64_t tile_end, int32_t layout, double *out, int64_t ld_out, uint64_t out_base,
                       int32_t ref_t, uint64_t ref_begin, uint64_t ref_end, void *stream);

/* Split mode: the contraction on the int8 tensor cores (tcgen05.mma
 * kind::i8, s32 accumulators in tensor memory) to FP64 accuracy -- the
 * Ozaki splitting scheme.  pcc_split_rows_f64 writes, for U rows
 * [row_lo, row_hi) (up to pcc_rows_padded(n), so pad rows become zero), 7
 * signed radix-128 digit planes (int8, pcc_split_slice_bytes(n, l) bytes,
 * 16-byte aligned) and one power-of-two scale per row (double[rows]); every
 * step is exact.  pcc_syrk_split_f64 then contracts GPU tiles
 * [tile_begin, tile_end) from those digits with the arguments, layouts and
 * errors of pcc_syrk_f64: 34 int8 products per K step (digit pairs
 * i + j <= 9), exact in s32, combined in FP64.  |result - U·Uᵀ| <= 9e-13 per
 * coefficient for l <= 8192 (K2s); l > 8192 is PCC_EINVAL. */
uint64_t pcc_split_slice_bytes(int64_t n, int64_t l);
int pcc_split_rows_f64(const double *u, int64_t n, int64_t l, int64_t ldu, int64_t row_lo,
                       int64_t row_hi, int8_t *slices, double *scale, void *stream);
int pcc_syrk_split_f64(const int8_t *slices, const double *scale, int64_t n, int64_t l,
                       uint64_t tile_begin, uint64_t tile_end, int32_t layout, double *out,
                       int64_t ld_out, uint64_t out_base, int32_t ref_t, uint64_t ref_begin,
                       uint64_t ref_end, void *stream);

/* Same as pcc_syrk_f64 with an explicit contraction kernel: 0 = the
 * production kernel, PCC_VARIANT_EXACT = the bit-exact dot8 kernel
 * (pcc_syrk_exact_f64); anything else is PCC_EINVAL.  The tools build of the
 * same source (tools/Makefile -> tools/libpcc_tune.so) also accepts the
 * measured alternative shapes 1..14 of DESIGN.md's tuning table; every shape
 * computes each cell with the same K order (bitwise identical results). */
int pcc_syrk_f64_variant(int32_t variant, const double *u, int64_t n, int64_t l, int64_t ldu,
                         uint64_t tile_begin, uint64_t tile_end, int32_t layout, double *out,
                         int64_t ld_out, uint64_t out_base, int32_t ref_t, uint64_t ref_begin,
                         uint64_t ref_end, void *stream);

/* Replaces _kernels.compute_tile_range(u, out, n, t, m, j_lo, j_hi, base)
 * (_kernels.py:351-373) with base = j_lo: fills out[0 .. (j_hi-j_lo)*t*t)
 * with the reference's t x t tiles [j_lo, j_hi), cells outside y <= x < n
 * exactly 0.0 -- the pass-buffer layout of tiles.compute_pass
 * (tiles.py:133-199).  Launches the GPU tiles that cover the range. */
int pcc_compute_pass_f64(const double *u, int64_t n, int64_t l, int64_t ldu, int64_t t,
                         uint64_t j_lo, uint64_t j_hi, double *out, void *stream);

/* pcc_compute_pass_f64 with the bit-exact contraction (pcc_syrk_exact_f64):
 * the pass buffer equals the reference's compute_tile_range output bit for
 * bit. */
int pcc_compute_pass_exact_f64(const double *u, int64_t n, int64_t l, int64_t ldu, int64_t t,
                               uint64_t j_lo, uint64_t j_hi, double *out, void *stream);

/* pcc_normalize_rows_f64 fused with pcc_split_rows_f64: rows [row_lo,
 * row_hi) of x (n x l, stride ldx, l <= 8192) are normalised exactly as the
 * reference does (same bits as pcc_normalize_rows_f64) and written straight
 * into split-mode digit planes and scales (the same bytes pcc_split_rows_f64
 * makes from that U); U itself is not written.  A range ending at row n
 * also zeroes the pad rows' digits and scales. */
int pcc_normalize_split_rows_f64(const double *x, int64_t ldx, int64_t n, int64_t l,
                                 uint8_t *zero_variance, int64_t row_lo, int64_t row_hi,
                                 int8_t *slices, double *scale, void *stream);

/* pcc_compute_pass_f64 from split-mode digit planes (pcc_split_rows_f64 over
 * every row the pass touches): the reference's pass-buffer layout, each
 * coefficient within 1e-12 of the reference's. */
int pcc_compute_pass_split_f64(const int8_t *slices, const double *scale, int64_t n, int64_t l,
                               int64_t t, uint64_t j_lo, uint64_t j_hi, double *out, void *stream);

/* Replaces _kernels.scatter_range(packed, values, first_tile, count, m, t, n)
 * (_kernels.py:322-348) on device: copies cells y <= x < n of `count`
 * consecutive t x t tiles from a flat pass buffer into the packed triangle. */
int pcc_scatter_range_f64(double *packed, const double *values, uint64_t first_tile,
                          uint64_t count, int64_t t, int64_t n, void *stream);

/* One-call fast path of engine.allpairs (engine.py:23-56) on the current
 * device: normalize x (n x l, stride ldx) into the caller's U workspace
 * (pcc_rows_padded(n) x ldu), then contract GPU tiles [tile_begin, tile_end)
 * into `out` (layout as pcc_syrk_f64).  tile_end == UINT64_MAX means all. */
int pcc_allpairs_f64(const double *x, int64_t n, int64_t l, int64_t ldx, double *u, int64_t ldu,
                     uint8_t *zero_variance, uint64_t tile_begin, uint64_t tile_end,
                     int32_t layout, double *out, int64_t ld_out, uint64_t out_base, void *stream);

/* GPU brute-force oracle (the product's `verify`): replaces
 * _kernels.constant_row_flags / pcc_naive_pair / naive_allpairs_packed
 * (_kernels.py:255-298), bit for bit.  pcc_row_stats_f64 computes, per row
 * of x (n x l, stride ldx), is_constant, mean = sum8/l and ssd = ssd8 in the
 * reference's order; pcc_naive_pairs_f64 then evaluates the definition for
 * packed job ids [id_lo, id_hi) into out[id - id_lo]. */
int pcc_row_stats_f64(const double *x, int64_t ldx, int64_t n, int64_t l, double *mean, double *ssd,
                      uint8_t *constant, void *stream);
int pcc_naive_pairs_f64(const double *x, int64_t ldx, int64_t n, int64_t l, const double *mean,
                        const double *ssd, const uint8_t *constant, uint64_t id_lo, uint64_t id_hi,
                        double *out, void *stream);

/* Diagnostics (host only, no GPU): the order in which the production
 * contraction visits the GPU tiles [tile_begin, tile_end) -- partial first
 * row, full rows in groups of `group` rows walked column by column, partial
 * last row.  Writes the (Y, X) tile coordinates of schedule slots
 * 0 .. tile_end - tile_begin - 1. */
int pcc_tile_schedule(int64_t n, uint64_t tile_begin, uint64_t tile_end, uint32_t group, uint64_t *ys,
                      uint64_t *xs);

/* Diagnostics: number of kernels pcc_syrk_f64 launches for the GPU tiles
 * [tile_begin, tile_end) on the current device (the main persistent kernel
 * and, when the last partial wave is small, the 64 x 64 quadrant tail
 * kernel: 0, 1 or 2).  bench.py's gpu_launches count. */
int pcc_syrk_launches(int64_t n, uint64_t tile_begin, uint64_t tile_end, int32_t *launches);

/* Diagnostics: measured FP64 tensor-pipe (DMMA) throughput of the current
 * device in TFLOP/s, from a register-resident mma.sync f64 loop (~20 ms).
 * Used by bench.py as the live roofline denominator. */
int pcc_probe_fp64_peak(double *tflops);

#ifdef __cplusplus
}
#endif

#endif /* PCC_B200_H */
