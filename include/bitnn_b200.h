/*
 * bitnn_b200.h — C ABI of the B200-native binary forward pass.
 *
 * Drop-in boundary for the packed backend of the reference `bitnn`
 * (/root/reference/pkg/src/bitnn).  Every entry point replaces one
 * reference Numba kernel (`_kernels.py`) or one fused stage of the
 * packed network (`network.py`), with the same data layout:
 *
 *   - packed lines are uint64 words, LSB-first, +1 -> bit 1, -1 -> bit 0,
 *     each line padded to whole words with ZERO padding bits;
 *   - every kernel writes its whole `out` (caller-provided, no
 *     allocation inside), like the reference's caller-provided `out`
 *     arrays (_kernels.py:15-16);
 *   - a leading `batch` argument runs the same kernel over `batch`
 *     independent images laid out back to back (the reference is
 *     batch-1 only, network.py:506-522).
 *
 * All pointers are DEVICE pointers unless named `h_*`; `stream` is a
 * cudaStream_t passed as void*.  Return value: 0 on success, otherwise a
 * cudaError_t code (or B2_EINVAL for bad arguments); no entry point
 * synchronizes the device.
 *
 * No torch types cross this boundary; the Python host layer
 * (paper_1705_07175_b200/) binds it through ctypes.
 */
#ifndef BITNN_B200_H
#define BITNN_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define B2_EINVAL 1000

/* Threshold plan of one batchnorm+sign stage, already on the device.
 * thresh:   int32 per channel, clamped to [-(B+1), B+1] where B bounds |acc|
 *           (exact — see DESIGN.md "threshold clamping"); used by the fused
 *           GEMM epilogues whose accumulators are int32;
 * thresh64: the unclamped int64 thresholds (sentinels +-2^62), used by the
 *           generic threshold-pack kernel (int64 / uint8 inputs);
 * ge_dir:   uint8 per channel, 1 -> bit = acc >= t, 0 -> bit = acc <= t.
 * Replaces BatchNormLayer.thresh/ge_dir (layers.py:146-191). */
typedef struct b2_thresh {
  const int32_t* thresh;
  const int64_t* thresh64;
  const uint8_t* ge_dir;
} b2_thresh;

/* ---------------------------------------------------------------- version */
const char* b2_version(void);
/* Number of kernel launches issued through this library since load
 * (host-side counter, for the bench's gpu_launches claim). */
int64_t b2_launch_count(void);
/* Programmatic dependent launch (each kernel's launch and prologue overlap
 * the previous kernel on the stream): 1 on, 0 off.  Initially on unless the
 * environment sets B2_PDL=0.  Returns the previous setting.  Launches
 * already captured into a CUDA graph keep the setting they were made with. */
int b2_set_pdl(int on);

/* ---------------------------------------------------------------- packing */

/* _kernels.py:43-54 pack_lines: bit = !(x < 0) (0.0, -0.0, NaN -> 1).
 * lines (n_lines, bits) float32 row-major -> out (n_lines, ceil(bits/64)). */
int b2_pack_lines_f32(const float* lines, int64_t n_lines, int64_t bits, uint64_t* out, void* stream);

/* _kernels.py:57-64 unpack_lines: -> +/-1.0 float32 (n_lines, bits). */
int b2_unpack_lines_f32(const uint64_t* words, int64_t n_lines, int64_t bits, float* out, void* stream);

/* _kernels.py:67-82 pack_byte_planes: uint8 (n_lines, bits) ->
 * out (8, n_lines, ceil(bits/64)). */
int b2_pack_byte_planes(const uint8_t* lines, int64_t n_lines, int64_t bits, uint64_t* out, void* stream);

/* ---------------------------------------------------------------- GEMM */

/* _kernels.py:85-106 bgemm_packed: out[m,n] = k - 2*popc(a_m XOR b_n), int32.
 * a (m, wpl) row-packed, b (n, wpl) column-packed (both K-major), out (m, n). */
int b2_bgemm(const uint64_t* a, int64_t m, const uint64_t* b, int64_t n, int64_t wpl, int32_t k, int32_t* out,
             void* stream);

/* _kernels.py:109-117 bgemv_packed, batched over `batch` activation lines:
 * out[i, u] = k - 2*popc(w_u XOR x_i); w (units, wpl), x (batch, wpl). */
int b2_bgemv(const uint64_t* w, int64_t units, int64_t wpl, const uint64_t* x, int64_t batch, int32_t k, int32_t* out,
             void* stream);

/* _kernels.py:120-147 count_plane_bits + bitplane_matvec, batched:
 * planes (8, batch, wpl) as written by b2_pack_byte_planes -> out (batch,
 * units) int64, w (units, wpl). */
int b2_bitplane_gemv(const uint64_t* planes, int64_t batch, const uint64_t* w, int64_t units, int64_t wpl,
                     int64_t* out, void* stream);

/* ---------------------------------------------------------------- conv */

/* _kernels.py:170-199 unroll_packed (bit im2col), batched: lines of `batch`
 * images (channel axis iff c > 1, tensor.py:165-166) -> out
 * (batch * h_out * w_out, ceil(kh*kw*c/64)); OOB window sites stay 0 bits. */
int b2_unroll_packed(const uint64_t* lines, int64_t batch, int h, int w, int c, int kh, int kw, int stride, int pad,
                     uint64_t* out, void* stream);

/* layers.py:224-252 compute_correction from packed filter lines
 * (filters, ceil(kh*kw*c/64)) -> corr (h_out*w_out, filters) int32. */
int b2_conv_correction(const uint64_t* wwords, int64_t filters, int h, int w, int c, int kh, int kw, int stride,
                       int pad, int32_t* corr, void* stream);

/* layers.py:255-266 conv_forward / network.py:193-198 _PackedConv.run,
 * batched, int32 output (batch, h_out, w_out, filters), correction added.
 * `scratch` must hold batch*h_out*w_out*ceil(kh*kw*c/64) uint64 words when
 * the implicit-im2col fast path does not apply (c % 32 != 0); pass NULL
 * otherwise (b2_conv_scratch_words tells). */
int64_t b2_conv_scratch_words(int64_t batch, int h, int w, int c, int kh, int kw, int stride, int pad);
int b2_conv_forward(const uint64_t* lines, int64_t batch, int h, int w, int c, const uint64_t* wwords,
                    int64_t filters, int kh, int kw, int stride, int pad, const int32_t* corr, uint64_t* scratch,
                    int32_t* out, void* stream);

/* layers.py:265 / network.py:197 `acc += correction`, batched:
 * acc[i] += corr[i % per_image] for i < n (corr broadcast over images). */
int b2_add_correction_i32(int32_t* acc, const int32_t* corr, int64_t n, int64_t per_image, void* stream);

/* Fused conv stage: implicit-im2col XOR-popc GEMM + correction +
 * [2x2/2 max-pool when pool != 0] + batchnorm-threshold + sign + repack,
 * i.e. network.py _PackedConv -> _Pool -> _PackedBN in one kernel.
 * Requires c % 32 == 0 (site lines are whole uint32 words) and, with
 * pool, even h_out/w_out.  out: (batch, sites_out, ceil(filters/64)) words.
 * Returns B2_EINVAL when the shape is not eligible (use the unfused ops). */
int b2_conv_bn_pack(const uint64_t* lines, int64_t batch, int h, int w, int c, const uint64_t* wwords,
                    int64_t filters, int kh, int kw, int stride, int pad, const int32_t* corr, int pool, b2_thresh th,
                    uint64_t* out, void* stream);

/* ---------------------------------------------------------------- epilogues */

/* _kernels.py:224-240 maxpool on int32 (batch, h, w, c) -> (batch, ho, wo, c). */
int b2_maxpool_i32(const int32_t* x, int64_t batch, int h, int w, int c, int ph, int pw, int stride, int32_t* out,
                   void* stream);

/* _kernels.py:243-267 threshold_sign_pack, batched; x (batch, sites, c) of
 * dtype xkind (0 int32, 1 int64, 2 uint8).  flat=0: out (batch, sites,
 * ceil(c/64)); flat=1: out (batch, ceil(sites*c/64)) in layout order. */
int b2_threshold_pack(const void* x, int xkind, int64_t batch, int64_t sites, int64_t c, b2_thresh th, int flat,
                      uint64_t* out, void* stream);

/* _kernels.py:285-295 bn_affine: (double(x) - mean) * scale + beta, three
 * separately rounded IEEE ops (no FMA), x (n) of xkind (0 int32, 1 int64,
 * 3 float64), channel = i % c -> out (n) float64. */
int b2_bn_affine_f64(const void* x, int xkind, int64_t n, const double* mean, const double* scale,
                     const double* beta, int64_t c, double* out, void* stream);

/* layers.py:137-191 BatchNormLayer: float64 scale = gamma/sqrt(var+eps) and
 * the integer threshold by binary search (sentinels ALWAYS=-2^62,
 * NEVER=2^62), on the device.  Inputs float32 (c); outputs scale64 (c)
 * float64, thresh64 (c) int64, ge_dir (c) uint8, and thresh32 (c) int32 =
 * clamp(thresh64, -(bound+1), bound+1). */
int b2_bn_calibrate(const float* mean, const float* var, const float* gamma, const float* beta, double eps, int64_t c,
                    int64_t bound, double* scale64, int64_t* thresh64, uint8_t* ge_dir, int32_t* thresh32,
                    void* stream);

/* ---------------------------------------------------------------- fused dense */

/* network.py _PackedDense -> _PackedBN (flat): batched XOR-popc GEMM with
 * fused threshold + repack.  x (batch, wpl) activation lines, w (units,
 * wpl) -> out (batch, ceil(units/64)) packed words. */
int b2_dense_bn_pack(const uint64_t* x, int64_t batch, const uint64_t* w, int64_t units, int64_t wpl, int32_t k,
                     b2_thresh th, uint64_t* out, void* stream);

/* network.py _PackedInput8 -> _PackedBN (flat): uint8 images (batch, k)
 * -> bit-planes -> AND-popc GEMM -> threshold + repack, one kernel.
 * w (units, ceil(k/64)) -> out (batch, ceil(units/64)). */
int b2_input8_bn_pack(const uint8_t* x, int64_t batch, int64_t k, const uint64_t* w, int64_t units, b2_thresh th,
                      uint64_t* out, void* stream);

/* network.py _PackedByteBN (first-layer byte batchnorm) fused with the
 * first conv (_PackedConv, kh*kw*c <= 32 bits per window) and its
 * batchnorm (_PackedBN), one kernel: uint8 (batch, h, w, c) ->
 * out (batch, h_out*w_out, ceil(filters/64)) words (filters <= 1024).
 * Padding is handled by masking the out-of-bounds window bits, which equals
 * the reference's pad-as--1 product plus its correction map exactly. */
int b2_byte_conv_bn_pack(const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in,
                         const uint64_t* wwords, int64_t filters, int kh, int kw, int stride, int pad,
                         b2_thresh th_out, uint64_t* out, void* stream);

/* ---------------------------------------------------------------- tensor-core path
 *
 * The same operators on the 5th-generation tensor cores (tcgen05.mma
 * kind::i8): a bit encodes +1/-1, so popc-XOR dot products are int8 dot
 * products of +/-1 bytes with 0 for every element outside the operand
 * (padding), computed exactly in int32.  Activations stay bit-packed in HBM
 * and are widened on chip; weights are widened once (b2_expand_i8).  See
 * DESIGN.md "tensor-core binary GEMM".  Zero padding makes the reference's
 * correction map (layers.py:224-252) implicit: conv results already equal
 * conv_forward's "bgemm + correction". */

/* K rounded up to the 512-element granule of the tcgen05 int8 GEMM weight rows. */
int64_t b2_i8_kpad(int64_t k);

/* Widen packed +/-1 lines to int8 for the tensor pipe (_kernels.py:57-64
 * unpack_lines semantics, signed bytes): w (rows, wpl) with k valid bits ->
 * out (rows, b2_i8_kpad(k)) int8, +1 / -1 for k' < k and 0 for the padding.
 * permute=1: K order permuted inside each 32-group to match the on-chip
 * widening of packed A operands (all bit-packed entry points below);
 * permute=0: natural K order (b2_tc_input8_bn_pack, whose A is raw bytes). */
int b2_expand_i8(const uint64_t* w, int64_t rows, int64_t wpl, int64_t k, int permute, int8_t* out, void* stream);

/* _kernels.py:85-106 bgemm_packed: a (m, wpl) packed rows, b_i8 =
 * b2_expand_i8(permute=1) of the (n, wpl) packed columns -> out (m, n) int32
 * = k - 2*popc(a_m XOR b_n). */
int b2_tc_bgemm(const uint64_t* a, int64_t m, const int8_t* b_i8, int64_t n, int64_t wpl, int32_t k, int32_t* out,
                void* stream);

/* network.py _PackedDense -> _FinalBN: the last dense layer with the final
 * float64 batch-norm (_kernels.py:285-295 bn_affine, three separately
 * rounded ops, no FMA) in its epilogue: out (batch, units) float64 scores.
 * mean/scale/beta: float64 per unit, as b2_bn_affine_f64. */
int b2_tc_dense_affine_f64(const uint64_t* x, int64_t batch, const int8_t* w_i8, int64_t units, int64_t wpl,
                           int32_t k, const double* mean, const double* scale, const double* beta, double* out,
                           void* stream);

/* network.py _PackedDense -> _PackedBN (flat), as b2_dense_bn_pack. */
int b2_tc_dense_bn_pack(const uint64_t* x, int64_t batch, const int8_t* w_i8, int64_t units, int64_t wpl, int32_t k,
                        b2_thresh th, uint64_t* out, void* stream);

/* layers.py:255-266 conv_forward (correction included), implicit bit-im2col,
 * batched; requires c % 64 == 0.  out (batch, h_out, w_out, filters) int32. */
int b2_tc_conv_forward(const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* w_i8,
                       int64_t filters, int kh, int kw, int stride, int pad, int32_t* out, void* stream);

/* _PackedConv [-> _Pool 2x2/2] -> _PackedBN, as b2_conv_bn_pack; c % 64 == 0. */
int b2_tc_conv_bn_pack(const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* w_i8,
                       int64_t filters, int kh, int kw, int stride, int pad, int pool, b2_thresh th, uint64_t* out,
                       void* stream);

/* _PackedInput8 -> _PackedBN (flat): uint8 (batch, k) x +/-1 weights
 * (b2_expand_i8 permute=0) = the bit-plane sum of gemm.py:120-146 exactly,
 * then threshold + repack; k % 4 == 0. */
int b2_tc_input8_bn_pack(const uint8_t* x, int64_t batch, int64_t k, const int8_t* w_i8, int64_t units, b2_thresh th,
                         uint64_t* out, void* stream);

/* _PackedByteBN -> _PackedConv [-> _Pool 2x2/2] -> _PackedBN, as
 * b2_byte_conv_bn_pack (kh*kw*c <= 128, c <= 8).  Two launches: the byte batchnorm
 * + bit im2col (_kernels.py:170-199) of every output pixel into `scratch`
 * (b2_tc_byte_conv_scratch_bytes bytes: window bits plus a validity mask,
 * padding cells invalid), then the tensor-core GEMM with zero padding. */
/* Kernel b2_tc_byte_conv_bn_pack (int8 weights) runs for these arguments:
 * 1 = the fused first-layer kernel (one launch, `scratch` unused): stride 1,
 * odd kh == kw with pad = (kh - 1) / 2, c <= 3, kh*kw*c <= 31, <= 256 filters,
 * no pool, w a power of two dividing 128, h*w a multiple of 128, and an
 * image row of w*c bytes that is a multiple of 16 and at most 256; the
 * window and the output threshold go through ONE int8 MMA per 128 pixels;
 * 0 = the byte unroll into `scratch` + the tensor-core GEMM (two launches);
 * -1 = invalid arguments.  B2_BYTECONV_FUSED=0 disables the fused kernel. */
int b2_tc_byte_conv_path(int64_t batch, int h, int w, int c, int64_t filters, int kh, int kw, int stride, int pad,
                         int pool);
int64_t b2_tc_byte_conv_scratch_bytes(int64_t batch, int h, int w, int c, int kh, int kw, int stride, int pad);
int b2_tc_byte_conv_bn_pack(const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in,
                            const int8_t* w_i8, int64_t filters, int kh, int kw, int stride, int pad, int pool,
                            b2_thresh th_out, void* scratch, uint64_t* out, void* stream);

/* ---------------------------------------------------------------- fp4 tensor-core path
 *
 * The same operators on tcgen05.mma kind::mxf4: +1 / -1 / 0 are exact e2m1
 * values (0x2 / 0xA / 0x0), the block scales are all 2^0, and the fp32
 * accumulator holds the exact integer dot product (|dot| < 2^24; the b2_tc4_*
 * entry points return B2_EINVAL for K > 2^22, the epilogue's exact float ->
 * int conversion).  Twice the
 * int8 MMA rate and half the operand bytes.  Weights come from
 * b2_expand_f4; each b2_tc4_X takes exactly the arguments of b2_tc_X with
 * its weight pointer in that format.  Results are identical to b2_tc_X. */

/* K rounded up to the 1024-element granule of the fp4 weight rows. */
int64_t b2_f4_kpad(int64_t k);

/* Packed +/-1 lines -> e2m1 nibbles for the fp4 path: w (rows, wpl) with k
 * valid bits -> out (rows, b2_f4_kpad(k) / 2) bytes; K permuted inside each
 * 32-group like the on-chip widening of the A operand; 0 beyond k. */
int b2_expand_f4(const uint64_t* w, int64_t rows, int64_t wpl, int64_t k, uint8_t* out, void* stream);

int b2_tc4_bgemm(const uint64_t* a, int64_t m, const int8_t* b_f4, int64_t n, int64_t wpl, int32_t k, int32_t* out,
                 void* stream);
int b2_tc4_dense_affine_f64(const uint64_t* x, int64_t batch, const int8_t* w_f4, int64_t units, int64_t wpl,
                            int32_t k, const double* mean, const double* scale, const double* beta, double* out,
                            void* stream);
int b2_tc4_dense_bn_pack(const uint64_t* x, int64_t batch, const int8_t* w_f4, int64_t units, int64_t wpl, int32_t k,
                         b2_thresh th, uint64_t* out, void* stream);
int b2_tc4_conv_forward(const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* w_f4,
                        int64_t filters, int kh, int kw, int stride, int pad, int32_t* out, void* stream);
/* Kernel choice of b2_tc4_conv_bn_pack (same results on every path; the
 * call allocates nothing):
 *  - stride-1 same-size convs with odd kh == kw, pad = (kh - 1) / 2,
 *    c % 128 == 0, <= 256 filters, w a power of two dividing 128, h*w a
 *    multiple of 128 (pooled: 128 / w even), weights plus >= 2 band slots in
 *    shared memory and >= one 128-pixel tile per SM: the ROW-ALIGNED
 *    padded-row implicit GEMM, pooling fused into its epilogue (DESIGN.md
 *    §3.1b); 129-256 filters run as two 128-filter launches (each writes its
 *    own output words; B2_ALIGN_SPLIT=0 keeps one 256-column launch where it
 *    fits);
 *  - otherwise unpooled stride-1 same-size convs with c % 128 == 0, <= 256
 *    filters (K <= 1536 up to 128 filters, <= 1280 above), a band the producer
 *    warps cover (c = 128: w <= 190), weights resident, and enough virtual
 *    rows to fill the GPU: the virtual-grid padded-row kernel;
 *  - everything else: the implicit-im2col kernel (pool fused in its epilogue),
 *    or cluster split-K for few-tile launches with deep K.
 * B2_PADROW=0 / B2_PADROW_ALIGN=0 in the environment disable the padded-row
 * kernels.  b2_tc4_conv_path returns the path a call with these arguments
 * takes: 0 im2col, 1 split-K, 2 padded-row, 3 row-aligned padded-row (-1:
 * invalid arguments). */
int b2_tc4_conv_path(int64_t batch, int h, int w, int c, int64_t filters, int kh, int kw, int stride, int pad,
                     int pool);
int b2_tc4_conv_bn_pack(const uint64_t* lines, int64_t batch, int h, int w, int c, const int8_t* w_f4,
                        int64_t filters, int kh, int kw, int stride, int pad, int pool, b2_thresh th, uint64_t* out,
                        void* stream);
int b2_tc4_byte_conv_bn_pack(const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in,
                             const int8_t* w_f4, int64_t filters, int kh, int kw, int stride, int pad, int pool,
                             b2_thresh th_out, void* scratch, uint64_t* out, void* stream);

/* Byte-BN first layer on the padded-row fp4 kernel (_PackedByteBN ->
 * _PackedConv [-> _Pool 2x2/2] -> _PackedBN, as b2_byte_conv_bn_pack):
 * stride 1, odd kh == kw, pad = (kh - 1) / 2, c <= 8, filters <= 128.  The
 * image is thresholded per channel while the band is built (no unrolled
 * scratch); each window cell is one K=64 MMA.  Weights in the per-cell
 * layout of b2_expand_f4_cells: rows of b2_f4_cells_row_bytes(kh * kw)
 * bytes (per cell 64 e2m1 elements, the cell's c channel bits then zeros).
 * Pooled calls take a stream-ordered scratch like b2_tc4_conv_bn_pack.
 * Also B2_EINVAL: a tile's band over 512 rows (w > 190 for 3x3: the
 * producer warps cover one band row per thread) and weights plus the band
 * ring over 227 KB of shared memory (e.g. any 7x7 window: 13 weight atoms).
 * Measured on BCNN conv1 (3 channels): 0.60 ms vs 0.36 ms for
 * b2_tc_byte_conv_bn_pack (nine K=64 MMAs per tile with 3 useful elements
 * each), so the network keeps the unrolled path; this entry is an opt-in
 * for wider first layers. */
int64_t b2_f4_cells_row_bytes(int cells);
int b2_expand_f4_cells(const uint64_t* w, int64_t rows, int64_t wpl, int cells, int c, uint8_t* out, void* stream);
int b2_tc4_byte_conv_padrow(const uint8_t* x, int64_t batch, int h, int w, int c, b2_thresh th_in,
                            const uint8_t* w_cells, int64_t filters, int kh, int kw, int pad, int pool,
                            b2_thresh th_out, uint64_t* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* BITNN_B200_H */
