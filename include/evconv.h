/*
 * evconv.h -- C ABI of libevconv.so, the sm_100a implementation of EvConv's
 * incremental inference path (arXiv 2303.04670).
 *
 * The reference (evincr 0.1.0, /root/reference/pkg/src/evincr) is pure
 * Python + numpy and has no FFI; its "operator API" is the set of Python
 * functions in increment_ops.py / sparsify.py / tensors.py / events.py that
 * Graph.incr_step (graph.py:573-630) dispatches to.  Each entry point below
 * replaces one of those functions (cited per function); the Python package
 * paper_2303_04670_b200 binds them with ctypes and keeps the reference names
 * and signatures.  See INTEGRATION.md for the binding.
 *
 * Conventions
 *  - Plain C types only: device pointers, int32/int64 sizes, cudaStream_t
 *    (passed as void*).  No torch types cross this boundary.
 *  - Every entry point is asynchronous on `stream`, never allocates, never
 *    synchronises, and is safe to record into a CUDA graph.  Host-visible
 *    results (FLOP meters, counts, norms) are written to device memory.
 *  - Return 0 on success or a negative EVC_E* code; evc_last_error() returns
 *    a thread-local message for the last failure.  Shape validation with the
 *    reference's exception texts happens in Python before the call.
 *  - Tensors are float32, channel-planar (C, H, W) exactly like the
 *    reference (tensors.py:1-6), with a leading "session" index s for
 *    batched independent streams.  Tile masks are uint8 (0/1) grids
 *    (C, ceil(H/th), ceil(W/tw)) like TileMask.flags (tensors.py:65-90).
 */
#ifndef EVCONV_H
#define EVCONV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVC_ABI_VERSION 3

enum {
  EVC_OK = 0,
  EVC_EINVAL = -1, /* bad argument */
  EVC_ECUDA = -2,  /* CUDA runtime error */
  EVC_ENOSPC = -3  /* workspace too small */
};

/* A batch of S increment tensors (one per session) sharing one shape.
 * value (s,c,h,w) lives at vals[s*vstride + (c*H + h)*W + w];
 * flag  (s,c,i,j) lives at flags[s*fstride + (c*GH + i)*GW + j],
 * GH = ceil(H/th), GW = ceil(W/tw).  vstride/fstride let a tensor be a
 * channel slice of a larger concat buffer (zero-copy inc_concat). */
typedef struct evc_tensor {
  float* vals;
  uint8_t* flags; /* NULL for dense (unmasked) tensors */
  int64_t vstride;
  int64_t fstride;
  int32_t C, H, W;
  int32_t th, tw;
} evc_tensor;

/* Static convolution geometry (ConvParams, increment_ops.py:58-77). */
typedef struct evc_conv_geom {
  int32_t c_in, c_out, kh, kw, stride, pad;
  int32_t H, W, Ho, Wo;
  int32_t th, tw;
} evc_conv_geom;

/* ---- library ---------------------------------------------------------- */
int evc_version(void);
const char* evc_last_error(void);
/* Loads every kernel module and sets smem attributes (call once, outside
 * graph capture). */
int evc_init(void);
/* Programmatic dependent launch for the step kernels: each kernel
 * may start while its predecessor on the stream drains and waits on the device
 * (griddepcontrol.wait) before reading upstream results.  Default off:
 * CUDA-graph replay already hides the launch latency (measured). */
int evc_set_pdl(int32_t on);

/* ---- tile masks (tensors.py) ------------------------------------------ */

/* step_increment (events.py:295-302) + make_tile_mask (tensors.py:93-107):
 * out.vals = cur - prev, out.flags = exact per-tile any(!=0).
 * prev/cur are dense batches with per-session stride `in_stride`. */
int evc_diff_mask(const float* prev, const float* cur, int64_t in_stride,
                  const evc_tensor* out, int32_t S, void* stream);

/* make_tile_mask (tensors.py:93-107): recompute t.flags from t.vals. */
int evc_make_tile_mask(const evc_tensor* t, int32_t S, void* stream);

/* np.flatnonzero(flags) for n flags: ascending indices of nonzero bytes,
 * count written to *count.  Warp-ballot + block prefix scan in two
 * deterministic launches.  idx must hold n entries; scratch must hold
 * evc_compact_scratch(n) int32 entries. */
int64_t evc_compact_scratch(int64_t n);
int evc_compact(const uint8_t* flags, int64_t n, int32_t* idx, int32_t* count,
                int32_t* scratch, void* stream);

/* Per-session count of True flags of t (TileMask.false_fraction,
 * tensors.py:86-87; graph.py:632-636).  counts[s] (int32) is ACCUMULATED
 * into -- zero it first. */
int evc_count_flags(const evc_tensor* t, int32_t S, int32_t* counts, void* stream);

/* integrate (tensors.py:167-174, graph.py:615-616): y_run += dx on live
 * tiles.  y_run is a dense batch with stride y_stride. */
int evc_integrate(float* y_run, int64_t y_stride, const evc_tensor* dx,
                  int32_t S, void* stream);

/* Copy a masked tensor (values on live-or-previously-live tiles, flags)
 * into another (used when a concat part cannot be aliased). */
int evc_copy_masked(const evc_tensor* src, const evc_tensor* dst, int32_t S,
                    void* stream);

/* Dense strided copy of S x (C,H,W) float blocks. */
int evc_copy_dense(const float* src, int64_t src_stride, float* dst,
                   int64_t dst_stride, int64_t n_per_session, int32_t S,
                   void* stream);

/* Serving-path ingest of S sessions per step (events.py:35-37 records,
 * events.py:251-280 encodings).  Each session keeps its recent events in a device ring of `ring`
 * (power of two) slots per column; event with absolute index e lives at slot e & (ring - 1).
 * evc_ingest_ring: desc[s] = {first record of session s in `records`, count, absolute index of
 * its first new event}; records = the step's packed EVB records of all sessions, concatenated.
 * evc_encode_windows: win[s] = {lo, hi (absolute event indices), tau, delta}; writes count
 * (mode 1), timestamp (mode 2) or count + timestamp (mode 3, 4 channels) of every window into
 * out[s * out_stride] (zeroed here), bit-identical to encode(); max_events >= max(hi - lo). */
int evc_ingest_ring(const uint8_t* records, const int64_t* desc, int64_t max_new, int64_t ring, uint64_t* t,
                    uint16_t* x, uint16_t* y, int8_t* p, int32_t S, void* stream);
int evc_encode_windows(const uint64_t* t, const uint16_t* x, const uint16_t* y, const int8_t* p, int64_t ring,
                       const int64_t* win, int64_t max_events, int32_t H, int32_t W, int32_t mode, float* out,
                       int64_t out_stride, int32_t S, void* stream);

/* Input-stationary incremental conv (inc_conv2d increment_ops.py:156-194 value
 * path): live input tiles compacted, gathered into 3xTF32 tcgen05 tiles with every tap along N,
 * scattered into per-tile output patches and summed per output tile in a fixed order.  Values only:
 * output flags and the FLOP meter come from evc_conv_mask.  Geometry: stride 1, "same" output,
 * k <= 3, th * tw <= 36.  fresh_out != 0: the output buffer was zeroed since the last call (else only
 * tiles that held values and are dead now are rewritten with zeros). */
int evc_conv_scatter_supported(const evc_conv_geom* g);
int64_t evc_conv_scatter_pack_len(const evc_conv_geom* g);
int evc_conv_scatter_pack(const float* w, const evc_conv_geom* g, float* out);
int64_t evc_conv_scatter_workspace(const evc_conv_geom* g, int32_t S);
int evc_conv_scatter(const evc_conv_geom* g, const evc_tensor* in, const float* wpack, const evc_tensor* out,
                     void* workspace, int64_t ws_bytes, int32_t fresh_out, int32_t S, void* stream);

/* Strided byte copy of S blocks of `nbytes` (cudaMemcpy2DAsync, capturable in a CUDA
 * graph): the recurrent delay node's pending increment (values and tile flags) moved
 * between its state buffers and its output slot. */
int evc_copy_bytes(const void* src, int64_t src_stride, void* dst, int64_t dst_stride,
                   int64_t nbytes, int32_t S, void* stream);

/* Graph.drift (graph.py:646-654): out[s] = max|a - b| (float32 bits kept
 * exact).  out must be zeroed first. */
int evc_max_abs_diff(const float* a, int64_t a_stride, const float* b,
                     int64_t b_stride, int64_t n_per_session, int32_t S,
                     float* out, void* stream);

/* ---- convolution (increment_ops.py:126-194, tensors.py:205-228) ------- */

/* Host helper: length (int32 entries) of the static per-layer table used
 * by the mask/meter and gather kernels, and its contents.  Upload the
 * table to device memory once per layer. */
int64_t evc_conv_table_len(const evc_conv_geom* g);
int evc_conv_table_fill(const evc_conv_geom* g, int32_t* host_table);

/* Mask propagation + FLOP meter of inc_conv2d for a batch (two launches):
 *  - in_true[s] += number of True input flags (TileMask.false_fraction and
 *    the all-false / all-true shortcuts, increment_ops.py:148-154),
 *  - writes out.flags (broadcast over C_out, increment_ops.py:193-194) and
 *    zeroes output tiles that were live last step and are dead now,
 *  - appends every live output tile (s*T + t, T = output tiles per session)
 *    to tile_list and counts them in *tile_count (work list of
 *    evc_conv_gemm; the GEMM result does not depend on list order),
 *  - meter[s] += performed FLOPs (int64, the exact reference meter).
 * With region_flags != NULL it also sets region_flags[s][ri*RWn + rj] = 1
 * for every 4x32 output region (rows of 4, columns of 32) overlapping a live
 * tile.  tile_list/tile_count may be NULL when only regions are wanted.
 * scratch (evc_conv_mask_scratch int32 entries), in_true, tile_count and
 * region_flags must be zeroed before the call.  `table` is the device copy
 * of evc_conv_table_fill's output. */
int64_t evc_conv_mask_scratch(const evc_conv_geom* g, int32_t S);
int evc_conv_mask(const evc_conv_geom* g, const evc_tensor* in,
                  const evc_tensor* out, const int32_t* table,
                  int32_t* scratch, int32_t* in_true, int32_t* tile_list,
                  int32_t* tile_count, uint8_t* region_flags, int64_t* meter,
                  int32_t S, void* stream);

/* Channels-innermost hi/lo shadow of a conv input (hwc.cu).  The buffer holds
 * (H + 2 pad) x (W + 2 pad) pixels of 2*cp floats (cp = evc_hwc_channels(C_in)):
 * TF32 heads and tails; the border stays zero (the conv's padding).  Producers get
 * y = the interior origin (pixel (0, 0)) and pitch = W + 2 pad; pixel (s, y, x) starts at
 * y[s*stride + (y*pitch + x)*2cp].  Within a pixel, for cp a multiple of 32 (TMA path):
 * 32-channel chunks [32 heads | 32 tails], channel c's head at (c/32)*64 + c%32 and its
 * tail 32 floats later; otherwise (CUDA-core path) heads at c, tails at cp + c.
 * A negative cp selects the fp32 shadow of -cp channels read only by the CUDA-core (thin)
 * conv: -cp floats per pixel, channel c's value at c (half the bytes; every producer taking
 * cp -- to_hwc, sparsify, up_sparsify, the fused conv sparsify -- writes either layout). */
int32_t evc_hwc_channels(int32_t c);
int evc_to_hwc(const evc_tensor* x, float* y, int64_t y_stride, int32_t cp,
               int32_t pitch, int32_t S, void* stream);

/* ---- fused incremental convolution (conv_fused.cu) --------------------
 * inc_conv2d (increment_ops.py:126-194) in ONE launch: region test against the
 * any-channel input tile map, output tile flags, the exact FLOP-meter terms,
 * the TMA/tcgen05 3xTF32 GEMM over live RH x RW output regions, split-K over a
 * thread-block cluster reduced deterministically through DSMEM, and optionally
 * the activation delta of the following inc_activation (increment_ops.py:232-238)
 * in the epilogue.  Launch configuration: */
typedef struct evc_conv_cfg {
  int32_t bn;     /* output channels per CTA: 16, 32, 64, 128 or 256 */
  int32_t rh, rw; /* tap mode: output region rows x cols, rh * rw = 128, rw in {8, 16, 32} */
  int32_t splits; /* K-splits = cluster size along z, 1..16 */
  int32_t row;    /* 1: row mode (stride 1): regions = 128 consecutive sites of the output grid
                     flattened with pitch W + 2 pad; a K-block is one kernel row x 32 channels,
                     loaded once (128 + kw - 1 shadow pixels) for all kw taps */
  int32_t thin;   /* 1: CUDA-core fp32 path (C_in <= 8 or C_out <= 8, C_out <= 32), tap-mode regions */
  int32_t drain;  /* > 0: K-blocks per TMEM accumulation segment -- every segment's partial sum is promoted
                     into fp32 registers of the epilogue warps (RN adds) while the MMAs fill the other of
                     two accumulator blocks, so no tensor-core accumulation chain is longer than one
                     segment; 0: one chain per accumulator block (the config sets 1 in row mode, 2 in
                     tap / packed mode; the dense pass never runs with 0) */
} evc_conv_cfg;

/* 1 if the fused path handles this geometry (pad < kernel, stride <= 8). */
int evc_conv_fused_supported(const evc_conv_geom* g);
/* Heuristic launch configuration for S sessions (max_splits <= 0: 8). */
int evc_conv_fused_config(const evc_conv_geom* g, int32_t S, int32_t max_splits, evc_conv_cfg* cfg);
/* Pre-split (TF32 hi / lo), 128B-swizzled, K-major weight images (floats). */
int64_t evc_conv_fused_pack_len(const evc_conv_geom* g, const evc_conv_cfg* cfg);
int evc_conv_fused_pack(const float* w, const evc_conv_geom* g, const evc_conv_cfg* cfg, float* out);
/* Bytes of the persistent per-(session, region, channel block) "computed last
 * step" state; zero it whenever the output increment buffers are zeroed. */
int64_t evc_conv_fused_state_len(const evc_conv_geom* g, const evc_conv_cfg* cfg, int32_t S);
/* in_hwc: channels-innermost shadow of the input (see evc_to_hwc).
 * Incremental mode (dense == 0): `in` supplies the per-channel input flags,
 * fany[s][tile] the any-channel map (evc_tile_any, or written by the producing
 * sparsify), table = evc_conv_table_fill output; every CTA writes its meter partial
 * meter_part[(s * evc_conv_fused_ctas + cta) * 2 + {0, 1}] (int64, no zeroing needed),
 * resolved by evc_meter_step.
 * Output flags are written to act_out when act >= 0, else to out.
 * out may be NULL when act >= 0 (the conv values are then not materialised);
 * act_out->vals may be NULL when sp != NULL (the activation is only read through
 * the fused sparsify).
 * Dense mode (dense != 0): every region, bias added; with act >= 0 the
 * activation y = f(x) is written to act_out and acc = x when acc != NULL. */
/* Optional fused sparsify_step at t_p = 0 (sparsify.py:54-78) of the conv (or fused
 * activation) output, when that sparsify's only reader is another fused conv: the
 * epilogue writes that conv's hi/lo shadow, the sparsify's per-channel tile flags and
 * the any-channel map (both must be zeroed per step; only ever set to 1), and one
 * sum of squares per CTA (partials[s * evc_conv_fused_ctas(g, cfg) + cta]) for the
 * deferred norm fold of evc_meter_step. */
typedef struct evc_conv_sparsify {
  float* hwc; /* interior origin of the next conv's shadow (see evc_to_hwc) */
  int64_t hwc_stride;
  int32_t cp;
  int32_t pitch;
  uint8_t* flags;
  int64_t fstride;
  uint8_t* fany;
  double* partials;
} evc_conv_sparsify;
int64_t evc_conv_fused_ctas(const evc_conv_geom* g, const evc_conv_cfg* cfg); /* per session */
int evc_conv_fused(const evc_conv_geom* g, const evc_conv_cfg* cfg, const float* in_hwc, int32_t cp,
                   int64_t hwc_stride, const float* wpack, const float* bias, const evc_tensor* in,
                   const uint8_t* fany, const int32_t* table, uint8_t* rstate, int64_t* meter_part,
                   const evc_tensor* out, int32_t act, float alpha, float* acc,
                   int64_t acc_stride, const evc_tensor* act_out, const evc_conv_sparsify* sp,
                   int32_t dense, int32_t S, void* stream);
/* Sub-pixel form of "2x bilinear upsample -> sparsify(t_p = 0) -> 3x3 stride-1 pad-1 conv"
 * (increment_ops.py:271-285 -> sparsify.py:54-78 -> increment_ops.py:126-194): the conv runs on
 * the LOW-RES input x with composed weights (4 x c_out channels, phase-minor: composed channel
 * 4 c + 2 a + b -> channel c at output site (2i + a, 2j + b)), reading the low-res shadow that
 * evc_subpixel_input writes (edges replicated into the ring) instead of the upsampled one.
 * g / cfg: the composed low-res conv (c_out = 4 x sub->c_out; channel block >= 64, not packed);
 * fany: the low-res tile map of evc_subpixel_input; table: the evc_conv_table_fill output of the
 * REAL (high-res) conv; in: the sparsify output (high-res flags, from evc_subpixel_input);
 * out / act_out / sp: high-res tensors as in evc_conv_fused.  Flags and meter are the real
 * conv's; values within fp32 rounding of it. */
typedef struct evc_conv_subpixel {
  int32_t c_out;          /* output channels of the real conv (multiple of 4); tiles th, tw even */
  int32_t Ho, Wo;         /* its output size = 2 x the composed conv's */
  int32_t reserved;
  const uint8_t* fany_in; /* any-channel tile map of the high-res conv input (incremental mode) */
  const float* border;    /* [S][2 (Ho + Wo)][c_out] border correction (evc_subpixel_border) */
} evc_conv_subpixel;
int evc_conv_fused_subpixel(const evc_conv_geom* g, const evc_conv_cfg* cfg, const float* in_hwc, int32_t cp,
                            int64_t hwc_stride, const float* wpack, const float* bias, const evc_tensor* in,
                            const uint8_t* fany, const int32_t* table, uint8_t* rstate, int64_t* meter_part,
                            const evc_tensor* out, int32_t act, float alpha, float* acc, int64_t acc_stride,
                            const evc_tensor* act_out, const evc_conv_sparsify* sp, const evc_conv_subpixel* sub,
                            int32_t dense, int32_t S, void* stream);
/* The sub-pixel conv's input pass in one launch over x (replaces evc_upsample_sparsify at
 * t_p = 0 for that conv): the low-res shadow (interior origin hwc, pitch >= W + 2, cp a multiple
 * of 32 >= C, the one-pixel ring = the replicated edge), fany_lo[s][tile] |= any channel flag of
 * x, and for the 2x bilinear upsample U(x) -- never stored -- the sparsify output y's flags (every
 * tile written: U != 0 anywhere in it, sparsify.py:77-78, evaluated where x's flags mark the
 * support), fany_hi[s][tile] |= any channel, and one sum of U^2 per CTA at
 * partials[s * evc_subpixel_input_partials(x, cp) + cta] (norm fold: evc_meter_step).  Tiles of x
 * and y equal and even. */
int64_t evc_subpixel_input_partials(const evc_tensor* x, int32_t cp);
int evc_subpixel_input(const evc_tensor* x, const evc_tensor* y, double* partials, float* hwc, int32_t cp,
                       int64_t hwc_stride, int32_t pitch, uint8_t* fany_lo, uint8_t* fany_hi, int32_t S,
                       void* stream);
/* Border correction of evc_conv_fused_subpixel: out[s][line][c] for the high-res lines row 0
 * (index X), row Ho - 1, column 0 (index Y), column Wo - 1, = - sum over the taps leaving the
 * image of w . U(clamped site); w = the real conv's weights transposed to (C, 3, 3, c_out)
 * (device), c_out a multiple of 4. */
int evc_subpixel_border(const evc_tensor* x, const float* w, int32_t c_out, float* out, int32_t S, void* stream);

/* evc_subpixel_input and evc_subpixel_border in ONE launch (both only read x; the border GEMM's CTAs are
 * scheduled between the input pass's).  Same arguments and results as the two calls; partials are
 * indexed exactly as evc_subpixel_input's (evc_subpixel_input_partials). */
int evc_subpixel_input_border(const evc_tensor* x, const evc_tensor* y, double* partials, float* hwc, int32_t cp,
                              int64_t hwc_stride, int32_t pitch, uint8_t* fany_lo, uint8_t* fany_hi, const float* w,
                              int32_t c_out, float* border, int32_t S, void* stream);
/* Debug: subsequent evc_conv_fused launches record per-CTA phase clocks into
 * buf (16 uint64 per CTA, CTA index (z*gy + y)*gx + x); NULL turns it off. */
int evc_conv_trace(void* buf);
/* fany[s][t] = OR over channels of x's flags (input of a fused conv whose
 * producer does not emit the map). */
int evc_tile_any(const evc_tensor* x, uint8_t* fany, int32_t S, void* stream);
/* One sparsify node's deferred norm fold: partials[s*n + b] are the per-CTA sums
 * of corrected^2 written by evc_sparsify / evc_upsample_sparsify called with
 * ticket == NULL; norm_ema[s], k[s] as in evc_sparsify. */
typedef struct evc_sp_node {
  const double* partials;
  int64_t n;
  double* norm_ema;
  double* k;
  double tp, decay;
} evc_sp_node;

/* One meter node (conv / linear) of the end-of-step bookkeeping. */
typedef struct evc_meter_node {
  const int64_t* part; /* fused conv: per-CTA partials [S][n][2] (live input flags, weighted
                          meter term) written by evc_conv_fused; NULL: in_true / perf_step of
                          this node are already final (linear, unfused conv) */
  int64_t n;           /* partials per session */
  int64_t nflags;      /* input tile flags per session */
  int64_t dense;       /* dense-equivalent FLOPs */
  int32_t c_out;
  int32_t reserved;
} evc_meter_node;

/* End-of-step bookkeeping in one launch (graph.py:617-636):
 *  - n meter nodes (nodes: DEVICE array) x S sessions: a fused conv's performed =
 *    0 / dense / 2*C_out*(weighted term) by its live-flag count (increment_ops.py:148-154,
 *    191), written to in_true[l*S + s] and perf_step; then perf_cum += perf_step and
 *    the false-tile fraction ff_last = 1 - in_true / nflags, ff_sum += ff_last;
 *  - n_sp sparsify nodes (sp_nodes: DEVICE array): norm_ema / k update from the
 *    deferred partial sums in a fixed order (sparsify.py:72-76). */
int evc_meter_step(const evc_meter_node* nodes, int32_t n, int32_t S, int32_t* in_true,
                   int64_t* perf_step, int64_t* perf_cum, double* ff_last, double* ff_sum,
                   const evc_sp_node* sp_nodes, int32_t n_sp, void* stream);

/* Workspace floats needed by evc_conv_gemm for `max_tiles` active output
 * tiles and `splits` K-splits. */
int64_t evc_conv_workspace(const evc_conv_geom* g, int64_t max_tiles, int32_t splits);

/* Gather -> GEMM -> scatter over active output tiles.
 * tile_list/tile_count: (s*T + t) entries (evc_conv_mask output, any order);
 * tile_list == NULL means every tile of every session (dense pass).
 * wpack != NULL selects the tcgen05 tensor-core kernel (3xTF32 split, fp32
 * TMEM accumulation) with weights pre-packed by evc_conv_tc_pack;
 * otherwise `weight` ((C_out, C_in, KH, KW) fp32 as stored by the reference,
 * graph.py:457-467) feeds the FFMA kernel.  bias may be NULL (increments
 * drop it).  splits > 1 uses the fp32 workspace and a deterministic
 * reduction. */
int evc_conv_gemm(const evc_conv_geom* g, const evc_tensor* in,
                  const float* weight, const float* wpack, const float* bias,
                  const evc_tensor* out, const int32_t* table,
                  const int32_t* tile_list, const int32_t* tile_count,
                  int32_t S, int32_t splits, float* workspace, void* stream);

/* Host helpers for the tensor-core path: pack (C_out, K) fp32 weights into
 * the pre-split (hi = TF32 truncation, lo = w - hi), 128B-swizzled,
 * K-major SMEM images streamed by cp.async.bulk (length in floats). */
int64_t evc_conv_tc_pack_len(int32_t c_out, int64_t K);
int evc_conv_tc_pack(const float* w, int32_t c_out, int64_t K, float* out);

/* ---- nonlinearities / elementwise (increment_ops.py:226-310) ---------- */

enum { EVC_ACT_RELU = 0, EVC_ACT_SIGMOID = 1, EVC_ACT_TANH = 2, EVC_ACT_LEAKY = 3 };

/* inc_activation (increment_ops.py:232-238): y = f(acc+dx) - f(acc);
 * acc += dx; y.flags = dx.flags.  acc is a dense batch (stride acc_stride). */
int evc_act_delta(const evc_tensor* dx, float* acc, int64_t acc_stride,
                  const evc_tensor* y, int32_t kind, float alpha, int32_t S,
                  void* stream);

/* Dense activation (graph.py:523-526): y = f(x); acc = x when acc != NULL. */
int evc_act_dense(const float* x, int64_t x_stride, float* y, int64_t y_stride,
                  float* acc, int64_t acc_stride, int64_t n_per_session,
                  int32_t kind, float alpha, int32_t S, void* stream);

/* sparsify_step (sparsify.py:54-78) for a batch.  k[s], norm_ema[s] are
 * float64 device scalars (SparsifyState.k / .norm_ema); delta is the
 * residual (dense batch); dlive (uint8, per tile) tracks tiles whose
 * residual is nonzero.  partials (float64, S*C*GH) receives per-CTA sums of
 * corrected^2; the last CTA to retire (ticket: zeroed int32) folds them into
 * norm_ema / k in a fixed order (sparsify.py:72-76), so the whole step is
 * one launch.  ticket == NULL leaves the fold to evc_meter_step (graph runtime:
 * one end-of-step launch for every sparsify node). */
int64_t evc_sparsify_partials(const evc_tensor* dx); /* per session */
int evc_sparsify(const evc_tensor* dx, float* delta, int64_t delta_stride,
                 uint8_t* dlive, const evc_tensor* y, double* k,
                 double* norm_ema, double tp, double ema_decay,
                 double* partials, int32_t* ticket, float* hwc, int32_t cp,
                 int64_t hwc_stride, int32_t hwc_pitch, uint8_t* fany, int32_t write_chw,
                 int32_t delta_zero, int32_t S, void* stream);
/* (hwc, cp, hwc_stride, hwc_pitch: optional channels-innermost hi/lo shadow of y
 * for the TMA conv GEMM, interior origin and row pitch as in evc_to_hwc; fany: optional any-channel tile map of y
 * for evc_conv_fused, only ever set to 1 -- zero it per step;
 * write_chw = 0 skips the planar y values --
 * flags are always written.  delta_zero != 0 asserts tp == 0 and k == 0, so
 * the residual stays identically zero and is neither read nor written.) */

/* Fused inc_upsample (increment_ops.py:271-285) -> sparsify_step: y is the
 * sparsified upsample of x, computed without materialising the upsampled
 * increment (arguments as evc_upsample + evc_sparsify; partials sized by
 * evc_upsample_sparsify_partials(y) per session). */
int64_t evc_upsample_sparsify_partials(const evc_tensor* y);
int evc_upsample_sparsify(const evc_tensor* x, int32_t factor, int32_t mode,
                          float* delta, int64_t delta_stride, uint8_t* dlive,
                          const evc_tensor* y, double* k, double* norm_ema,
                          double tp, double ema_decay, double* partials,
                          int32_t* ticket, float* hwc, int32_t cp,
                          int64_t hwc_stride, int32_t hwc_pitch, uint8_t* fany, int32_t write_chw,
                          int32_t delta_zero, int32_t S, void* stream);

/* acc += dx on live tiles (AccState.fold, increment_ops.py:93-94). */
int evc_fold(const evc_tensor* dx, float* acc, int64_t acc_stride, int32_t S,
             void* stream);

/* Norm / EMA / k update from partial sums (one CTA, all S sessions), or
 * the reset (sparsify.py:43-51) when reset != 0 (norm_ema = norm, and
 * k = tp*norm if tp > 0).  n_partials per session. */
int evc_sparsify_finalize(const double* partials, int64_t n_partials,
                          double* norm_ema, double* k, double tp,
                          double ema_decay, int32_t reset, int32_t S,
                          void* stream);

/* Per-session partial sums of x^2 for the dense reset norm:
 * partials[s*n_blocks + b]; returns blocks used in *n_blocks_out (host). */
int evc_sumsq_dense(const float* x, int64_t x_stride, int64_t n_per_session,
                    double* partials, int32_t n_blocks, int32_t S, void* stream);

/* Byte fill of n segments in one launch: the resets of a dense refresh (graph.py:503-565 rebuilds
 * every AccState; the increment stores, flag grids and conv shadows return to exact zeros).
 * `segs` is a DEVICE array of n entries; value is the fill byte (low 8 bits). */
typedef struct evc_fill_segment {
  uint64_t addr;
  int64_t bytes;
  int64_t value;
} evc_fill_segment;
int evc_fill_segments(const evc_fill_segment* segs, int32_t n, int32_t n_blocks, void* stream);

/* inc_add (increment_ops.py:226-229). */
int evc_add(const evc_tensor* a, const evc_tensor* b, const evc_tensor* y,
            int32_t S, void* stream);

/* inc_add followed by inc_activation (increment_ops.py:226-229 then :232-238) in one pass,
 * for an add whose only reader is the activation: s = a + b, y = f(acc + s) - f(acc),
 * acc += s, y.flags = a.flags | b.flags -- the same float32 ops as the two calls. */
int evc_add_act(const evc_tensor* a, const evc_tensor* b, float* acc, int64_t acc_stride,
                const evc_tensor* y, int32_t kind, float alpha, int32_t S, void* stream);

/* inc_mul (increment_ops.py:241-254): y = (acc_a+a)*b + acc_b*a. */
int evc_mul(const evc_tensor* a, const evc_tensor* b, float* acc_a,
            float* acc_b, int64_t acc_stride, const evc_tensor* y, int32_t S,
            void* stream);

/* Dense elementwise for the dense pass: op 0 = add, 1 = mul (graph.py:530-537). */
int evc_binary_dense(const float* a, int64_t a_stride, const float* b,
                     int64_t b_stride, float* y, int64_t y_stride,
                     int64_t n_per_session, int32_t op, int32_t S, void* stream);

/* inc_upsample (increment_ops.py:271-285) / dense_upsample
 * (tensors.py:259-282): mode 0 nearest, 1 bilinear.  When in->flags is
 * NULL the call is the dense operator (no masks). */
int evc_upsample(const evc_tensor* in, const evc_tensor* out, int32_t factor,
                 int32_t mode, int32_t S, void* stream);

/* inc_maxpool (increment_ops.py:288-310): y = pool(acc+dx) - pool(acc),
 * then acc += dx.  Dense maxpool (tensors.py:242-256) when acc == NULL. */
int evc_maxpool(const evc_tensor* in, float* acc, int64_t acc_stride,
                const evc_tensor* out, int32_t wh, int32_t ww, int32_t stride,
                int32_t S, void* stream);

/* inc_linear + flatten_increment (increment_ops.py:197-223): runs of th*tw
 * flat elements.  With in->flags == NULL run liveness is recomputed from the
 * values (flatten_increment); otherwise `in` must be the (1,1,L) flattened
 * increment with tile (1,run) and its flags are used.  y[f] = sum over live runs;
 * meter[s] += 2*F*live_elements.  dense != 0 computes W@x + bias over all
 * runs (dense_linear, tensors.py:231-239) and skips the meter.
 * workspace: evc_linear_workspace() floats. */
int64_t evc_linear_workspace(int32_t F, int64_t L, int32_t run, int32_t S);
int evc_linear(const evc_tensor* in, const float* weight, const float* bias,
               const evc_tensor* out, int32_t F, int32_t dense,
               int64_t* meter, float* workspace, int32_t S, void* stream);

/* ---- events (events.py:240-302) -------------------------------------- */

enum { EVC_ENC_COUNT = 0, EVC_ENC_TIMESTAMP = 1, EVC_ENC_VOXEL = 2 };

/* Workspace bytes for evc_bin_events with up to n_events in the window. */
int64_t evc_bin_events_workspace(int64_t n_events, int32_t H, int32_t W, int32_t bins);

/* encode (events.py:251-292), atomic-free and bit-exact: events
 * [lo, hi) of the sorted stream are stable-radix-sorted by pixel key, then
 * each pixel run is folded in time order (voxel: all lower-hat adds, then
 * all upper-hat adds, each f32(f64(acc)+v)).  out is (C,H,W) float32 with
 * C = 2 (count/timestamp) or bins (voxel). */
int evc_bin_events(const uint64_t* t, const uint16_t* x, const uint16_t* y,
                   const int8_t* p, int64_t lo, int64_t hi, int64_t tau,
                   int64_t delta, int32_t H, int32_t W, int32_t kind,
                   int32_t bins, float* out, void* workspace,
                   int64_t workspace_bytes, void* stream);

/* Event ingest (ingest.cu).
 * read_events' EVB record view (events.py:185-206): n packed little-endian 13-byte
 * records {u64 t, u16 x, u16 y, i8 p} (events.py:35-37) already on the device ->
 * the t / x / y / p columns evc_bin_events reads. */
int evc_unpack_events(const uint8_t* records, int64_t n, uint64_t* t, uint16_t* x,
                      uint16_t* y, int8_t* p, void* stream);

/* step_increment(encode(prev, "count"), encode(cur, "count")) (events.py:295-302
 * over events.py:267-272) from only the events that leave ([lo_prev, lo_cur)) and
 * enter ([hi_prev, hi_cur)) the window: out (C = 2, one session) receives the
 * values and their exact tile mask, bit-identical to the two encodings' diff. */
int evc_count_increment(const uint16_t* x, const uint16_t* y, const int8_t* p,
                        int64_t lo_prev, int64_t hi_prev, int64_t lo_cur,
                        int64_t hi_cur, const evc_tensor* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EVCONV_H */
