// Fused incremental convolution: ONE launch per conv layer per step.
//
// Replaces the value path, the mask propagation and the FLOP meter of
// inc_conv2d (increment_ops.py:126-194) -- and, when the conv's only reader is
// an activation node, inc_activation (increment_ops.py:232-238) -- with a
// single TMA-fed tcgen05 kernel:
//
//  * M tile = an RH x RW region of output pixels (RH * RW = 128; RW = 32, 16 or
//    8 so narrow maps do not waste rows).  A CTA first decides whether its region
//    can change this step: it ORs the any-channel input tile map `fany` (written
//    by the producing sparsify kernel) over the region's receptive box.  Sites
//    whose taps all read dead tiles are exactly zero (mask soundness), so a dead
//    region is skipped -- or zeroed once when it was computed last step
//    (`rstate`), which restores the exact-zero invariant of TileMask.
//  * Live regions: K-block = one tap (r, s) x 32 channels; its A operand is two
//    TMA boxes (TF32 heads, TF32 tails) of the channels-innermost hi/lo shadow of
//    the input, each covering the whole RH x RW region (traversal stride = conv
//    stride; zero padding = TMA out-of-bounds fill).  3xTF32 (hi*hi + hi*lo +
//    lo*hi, fp32 TMEM accumulation) keeps fp32-grade accuracy; weights are
//    pre-split, pre-swizzled K-major images.
//  * Split-K runs across a thread-block cluster (grid z = cluster z = splits):
//    each CTA parks its fp32 partial tile in shared memory and CTA rank r sums
//    channel slice r over all ranks through DSMEM in rank order -- deterministic,
//    no workspace, no second launch.
//  * The epilogue adds the bias (dense pass) and optionally applies the
//    activation delta y = f(acc + dx) - f(acc), acc += dx in place.
//  * Warps 2-3 of every CTA (idle in the GEMM pipeline) compute the output tile
//    flags (live iff some input tile in the tile's receptive box is live in any
//    channel) and the exact reference meter terms:
//    the live-flag count and sum_c sum_ab F_c[a][b] RT[a] CT[b] + border padding
//    term, accumulated with integer atomics.  evc_meter_step turns them into
//    `performed` (with the all-false / all-true shortcuts, increment_ops.py:148-154).
//
// Roles (8 warps): warp 0 = region test + TMA producer (lane 0); warp 1 = TMEM
// alloc + MMA issuer (lane 0); warps 2-3 = flags + meter; warps 4-7 = epilogue.

#include <cooperative_groups.h>
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "conv_common.cuh"
// 1: the MMA issuer warp walks its K loop converged and one elected lane issues each tcgen05.mma / commit
// (operands in uniform registers, no per-MMA waterfall loop around a single active lane): 12 % faster on
// the tap-mode BN = 128 layers, whose single issuing thread was the bottleneck.  0: lane 0 issues alone.
#ifndef EVC_MMA_WARP
#define EVC_MMA_WARP 1
#endif
#ifndef EVC_TMA_WARP  // the same for the TMA producer warp
#define EVC_TMA_WARP 0
#endif
#include "tcgen05.cuh"

namespace evc {

namespace fz {

constexpr int BM = 128;
constexpr int THREADS = 256;


struct Args {
  int c_in, c_out, kh, kw, stride, pad, H, W, Ho, Wo, S;
  int RH, RW, RHn, RWn, cchunks, nkb, splits, kb_per_split, bn;
  int th, tw, cp;
  // row mode (stride 1): regions are 128 consecutive sites of the output grid flattened with
  // pitch P = W + 2 pad; a K-block is (kernel row, 32 channels) with the kw taps as row shifts
  int row, P, R, VM;  // row = 2: packed (kw taps along N, shifted sums in the epilogue); VM sites per region
  int ns, stage, a_half, b_bytes;  // pipeline depth and stage layout (bytes)
  int drain;                       // > 0: K-blocks per accumulation segment (promoted to fp32 registers)
  const float* wpack;
  const float* bias;
  // incremental mode (dense == 0)
  const uint8_t* fany;  // [S][GHi*GWi]
  const uint8_t* in_f;  // per-channel input flags
  int64_t in_fs;
  const int32_t* tab;
  uint8_t* oflags;  // output flag planes (conv output, or the fused activation's output)
  int64_t ofs;
  uint8_t* rstate;  // [S*R][nb]
  long long* mpart;  // [S][CTAs per session][2]: live input flags, weighted meter term (no atomics)
  // outputs
  float* out;  // conv values (nullable when the activation is fused and nothing else reads them)
  int64_t ovs;
  int act;  // -1 = none
  float alpha;
  float* acc;  // activation accumulator (nullable in dense mode = dense_oracle)
  int64_t accs;
  float* yact;
  int64_t yvs;
  int dense;
  // fused t_p = 0 sparsify of the output (the next conv's input): hi/lo shadow, per-channel
  // flags and any-channel map (both zeroed per step), per-CTA sums of squares [S][CTAs/session]
  float* sp_hwc;
  int64_t sp_hs;
  int sp_cp, sp_pitch, sp_GH, sp_GW;
  uint8_t* sp_flags;
  int64_t sp_fs;
  uint8_t* sp_fany;
  double* sp_part;
  unsigned long long* trace;  // debug: per-CTA phase timestamps (evc_conv_trace), normally NULL
  // output geometry of the emitted tensor (= Ho, Wo, c_out unless sub)
  int eHo, eWo, oc;
  // sub-pixel mode (evc_conv_fused_subpixel): this launch is the 2x bilinear upsample -> 3x3 conv
  // pair rewritten as a 3x3 conv on the low-res input with 4 * oc composed output channels
  // (phase p = n / oc -> output site (2u + p / 2, 2x + p % 2)); fany is then the low-res region map,
  // fany_side the any-channel map of the high-res conv input (flags, meter, output masking),
  // border[s][2 (eHo + eWo)][oc] the correction of the high-res border lines
  int sub;
  const uint8_t* fany_side;
  const float* border;
  int pf;  // epilogue warps prefetch the activation accumulators of their sites into L2 during the mainloop
};

static unsigned long long* g_trace = nullptr;

__device__ __forceinline__ unsigned long long clk() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TR(i)                                                                                              \
  do {                                                                                                     \
    if (a.trace)                                                                                           \
      a.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 + (i)] = clk() - t_start; \
  } while (0)

// Flags + meter share of one CTA (q of Qs CTAs of session s; t = thread 0..63).
// 32-bit indices: every per-session count here is far below 2^31.
__device__ __noinline__ void side_work(const Args& a, int s, int q, int Qs, int t) {
  const TabHdr& h = *reinterpret_cast<const TabHdr*>(a.tab);
  const int To = h.GHo * h.GWo, Ti = h.GHi * h.GWi, GWo = h.GWo, GWi = h.GWi;
  const int nthr = Qs * 64, gid = q * 64 + t;
  const uint8_t* fa = a.fany_side + (int64_t)s * Ti;
  const int32_t* boxr = a.tab + h.boxr;
  const int32_t* boxc = a.tab + h.boxc;
  // output tile flags: every channel's flag is the receptive-box OR of the any-channel map; work unit =
  // (tile, 16 channels): the box OR once per unit, 16 byte stores (coalesced across threads: consecutive tiles)
  uint8_t* of = a.oflags + (int64_t)s * a.ofs;
  const int nocj = (a.oc + 15) >> 4;
  for (int e = gid; e < nocj * To; e += nthr) {
    const int cj = e / To, tt = e - cj * To;
    const int i = tt / GWo, j = tt - i * GWo;
    const int r0 = boxr[2 * i], r1 = boxr[2 * i + 1], c0 = boxc[2 * j], c1 = boxc[2 * j + 1];
    int nf = 0;
    for (int r = r0; r <= r1; ++r)
      for (int c = c0; c <= c1; ++c) nf |= fa[r * GWi + c];
    const uint8_t v = nf != 0;
    uint8_t* o = of + (int64_t)(cj * 16) * To + tt;
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (cj * 16 + k < a.oc) o[(int64_t)k * To] = v;
  }
  // meter: live-flag count and weighted count; work unit = (tile, 8 channels): the tile's weight once,
  // eight independent flag loads (coalesced across threads: consecutive tiles)
  int cnt = 0;
  long long w = 0;
  const uint8_t* F = a.in_f + (int64_t)s * a.in_fs;
  const int32_t* rt = a.tab + h.rt;
  const int32_t* ct = a.tab + h.ct;
  const int nchk = (a.c_in + 7) >> 3, nunit = nchk * Ti;
  for (int e = gid; e < nunit; e += nthr) {
    const int ck = e / Ti, tt = e - ck * Ti;
    const uint8_t* Fc = F + (int64_t)(ck * 8) * Ti + tt;
    int live = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (ck * 8 + k < a.c_in) live += Fc[(int64_t)k * Ti] != 0;
    if (live) {
      const int i = tt / GWi;
      cnt += live;
      w += (long long)live * (rt[i] * ct[tt - i * GWi]);
    }
  }
  const int nbd = h.ngrp * a.c_in;
  for (int e = gid; e < nbd; e += nthr) {
    const int g = e / a.c_in, c = e - g * a.c_in;
    const int32_t* gp = a.tab + h.grp + 5 * g;
    const uint8_t* Fc = F + (int64_t)c * Ti;
    int live = 0;
    for (int p = 0; p < gp[1]; ++p)
      for (int qq = 0; qq < gp[3]; ++qq) live |= Fc[(gp[0] + p) * GWi + gp[2] + qq];
    if (live) w += gp[4];
  }
  // one partial per CTA (the two side-work warps meet at a named barrier): no global atomics
  __shared__ long long s_mp[2][2];
  const long long c2 = warp_sum_ll(cnt), w2 = warp_sum_ll(w);
  if ((t & 31) == 0) {
    s_mp[t >> 5][0] = c2;
    s_mp[t >> 5][1] = w2;
  }
  asm volatile("bar.sync 1, 64;" ::: "memory");
  if (t == 0) {
    long long* mp = a.mpart + ((int64_t)s * Qs + q) * 2;
    mp[0] = s_mp[0][0] + s_mp[1][0];
    mp[1] = s_mp[0][1] + s_mp[1][1];
  }
  // the persistent kernel calls this in a loop: s_mp is read before either warp refills it
  asm volatile("bar.sync 1, 64;" ::: "memory");
}

__device__ __noinline__ float act_other(float x, int kind, float alpha) { return act_apply(x, kind, alpha); }

// f of the fused activation: ReLU inline, the rest out of line (keeps the kernel small)
__device__ __forceinline__ float act_f(float x, int kind, float alpha) {
  return kind == EVC_ACT_RELU ? fmaxf(x, 0.0f) : act_other(x, kind, alpha);
}

// Sub-pixel mode: composed channel n of low-res site (u, x) -> output channel and high-res site.
// Composed channels are phase-minor: n = 4 c + 2 a + b (tensors.compose_subpixel), so an aligned
// group of 4k composed channels holds k real channels at all four phase sites of (u, x).
__device__ __forceinline__ void sub_site(const Args& a, int& u, int& x, int& n) {
  if (!a.sub) return;
  const int ph = n & 3;
  n >>= 2;
  if (u < a.Ho && x < a.Wo) {
    u = 2 * u + (ph >> 1);
    x = 2 * x + (ph & 1);
  } else {
    u = a.eHo;  // never valid
  }
}

// Sub-pixel mode, incremental: is output tile (u / th, x / tw) live?  The OR of the high-res input's
// any-channel map over its receptive box (what side_work writes as the output flags).  A composed
// value can be a rounding-level nonzero where the oracle's upsampled input is exactly zero; the flags
// say dead there, so the value is forced to the oracle's exact zero.
__device__ __forceinline__ bool sub_tile_live(const Args& a, int s, int u, int x) {
  const TabHdr& h = *reinterpret_cast<const TabHdr*>(a.tab);
  const int32_t* boxr = a.tab + h.boxr;
  const int32_t* boxc = a.tab + h.boxc;
  const int i = u / a.th, j = x / a.tw;
  const uint8_t* fa = a.fany_side + (int64_t)s * h.GHi * h.GWi;
  int nf = 0;
  for (int r = boxr[2 * i]; r <= boxr[2 * i + 1]; ++r)
    for (int c = boxc[2 * j]; c <= boxc[2 * j + 1]; ++c) nf |= fa[r * h.GWi + c];
  return nf != 0;
}

// Sub-pixel, incremental: the output-tile liveness shared by the four phase sites of low-res site
// (u, x) (-1 when not applicable), evaluated once per work item.
__device__ __forceinline__ int sub_live_of(const Args& a, int s, int u, int x) {
  if (!a.sub || a.dense || u >= a.Ho || x >= a.Wo) return -1;
  return sub_tile_live(a, s, 2 * u, 2 * x) ? 1 : 0;
}

// Final values of N channels (n0, n0 + step, ...) of output site (u, x) (region row-major).
// Every global load is issued before any store so the latencies overlap.  Returns the
// site's sum of squared sparsify outputs (0 if unfused).
template <int N>
__device__ __forceinline__ double emit_sub(const Args& a, int s, int u, int x, int n0, int cnt, const float* vals,
                                           int sub_live);

// L2 prefetch of the activation accumulator values emit() will read for output site (u, x), channels
// n0 .. n0 + nn - 1 (incremental mode): issued by the epilogue warps before they wait for the MMAs, so the
// epilogue's read-modify-write of acc finds its lines in L2 instead of HBM
__device__ __forceinline__ void prefetch_acc(const Args& a, int s, int u, int x, int n0, int nn) {
  if (!a.pf || a.dense || a.act < 0 || !a.acc || a.sub || u >= a.eHo || x >= a.eWo) return;
  nn = min(nn, a.c_out - n0);
  const int64_t plane = (int64_t)a.eHo * a.eWo;
  const float* p = a.acc + (int64_t)s * a.accs + (int64_t)n0 * plane + (int64_t)u * a.eWo + x;
  for (int j = 0; j < nn; ++j) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + j * plane));
}

// SUBOK: the instantiation can run in sub-pixel mode (BN >= 64, not packed -- the host enforces it),
// so kernels that never do carry no sub-pixel code (registers, instruction cache).
template <int N, bool SUBOK = false>
__device__ __forceinline__ double emit(const Args& a, int s, int u, int x, int n0, int step, int cnt,
                                       const float* vals, int sub_live = -1) {
  if constexpr (SUBOK && N % 4 == 0) {
    if (a.sub) return emit_sub<N>(a, s, u, x, n0, cnt, vals, sub_live);
  }
  const bool valid = u < a.eHo && x < a.eWo;
  const int64_t plane = (int64_t)a.eHo * a.eWo;
  const int64_t base = (int64_t)n0 * plane + (int64_t)u * a.eWo + x;
  const int64_t dn = (int64_t)step * plane;
  float v[N], y[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    v[j] = vals[j];
    if (valid && j < cnt && a.dense && a.bias) v[j] = __fadd_rn(v[j], __ldg(a.bias + n0 + j * step));
    y[j] = v[j];
  }
  if (valid && a.out) {
    float* __restrict__ o = a.out + (int64_t)s * a.ovs + base;
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (j < cnt) o[j * dn] = v[j];
  }
  if (valid && a.act >= 0) {
    float* __restrict__ ap = a.acc ? a.acc + (int64_t)s * a.accs + base : nullptr;
    float* __restrict__ yp = a.yact ? a.yact + (int64_t)s * a.yvs + base : nullptr;
    float acc0[N];
    if (!a.dense) {
#pragma unroll
      for (int j = 0; j < N; ++j) acc0[j] = j < cnt ? ap[j * dn] : 0.0f;
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (j >= cnt) continue;
      if (a.dense) {
        y[j] = act_f(v[j], a.act, a.alpha);
        if (ap) ap[j * dn] = v[j];
      } else {
        const float a1 = __fadd_rn(acc0[j], v[j]);
        y[j] = __fsub_rn(act_f(a1, a.act, a.alpha), act_f(acc0[j], a.act, a.alpha));
        ap[j * dn] = a1;
      }
      if (yp) yp[j * dn] = y[j];
    }
  }
  if (!a.sp_hwc) return 0.0;
  // fused sparsify_step at t_p = 0 (sparsify.py:63-71): out = 0 + y, residual stays 0; the mask is
  // recomputed from the values (sparsify.py:77-78): every site with a nonzero value stores 1 into its
  // (tile, channel) flag (benign: only ever set; the lanes of one tile merge into one store)
  float ss = 0.0f;  // <= 16 squares per call in fp32, widened once per site
  const int tile = valid ? (u / a.th) * a.sp_GW + x / a.tw : 0;
  float* sh = a.sp_hwc + (int64_t)s * a.sp_hs + ((int64_t)u * a.sp_pitch + x) * hwc_px(a.sp_cp);
  const int64_t To = (int64_t)a.sp_GH * a.sp_GW;
  uint8_t* fl = a.sp_flags + (int64_t)s * a.sp_fs + tile;
  bool any = false;
  float o[N];
#pragma unroll
  for (int j = 0; j < N; ++j) o[j] = __fadd_rn(0.0f, y[j]);
  if (N % 4 == 0 && step == 1 && cnt == N && (n0 & 3) == 0 && (a.sp_cp & 3) == 0) {
    if (valid && a.sp_cp < 0) {  // fp32 shadow: 16-byte runs of values
#pragma unroll
      for (int j = 0; j < N; j += 4)
        *reinterpret_cast<float4*>(sh + n0 + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
    } else if (valid) {  // 16-byte runs of heads and tails
#pragma unroll
      for (int j = 0; j < N; j += 4) {
        const float4 h = make_float4(tf32_head(o[j]), tf32_head(o[j + 1]), tf32_head(o[j + 2]), tf32_head(o[j + 3]));
        const float4 l = make_float4(__fsub_rn(o[j], h.x), __fsub_rn(o[j + 1], h.y), __fsub_rn(o[j + 2], h.z),
                                     __fsub_rn(o[j + 3], h.w));
        float* hp = sh + hwc_head(a.sp_cp, n0 + j);  // 4 channels never straddle a 32-chunk
        *reinterpret_cast<float4*>(hp) = h;
        *reinterpret_cast<float4*>(hp + hwc_unit(a.sp_cp)) = l;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (valid && j < cnt) hwc_store(sh, a.sp_cp, n0 + j * step, o[j]);
  }
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const bool in = valid && j < cnt;
    if (in) ss = __fmaf_rn(o[j], o[j], ss);
    if (in && o[j] != 0.0f) {
      fl[(int64_t)(n0 + j * step) * To] = 1;
      any = true;
    }
  }
  if (any) a.sp_fany[(int64_t)s * To + tile] = 1;
  return (double)ss;
}


// Sub-pixel emit: composed channels n0 .. n0 + N - 1 (n0 % 4 == 0) of low-res site (u, x) = NC = N / 4
// real channels c0 + k at the four high-res sites (2u + a, 2x + b).  Each (channel, row a) pair of
// sites is adjacent in x: every value, accumulator and activation access is a float2 (a warp covers
// 256 contiguous bytes of a row).  Adds the border-line correction, zeroes sites of dead output
// tiles (incremental; the four sites share one tile, th and tw even), then the activation and the
// fused t_p = 0 sparsify as in emit.
template <int N>
__device__ __forceinline__ double emit_sub(const Args& a, int s, int u, int x, int n0, int cnt, const float* vals,
                                           int sub_live) {
  constexpr int NC = N / 4;
  const int c0 = n0 >> 2, nc = cnt >> 2;
  const bool valid = u < a.Ho && x < a.Wo;
  const int U0 = 2 * u, X0 = 2 * x;
  const int64_t plane = (int64_t)a.eHo * a.eWo;
  float v[NC][2][2];
  const bool masked = valid && !a.dense && !(sub_live >= 0 ? sub_live != 0 : sub_tile_live(a, s, U0, X0));
#pragma unroll
  for (int k = 0; k < NC; ++k)
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        float t = masked ? 0.0f : vals[4 * k + 2 * r + b];
        if (valid && k < nc && a.dense && a.bias) t = __fadd_rn(t, __ldg(a.bias + c0 + k));
        v[k][r][b] = t;
      }
  if (valid && !masked && (U0 == 0 || X0 == 0 || U0 + 1 == a.eHo - 1 || X0 + 1 == a.eWo - 1)) {
    const int64_t lines = (int64_t)s * 2 * (a.eHo + a.eWo);
#pragma unroll
    for (int r = 0; r < 2; ++r)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const int uu = U0 + r, xx = X0 + b;
        if (uu != 0 && xx != 0 && uu != a.eHo - 1 && xx != a.eWo - 1) continue;
        const int li = uu == 0 ? xx : (uu == a.eHo - 1 ? a.eWo + xx : (xx == 0 ? 2 * a.eWo + uu : 2 * a.eWo + a.eHo + uu));
        const float* bc = a.border + (lines + li) * a.oc + c0;
#pragma unroll
        for (int k = 0; k < NC; ++k)
          if (k < nc) v[k][r][b] = __fadd_rn(v[k][r][b], bc[k]);
      }
  }
  float y[NC][2][2];
#pragma unroll
  for (int k = 0; k < NC; ++k)
#pragma unroll
    for (int r = 0; r < 2; ++r) y[k][r][0] = v[k][r][0], y[k][r][1] = v[k][r][1];
  const int64_t base = (int64_t)c0 * plane + (int64_t)U0 * a.eWo + X0;  // float2-aligned: X0, eWo even
  if (valid && a.out) {
    float* o = a.out + (int64_t)s * a.ovs + base;
#pragma unroll
    for (int k = 0; k < NC; ++k)
#pragma unroll
      for (int r = 0; r < 2; ++r)
        if (k < nc) *reinterpret_cast<float2*>(o + k * plane + r * a.eWo) = make_float2(v[k][r][0], v[k][r][1]);
  }
  if (valid && a.act >= 0) {
    float* ap = a.acc ? a.acc + (int64_t)s * a.accs + base : nullptr;
    float* yp = a.yact ? a.yact + (int64_t)s * a.yvs + base : nullptr;
    float2 acc0[NC][2];
    if (!a.dense) {
#pragma unroll
      for (int k = 0; k < NC; ++k)
#pragma unroll
        for (int r = 0; r < 2; ++r)
          acc0[k][r] = k < nc ? *reinterpret_cast<const float2*>(ap + k * plane + r * a.eWo) : make_float2(0.0f, 0.0f);
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if (k >= nc) continue;
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        float2 a1;
        if (a.dense) {
          y[k][r][0] = act_f(v[k][r][0], a.act, a.alpha);
          y[k][r][1] = act_f(v[k][r][1], a.act, a.alpha);
          a1 = make_float2(v[k][r][0], v[k][r][1]);
        } else {
          a1 = make_float2(__fadd_rn(acc0[k][r].x, v[k][r][0]), __fadd_rn(acc0[k][r].y, v[k][r][1]));
          y[k][r][0] = __fsub_rn(act_f(a1.x, a.act, a.alpha), act_f(acc0[k][r].x, a.act, a.alpha));
          y[k][r][1] = __fsub_rn(act_f(a1.y, a.act, a.alpha), act_f(acc0[k][r].y, a.act, a.alpha));
        }
        if (ap) *reinterpret_cast<float2*>(ap + k * plane + r * a.eWo) = a1;
        if (yp) *reinterpret_cast<float2*>(yp + k * plane + r * a.eWo) = make_float2(y[k][r][0], y[k][r][1]);
      }
    }
  }
  if (!a.sp_hwc) return 0.0;
  // fused sparsify_step at t_p = 0 of the four sites (see emit)
  float ss = 0.0f;
  const int tile = valid ? (U0 / a.th) * a.sp_GW + X0 / a.tw : 0;
  const int64_t To = (int64_t)a.sp_GH * a.sp_GW;
  uint8_t* fl = a.sp_flags + (int64_t)s * a.sp_fs + tile;
  bool any = false;
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (!valid) continue;
      float* sh = a.sp_hwc + (int64_t)s * a.sp_hs + ((int64_t)(U0 + r) * a.sp_pitch + X0 + b) * hwc_px(a.sp_cp);
      float o[NC];
#pragma unroll
      for (int k = 0; k < NC; ++k) o[k] = __fadd_rn(0.0f, y[k][r][b]);
      if (NC % 4 == 0 && nc == NC && (c0 & 3) == 0 && a.sp_cp < 0) {
#pragma unroll
        for (int k = 0; k < NC; k += 4) *reinterpret_cast<float4*>(sh + c0 + k) = make_float4(o[k], o[k + 1], o[k + 2], o[k + 3]);
      } else {
#pragma unroll
        for (int k = 0; k < NC; ++k)
          if (k < nc) hwc_store(sh, a.sp_cp, c0 + k, o[k]);
      }
#pragma unroll
      for (int k = 0; k < NC; ++k)
        if (k < nc) ss = __fmaf_rn(o[k], o[k], ss);
    }
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    const bool nz = valid && k < nc &&
                    (__fadd_rn(0.0f, y[k][0][0]) != 0.0f || __fadd_rn(0.0f, y[k][0][1]) != 0.0f ||
                     __fadd_rn(0.0f, y[k][1][0]) != 0.0f || __fadd_rn(0.0f, y[k][1][1]) != 0.0f);
    if (nz) {
      fl[(int64_t)(c0 + k) * To] = 1;
      any = true;
    }
  }
  if (any) a.sp_fany[(int64_t)s * To + tile] = 1;
  return (double)ss;
}

// Restore exact zeros of channel n at site (u, x) of a region computed last step and dead now.
__device__ __forceinline__ void zero_site(const Args& a, int s, int u, int x, int n) {
  sub_site(a, u, x, n);
  if (u >= a.eHo || x >= a.eWo) return;
  const int64_t off = (int64_t)n * a.eHo * a.eWo + (int64_t)u * a.eWo + x;
  if (a.out) a.out[(int64_t)s * a.ovs + off] = 0.0f;
  if (a.yact) a.yact[(int64_t)s * a.yvs + off] = 0.0f;
  if (a.sp_hwc) hwc_store(a.sp_hwc + (int64_t)s * a.sp_hs + ((int64_t)u * a.sp_pitch + x) * hwc_px(a.sp_cp), a.sp_cp, n, 0.0f);
}

// Output site of TMEM lane m in region rr.
__device__ __forceinline__ void site_of(const Args& a, int rr, int m, int& u, int& x) {
  if (a.row) {
    // packed row mode: a region holds VM = 128 - (kw - 1) sites (lanes >= VM only feed the shifts)
    const int i = rr * a.VM + m;
    u = i / a.P;
    x = i - u * a.P;
    if (m >= a.VM) u = a.Ho;  // never valid
  } else {
    u = (rr / a.RWn) * a.RH + m / a.RW;
    x = (rr % a.RWn) * a.RW + m % a.RW;
  }
}

template <int BN>
__global__ void __launch_bounds__(THREADS, (BN <= 16 ? 2 : 1)) k_conv_fused(const __grid_constant__ CUtensorMap tmap,
                                                           const __grid_constant__ Args a) {
  // 3xTF32 with the fewest MMA instructions (tcgen05.mma costs ~62 cycles for any N <= 128):
  //  CAT (BN <= 128): D_j[:, 0:2BN] += A_hi . [B_hi | B_lo]  (one MMA, N = 2 BN: hi*hi and hi*lo)
  //                   D_c[:, 0:BN]  += A_lo . B_hi           (one MMA)
  //  BN = 256:        hi*hi, hi*lo and lo*hi as three N = 256 MMAs (hi*lo + lo*hi share one accumulator)
  // NA rotating accumulator blocks j = K-block mod NA shorten every fp32 accumulation chain; the
  // epilogue sums all blocks in fp32 (RN), small terms first.
  constexpr bool CAT = BN <= 128;
  constexpr bool PACK = BN <= 32;  // packed row mode possible (2 kw BN <= 256 for kw <= 3... checked on host)
  constexpr int NA = BN >= 256 ? 1 : (BN >= 128 ? 1 : (BN >= 32 ? 3 : 4));
  constexpr int NEED0 = CAT ? NA * 2 * BN + BN : 2 * BN;
  constexpr int NEED = PACK ? (NEED0 > 6 * BN ? NEED0 : 6 * BN) : NEED0;  // packed: 3 taps x 2 x BN
  constexpr int TMEM_COLS = NEED <= 32 ? 32 : (NEED <= 64 ? 64 : (NEED <= 128 ? 128 : (NEED <= 256 ? 256 : 512)));
  // kind::tf32, fp32 accumulate, A and B K-major, M = 128, N = BN or 2 BN
  constexpr uint32_t IDESC_BASE = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BM >> 4) << 24);
  constexpr uint32_t IDESC = IDESC_BASE | ((uint32_t)(BN >> 3) << 17);
  constexpr uint32_t IDESC2 = IDESC_BASE | ((uint32_t)((CAT ? 2 * BN : BN) >> 3) << 17);
  constexpr int MAXNS = 4;

  const unsigned long long t_start = clk();
  if (a.trace && threadIdx.x == 0)
    a.trace[((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * 16 + 15] = gtime();
  const int R = a.R;
  const int reg = blockIdx.x;  // s * R + region
  const int s = reg / R, rr = reg % R;
  const int nblk = blockIdx.y, z = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rs_idx = (int64_t)reg * gridDim.y + nblk;
  const int kb0 = z * a.kb_per_split, kb1 = min(a.nkb, kb0 + a.kb_per_split), nk = kb1 - kb0;
  const int NS = a.ns, STAGE = a.stage;
  const int npre = min(NS, nk);
  const uint32_t A_HALF = (uint32_t)a.a_half, B_BYTES = (uint32_t)a.b_bytes;
  const int taps = a.row == 1 ? a.kw : 1;                      // MMA groups per K-block
  const uint32_t A_TX = a.row ? (uint32_t)(BM + a.kw - 1) * 128u : (uint32_t)BM * 128u;  // bytes per A box

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * STAGE);  // tma[4], empty[4], acc, seg[2], free[2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * MAXNS + 5);
  volatile int* s_flag = reinterpret_cast<volatile int*>(tslot + 1);  // [0] live, [1] computed last step
  const uint32_t sb = su32(smem), b0 = su32(bars);
  auto tma_bar = [&](int i) { return b0 + 8u * i; };
  auto empty_bar = [&](int i) { return b0 + 8u * (MAXNS + i); };
  const uint32_t acc_bar = b0 + 8u * (2 * MAXNS);
  // promotion mode: segment g of a.drain K-blocks accumulates hi.hi into TMEM block g & 1 (BN columns
  // at j * BN); the small terms hi.lo + lo.hi go to one block at 2 BN for the whole K range (their
  // magnitude is 2^-11 of the main term, so their chain length is harmless).  Three N = BN MMAs per K8
  // step, none of them partially overlapping another's accumulator.  seg_bar[j] = block j's segment
  // complete, free_bar[j] = the epilogue warps have added it to their fp32 register sums
  const int D = (CAT && !(PACK && a.row == 2)) ? max(1, a.drain) : 0;
  auto seg_bar = [&](int j) { return b0 + 8u * (2 * MAXNS + 1 + j); };
  auto free_bar = [&](int j) { return b0 + 8u * (2 * MAXNS + 3 + j); };
  const char* wsrc = reinterpret_cast<const char*>(a.wpack) + (int64_t)nblk * a.nkb * B_BYTES;

  // valid output rows / columns of this region (receptive-box test, prefetch)
  int ulo, uhi, xlo, xhi;
  if (a.row) {
    const int i0 = rr * a.VM;
    ulo = i0 / a.P;
    uhi = min(a.Ho - 1, (i0 + a.VM - 1) / a.P);
    if (ulo == uhi) {
      xlo = i0 - ulo * a.P;
      xhi = min(a.Wo - 1, i0 + a.VM - 1 - ulo * a.P);
    } else {
      xlo = 0;
      xhi = a.Wo - 1;
    }
  } else {
    ulo = (rr / a.RWn) * a.RH;
    uhi = min(ulo + a.RH, a.Ho) - 1;
    xlo = (rr % a.RWn) * a.RW;
    xhi = min(xlo + a.RW, a.Wo) - 1;
  }

  // ---- prologue that reads nothing an upstream kernel writes
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      bar_init(tma_bar(i), 1);
      bar_init(empty_bar(i), 1);
    }
    bar_init(acc_bar, 1);
    for (int j = 0; j < 2; ++j) {
      bar_init(seg_bar(j), 1);
      bar_init(free_bar(j), 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    // the first stages' weights are static: stream them now (their arrive comes with the A boxes)
    for (int i = 0; i < npre; ++i) {
      bar_expect_tx(tma_bar(i), B_BYTES);
      bulk_load(sb + i * STAGE + 2 * A_HALF, wsrc + (int64_t)(kb0 + i) * B_BYTES, B_BYTES, tma_bar(i));
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_trigger();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) TR(2);
  pdl_wait();  // upstream results (input shadow, flags, fany, accumulators) are visible from here

  // ---- region test: OR of the any-channel input tile map over the receptive box
  if (warp == 0) {
    int live = 1;
    if (!a.dense) {
      live = 0;
      if (ulo <= uhi && xlo <= xhi) {
        const int y_lo = max(0, ulo * a.stride - a.pad);
        const int y_hi = min(a.H - 1, uhi * a.stride - a.pad + a.kh - 1);
        const int x_lo = max(0, xlo * a.stride - a.pad);
        const int x_hi = min(a.W - 1, xhi * a.stride - a.pad + a.kw - 1);
        if (y_lo <= y_hi && x_lo <= x_hi) {
          const int GWi = (a.W + a.tw - 1) / a.tw, GHi = (a.H + a.th - 1) / a.th;
          const int ra = y_lo / a.th, nr = y_hi / a.th - ra + 1;
          const int ca = x_lo / a.tw, nc = x_hi / a.tw - ca + 1;
          const uint8_t* fa = a.fany + (int64_t)s * GHi * GWi;
          for (int e = lane; e < nr * nc; e += 32) live |= fa[(ra + e / nc) * GWi + ca + e % nc];
        }
      }
      live = __any_sync(0xffffffffu, live);
    }
    if (lane == 0) {
      s_flag[0] = live;
      s_flag[1] = a.dense ? 0 : a.rstate[rs_idx];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) TR(1);
  const bool live = s_flag[0] != 0;
  const int Qs = R * gridDim.y * gridDim.z;
  const int q = ((int)blockIdx.z * (int)gridDim.y + nblk) * R + rr;
  double ssq = 0.0;  // fused sparsify: this thread's share of sum(out^2)

  if (!live) {
    if (!a.dense && warp >= 2 && warp < 4) side_work(a, s, q, Qs, threadIdx.x - 64);
    if (!a.dense && z == 0 && s_flag[1]) {  // computed last step, dead now: restore exact zeros
      const int n0 = nblk * a.bn, nn = min(a.bn, a.c_out - n0);
      for (int e = threadIdx.x; e < nn * BM; e += THREADS) {
        const int n = n0 + e / BM, m = e % BM;
        int u, x;
        site_of(a, rr, m, u, x);
        zero_site(a, s, u, x, n);
      }
      if (threadIdx.x == 0) a.rstate[rs_idx] = 0;
    }
    if (a.sp_part && threadIdx.x == 0) a.sp_part[(int64_t)s * Qs + q] = 0.0;
    if (threadIdx.x == 0) {  // drain the prefetched weight copies before the shared memory is released
      for (int i = 0; i < npre; ++i) {
        bar_arrive(tma_bar(i));
        bar_wait(tma_bar(i), 0);
      }
    }
    fence_before();
    __syncthreads();
    if (warp == 1) {
      fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
    }
    return;
  }
  if (!a.dense && z == 0 && threadIdx.x == 0 && !s_flag[1]) a.rstate[rs_idx] = 1;

  // non-packed epilogue over channels [cb, ce) of the block (TMEM lane quarter = warp % 4).
  // With a wide block and no split-K, warps 0-3 -- idle once the mainloop is issued -- drain the
  // upper half of the channels while warps 4-7 drain the lower half.
  const bool wide = CAT && BN >= 64 && a.splits == 1 && !(PACK && a.row == 2);
  auto drain = [&](int cb, int ce) {
    const int m = 32 * (warp & 3) + lane;
    int u, x;
    site_of(a, rr, m, u, x);
    const int sl = sub_live_of(a, s, u, x);
    const int n_main = nk < NA ? nk : NA;
    const uint32_t trow = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    float* P = reinterpret_cast<float*>(smem);
  #pragma unroll 1
      for (int c0 = cb; c0 < ce; c0 += 16) {
        float vals[16];
        {  // corrections first (small terms), then the main products
          uint32_t r[NA + 1][16];
          const uint32_t cbase = CAT ? (uint32_t)(NA * 2 * BN) : (uint32_t)BN;
          tmem_ld16_issue(trow + cbase + (uint32_t)c0, r[NA]);
          if (CAT) {
  #pragma unroll
            for (int j = 0; j < NA; ++j) tmem_ld16_issue(trow + (uint32_t)(j * 2 * BN + BN + c0), r[j]);
          }
          tmem_wait_ld();
  #pragma unroll
          for (int j = 0; j <= NA; ++j)
  #pragma unroll
            for (int e = 0; e < 16; ++e) asm volatile("" : "+r"(r[j][e]));  // uses stay after the wait
  #pragma unroll
          for (int e = 0; e < 16; ++e) vals[e] = __uint_as_float(r[NA][e]);
          if (CAT) {
  #pragma unroll
            for (int j = 0; j < NA; ++j)
              if (j < n_main) {
  #pragma unroll
                for (int e = 0; e < 16; ++e) vals[e] = __fadd_rn(vals[e], __uint_as_float(r[j][e]));
              }
          }
        }
        {
          uint32_t r[NA][16];
  #pragma unroll
          for (int j = 0; j < NA; ++j) tmem_ld16_issue(trow + (uint32_t)(j * (CAT ? 2 * BN : BN) + c0), r[j]);
          tmem_wait_ld();
  #pragma unroll
          for (int j = 0; j < NA; ++j)
  #pragma unroll
            for (int e = 0; e < 16; ++e) asm volatile("" : "+r"(r[j][e]));
  #pragma unroll
          for (int j = 0; j < NA; ++j)
            if (j < n_main) {
  #pragma unroll
              for (int e = 0; e < 16; ++e) vals[e] = __fadd_rn(vals[e], __uint_as_float(r[j][e]));
            }
        }
        if (a.splits == 1) {
          const int n0 = nblk * BN + c0;
          ssq += emit<16, (BN >= 64)>(a, s, u, x, n0, 1, min(16, a.c_out - n0), vals, sl);
        } else {
  #pragma unroll
          for (int j = 0; j < 16; ++j) P[(c0 + j) * BM + m] = vals[j];
        }
      }
  };

  if (warp == 0) {
#if EVC_TMA_WARP
#define ARRIVE_TX_ bar_arrive_tx_w
#define BULK_ bulk_load_w
#define TMA3_ tma_load_3d_w
#define TMA4_ tma_load_4d_w
#else
#define ARRIVE_TX_ bar_arrive_tx
#define BULK_ bulk_load
#define TMA3_ tma_load_3d
#define TMA4_ tma_load_4d
#endif
    if (EVC_TMA_WARP || lane == 0) {  // ------------------------------------------------ TMA producer
      for (int i = 0; i < nk; ++i) {
        const int st = i % NS;
        const int kb = kb0 + i;
        const uint32_t abuf = sb + st * STAGE;
        if (i < npre) {
          ARRIVE_TX_(tma_bar(st), 2 * A_TX);  // weights already in flight
        } else {
          bar_spin(empty_bar(st), ((i / NS) & 1) ^ 1);
          ARRIVE_TX_(tma_bar(st), 2 * A_TX + B_BYTES);
          BULK_(abuf + 2 * A_HALF, wsrc + (int64_t)kb * B_BYTES, B_BYTES, tma_bar(st));
        }
        if (a.row) {  // kernel row r of the flattened padded shadow: 128 + kw - 1 pixel rows
          const int r = kb / a.cchunks, c0 = (kb % a.cchunks) * 32;
          const int i0 = rr * a.VM + r * a.P;
          TMA3_(abuf, &tmap, 2 * c0, i0, s, tma_bar(st));  // chunk = [32 heads | 32 tails]
          TMA3_(abuf + A_HALF, &tmap, 2 * c0 + 32, i0, s, tma_bar(st));
        } else {  // one box = the whole RH x RW region for this tap (padded coordinates)
          const int tap = kb / a.cchunks, c0 = (kb % a.cchunks) * 32;
          const int r = tap / a.kw, qq = tap % a.kw;
          const int xs = xlo * a.stride + qq, ys = ulo * a.stride + r;
          TMA4_(abuf, &tmap, 2 * c0, xs, ys, s, tma_bar(st));
          TMA4_(abuf + A_HALF, &tmap, 2 * c0 + 32, xs, ys, s, tma_bar(st));
        }
        if (i == 0 && lane == 0) TR(3);
      }
      if (lane == 0) TR(11);
    }
    __syncwarp();
#undef ARRIVE_TX_
#undef BULK_
#undef TMA3_
#undef TMA4_
  } else if (warp == 1) {
#if EVC_MMA_WARP
    // the whole warp walks the K loop with warp-uniform operands; one elected lane issues each MMA / commit
#define MMA_ mma_w
#define COMMIT_ commit_w
    {  // ------------------------------------------------ MMA issuer
#else
#define MMA_ mma
#define COMMIT_ commit
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
#endif
      for (int i = 0; i < nk; ++i) {
        const int st = i % NS;
        bar_spin(tma_bar(st), (i / NS) & 1);
        fence_after();
        const uint32_t ah = sb + st * STAGE, al = ah + A_HALF, bb = ah + 2 * A_HALF;
        // K-steps of 8 channels holding real input channels (the zero-padded tail chunk is skipped)
        const int kbi = kb0 + i, c0k = (kbi % a.cchunks) * 32, nkk = min(4, (a.c_in - c0k + 7) >> 3);
        if (PACK && a.row == 2) {
          // D[j, (s, hi|lo, n)] += A_lo[j] . B_s + A_hi[j] . B_s for all kw taps s at once (the A tail
          // terms land in the same accumulator: lo . hi is ~2^-11 of hi . hi, far above fp32 rounding)
          const uint32_t idp = IDESC_BASE | ((uint32_t)((a.kw * 2 * BN) >> 3) << 17);
          const uint64_t dl = desc_k(al), dh = desc_k(ah), db = desc_k(bb);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K=8 tf32 = 32 bytes = +2 in the descriptor's address field
            if (kk >= nkk) break;
            MMA_(tmem, dl + 2 * kk, db + 2 * kk, idp, (i || kk) ? 1u : 0u);  // small terms first
            MMA_(tmem, dh + 2 * kk, db + 2 * kk, idp, 1u);
          }
          COMMIT_(empty_bar(st));
          continue;
        }
        if (CAT && D > 0) {
          // promotion mode: K-block i belongs to segment g = i / D in TMEM block g & 1
          const int g = i / D, j = g & 1;
          const bool seg0 = i % D == 0;
          if (seg0 && g >= 2) {  // block j's previous segment (g - 2) must have been promoted
            bar_spin(free_bar(j), (uint32_t)(((g >> 1) - 1) & 1));
            fence_after();
          }
          const uint32_t tj = tmem + (uint32_t)(j * BN), ts = tmem + (uint32_t)(2 * BN);
          for (int t = 0; t < taps; ++t) {
            const uint32_t bh = bb + t * 2 * BN * 128;
            const uint64_t da = desc_k(ah + t * 128), dl = desc_k(al + t * 128), dbh = desc_k(bh),
                           dbl = desc_k(bh + BN * 128);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (kk >= nkk) break;
              MMA_(tj, da + 2 * kk, dbh + 2 * kk, IDESC, (seg0 && t == 0 && kk == 0) ? 0u : 1u);  // hi.hi
              MMA_(ts, da + 2 * kk, dbl + 2 * kk, IDESC, (i == 0 && t == 0 && kk == 0) ? 0u : 1u);  // hi.lo
              MMA_(ts, dl + 2 * kk, dbh + 2 * kk, IDESC, 1u);                                      // lo.hi
            }
          }
          COMMIT_(empty_bar(st));
          if (i % D == D - 1 || i == nk - 1) COMMIT_(seg_bar(j));
          if (i == 0 && lane == 0) TR(12);
          continue;
        }
        for (int t = 0; t < taps; ++t) {
          // row mode: tap t = the A rows shifted by t pixels (any 128-byte row offset is a valid
          // SW128 descriptor start: the swizzle follows the absolute address, scripts/shift_probe.cu)
          const uint32_t at = ah + t * 128, lt = al + t * 128, bh = bb + t * 2 * BN * 128, bl = bh + BN * 128;
          const bool first = t == 0;
          if (CAT) {
            const uint32_t tj = tmem + (uint32_t)((i % NA) * 2 * BN), tc = tmem + (uint32_t)(NA * 2 * BN);
            const uint64_t da = desc_k(at), dl = desc_k(lt), db = desc_k(bh);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // K=8 tf32 = 32 bytes = +2 in the descriptor's address field
              if (kk >= nkk) break;
              MMA_(tj, da + 2 * kk, db + 2 * kk, IDESC2, (i >= NA || kk || !first) ? 1u : 0u);
              MMA_(tc, dl + 2 * kk, db + 2 * kk, IDESC, (i || kk || !first) ? 1u : 0u);
            }
          } else {
            const uint32_t tmain = tmem, tcorr = tmem + (uint32_t)BN;
            const uint64_t da = desc_k(at), dl = desc_k(lt), dbh = desc_k(bh), dbl = desc_k(bl);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (kk >= nkk) break;
              MMA_(tmain, da + 2 * kk, dbh + 2 * kk, IDESC, (i || kk || !first) ? 1u : 0u);
              MMA_(tcorr, da + 2 * kk, dbl + 2 * kk, IDESC, (i || kk || !first) ? 1u : 0u);
              MMA_(tcorr, dl + 2 * kk, dbh + 2 * kk, IDESC, 1u);
            }
          }
        }
        COMMIT_(empty_bar(st));
        if (i == 0 && lane == 0) TR(12);
      }
      COMMIT_(acc_bar);
      if (lane == 0) TR(5);
    }
#undef MMA_
#undef COMMIT_
    __syncwarp();
  } else if (warp < 4) {
    if (!a.dense) {
      if (a.act >= 0 && !a.sub) {  // warm L2 with the accumulator lines the epilogue will read
        const int per = (a.bn + a.splits - 1) / a.splits;
        const int lo = a.splits > 1 ? z * per : 0, hi = a.splits > 1 ? min(a.bn, lo + per) : a.bn;
        const int64_t plane = (int64_t)a.Ho * a.Wo;
        for (int e = threadIdx.x - 64; e < (hi - lo) * (BM / 16); e += 64) {
          const int n = nblk * a.bn + lo + e / (BM / 16), m = (e % (BM / 16)) * 16;
          int u, x;
          site_of(a, rr, m, u, x);
          if (n >= a.c_out || u >= a.Ho || x >= a.Wo) continue;
          const float* p = a.acc + (int64_t)s * a.accs + n * plane + (int64_t)u * a.Wo + x;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
        }
      }
      side_work(a, s, q, Qs, threadIdx.x - 64);
      if (threadIdx.x == 64) TR(10);
    }
  } else {
    // ------------------------------------------------------------- epilogue (TMEM -> values)
    const int m = 32 * (warp & 3) + lane;  // TMEM lane = region site
    int u, x;
    site_of(a, rr, m, u, x);
    const int sl = sub_live_of(a, s, u, x);
    if (a.splits == 1) prefetch_acc(a, s, u, x, nblk * a.bn, BN);
    if (D == 0) {  // (promotion mode waits segment by segment: the MMAs need the promoted blocks back)
      bar_wait(acc_bar, 0);
      fence_after();
    }
    if (threadIdx.x == 128) TR(6);
    const int n_main = nk < NA ? nk : NA;
    const uint32_t trow = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    float* P = reinterpret_cast<float*>(smem);  // [BN][BM] partial tile (split-K only)
    if (PACK && a.row == 2) {
      // out[m] = sum_s v_s[m + s] with v_s[j] = (A . B_lo) + (A . B_hi) of tap s at TMEM row j:
      // shifts by s rows = shuffles inside the warp, the next warp's first rows through shared memory
      __shared__ float s_xch[4][3][3][8];
      const int q4 = warp & 3, KW = a.kw;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 8) {
        float v[3][8];
        {
          uint32_t r4[3][2][8];  // [tap][B tail part, B head part]: every load in flight, one wait
#pragma unroll
          for (int s2 = 0; s2 < 3; ++s2)
            if (s2 < KW) {
              const uint32_t cb = (uint32_t)(s2 * 2 * BN + c0);
              tmem_ld8_issue(trow + cb + BN, r4[s2][0]);  // A . B_lo
              tmem_ld8_issue(trow + cb, r4[s2][1]);       // A . B_hi
            }
          tmem_wait_ld();
#pragma unroll
          for (int s2 = 0; s2 < 3; ++s2)
#pragma unroll
            for (int j = 0; j < 2; ++j)
#pragma unroll
              for (int e = 0; e < 8; ++e) asm volatile("" : "+r"(r4[s2][j][e]));
#pragma unroll
          for (int s2 = 0; s2 < 3; ++s2)
#pragma unroll
            for (int e = 0; e < 8; ++e)
              v[s2][e] = s2 < KW ? __fadd_rn(__uint_as_float(r4[s2][0][e]), __uint_as_float(r4[s2][1][e])) : 0.0f;
        }
#pragma unroll
        for (int s2 = 1; s2 < 3; ++s2)
          if (s2 < KW && lane < s2) {
#pragma unroll
            for (int e = 0; e < 8; ++e) s_xch[q4][s2][lane][e] = v[s2][e];
          }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        float o[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = v[0][e];
#pragma unroll
        for (int s2 = 1; s2 < 3; ++s2) {
          if (s2 >= KW) break;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            float t = __shfl_down_sync(0xffffffffu, v[s2][e], s2);
            if (lane >= 32 - s2) t = q4 < 3 ? s_xch[q4 + 1][s2][lane + s2 - 32][e] : 0.0f;
            o[e] = __fadd_rn(o[e], t);
          }
        }
        asm volatile("bar.sync 2, 128;" ::: "memory");
        const int n0 = nblk * BN + c0;
        ssq += emit<8>(a, s, u, x, n0, 1, min(8, a.c_out - n0), o, sl);
      }
    } else if (D > 0) {
      // promotion: every segment's [main | small] block is added into fp32 register sums (RN) while
      // the MMAs fill the other block -- no tensor-core accumulation chain spans more than a.drain
      // K-blocks (the accumulate truncates; long chains drift, short ones keep fp32 accuracy)
      constexpr int BP = BN < 128 ? BN : 128;  // (the BN = 256 kernel never runs promoted: CAT)
      float sum[BP];
      const int G = (nk + D - 1) / D;
#pragma unroll
      for (int c = 0; c < BP; ++c) sum[c] = 0.0f;
#pragma unroll 1
      for (int g = 0; g < G; ++g) {
        const int j = g & 1;
        bar_wait(seg_bar(j), (uint32_t)((g >> 1) & 1));
        fence_after();
        const uint32_t tb = trow + (uint32_t)(j * BN);
        constexpr int LW = BP >= 32 ? 32 : 16;  // columns per wait (latency-bound: wide loads)
#pragma unroll
        for (int c0 = 0; c0 < BP; c0 += LW) {
          uint32_t rm[LW];
#pragma unroll
          for (int q = 0; q < LW; q += 16) {
            if (LW >= 32 && q % 32 == 0) tmem_ld32_issue(tb + (uint32_t)(c0 + q), rm + q);
            else if (LW < 32) tmem_ld16_issue(tb + (uint32_t)(c0 + q), rm + q);
          }
          tmem_wait_ld();
#pragma unroll
          for (int e = 0; e < LW; ++e) {
            asm volatile("" : "+r"(rm[e]));
            sum[c0 + e] = g ? __fadd_rn(sum[c0 + e], __uint_as_float(rm[e])) : __uint_as_float(rm[e]);
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) bar_arrive(free_bar(j));
      }
      // the small terms (complete with the last segment)
#pragma unroll
      for (int c0 = 0; c0 < BP; c0 += 32) {
        uint32_t rs[32];
        if (BP >= 32) {
          tmem_ld32_issue(trow + (uint32_t)(2 * BN + c0), rs);
        } else {
          tmem_ld16_issue(trow + (uint32_t)(2 * BN + c0), rs);
        }
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < (BP >= 32 ? 32 : 16); ++e) {
          asm volatile("" : "+r"(rs[e]));
          sum[c0 + e] = __fadd_rn(sum[c0 + e], __uint_as_float(rs[e]));
        }
      }
      // the sums go to shared memory ([channel][site], the stages are idle: every MMA and TMA of the
      // CTA has completed) -- the split-K partial tile as is, else the emit reads them back in a
      // rolled loop (one inlined emit: the unrolled form bloats the kernel past the I-cache); a wide
      // block hands the upper half of the channels to warps 0-3, so eight warps emit
#pragma unroll
      for (int c = 0; c < BP; ++c) P[c * BM + m] = sum[c];
    } else if (!CAT) {
      drain(0, wide ? BN / 2 : BN);
    }
  }
  if (!CAT && wide && warp < 4) {
    bar_wait(acc_bar, 0);
    fence_after();
    drain(BN / 2, BN);
  }
  if (CAT && D > 0 && a.splits == 1) {
    // promoted sums in shared memory ([channel][site]): one rolled emit loop for every warp that
    // emits (one inlined emit -- unrolled copies bloat the kernel past the instruction cache); a
    // wide block splits the channels between warps 4-7 (lower half) and warps 0-3 (upper half)
    if (wide) asm volatile("bar.sync 5, 256;" ::: "memory");
    if (warp >= 4 || wide) {
      constexpr int BP = BN < 128 ? BN : 128;
      const int m = 32 * (warp & 3) + lane;
      int u, x;
      site_of(a, rr, m, u, x);
      const int sl = sub_live_of(a, s, u, x);
      const int cb = (wide && warp < 4) ? BP / 2 : 0, ce = (wide && warp >= 4) ? BP / 2 : BP;
      const float* X = reinterpret_cast<const float*>(smem);
#pragma unroll 1
      for (int c0 = cb; c0 < ce; c0 += 16) {
        float vals[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) vals[e] = X[(c0 + e) * BM + m];
        const int n0 = nblk * BN + c0;
        if (n0 < a.c_out) ssq += emit<16, (BN >= 64)>(a, s, u, x, n0, 1, min(16, a.c_out - n0), vals, sl);
      }
    }
  }
  if (threadIdx.x == 128) TR(7);
  if (a.splits > 1) {
    // deterministic split-K: rank r sums channel slice r over all ranks in rank order
    cluster_sync();
    if (threadIdx.x == 0) TR(8);
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int nsp = a.splits;
    const int per = (((BN + nsp - 1) / nsp) + 3) & ~3;  // 4-aligned slices: emit groups never straddle a phase
    const int rank = (int)cl.block_rank();
    const int lo = rank * per, hi = min(BN, lo + per);
    float* P = reinterpret_cast<float*>(smem);
    const int m = threadIdx.x % BM, g = threadIdx.x / BM;  // 2 groups of 128 sites, 4 contiguous channels each
    int u, x;
    site_of(a, rr, m, u, x);
    const int sl = sub_live_of(a, s, u, x);
    constexpr int NB = 4;
    for (int nl0 = lo + NB * g; nl0 < hi; nl0 += 2 * NB) {
      const int cnt = min(NB, hi - nl0);
      float t[16][NB];  // every rank's partials first (latencies overlap), then the ordered sum
#pragma unroll
      for (int zz = 0; zz < 16; ++zz) {
        if (zz < nsp) {
          const float* Rz = cl.map_shared_rank(P, zz);
#pragma unroll
          for (int j = 0; j < NB; ++j) t[zz][j] = j < cnt ? Rz[(nl0 + j) * BM + m] : 0.0f;
        }
      }
      float sum[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        sum[j] = 0.0f;
#pragma unroll
        for (int zz = 0; zz < 16; ++zz)
          if (zz < nsp) sum[j] = __fadd_rn(sum[j], t[zz][j]);
      }
      const int n0 = nblk * BN + nl0;
      ssq += emit<NB, (BN >= 64)>(a, s, u, x, n0, 1, min(cnt, a.c_out - n0), sum, sl);
    }
    cluster_sync();
  }
  if (threadIdx.x == 128) TR(9);
  if (a.sp_part) {
    ssq = block_sum<double>(ssq, [](double v) { return warp_sum_d(v); });
    if (threadIdx.x == 0) a.sp_part[(int64_t)s * Qs + q] = ssq;
  }
  fence_before();
  __syncthreads();
  if (threadIdx.x == 0) TR(13);
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------------------------
// Persistent variant (no split-K, BN <= 64): each CTA walks work items (region, channel block)
// with a continuous TMA/MMA stage ring and TWO TMEM accumulator buffers, so the epilogue of item
// i (TMEM drain, activation, fused sparsify stores) overlaps the MMAs of item i + 1 and the
// prologue is paid once per CTA.  Every role evaluates the region test itself (same inputs,
// same answer), so no per-item hand-off is needed besides the TMEM full / empty barriers.
// ---------------------------------------------------------------------------------------------
// (Divisions through fp32 reciprocals, fdiv: exact for these small operands, and no state held
// across the callers' item loops.)
__device__ __forceinline__ bool region_live_warp(const Args& a, int s, int rr) {
  if (a.dense) return true;
  struct {
    FDiv P, th, tw;
    int GWi, GHi;
  } d;
  d.P = fdiv_of(max(1, a.P));
  d.th = fdiv_of(a.th);
  d.tw = fdiv_of(a.tw);
  d.GWi = fdiv(a.W + a.tw - 1, d.tw);
  d.GHi = fdiv(a.H + a.th - 1, d.th);
  int ulo, uhi, xlo, xhi;
  if (a.row) {
    const int i0 = rr * a.VM;
    ulo = fdiv(i0, d.P);
    uhi = min(a.Ho - 1, fdiv(i0 + a.VM - 1, d.P));
    if (ulo == uhi) {
      xlo = i0 - ulo * a.P;
      xhi = min(a.Wo - 1, i0 + a.VM - 1 - ulo * a.P);
    } else {
      xlo = 0;
      xhi = a.Wo - 1;
    }
  } else {
    ulo = (rr / a.RWn) * a.RH;
    uhi = min(ulo + a.RH, a.Ho) - 1;
    xlo = (rr % a.RWn) * a.RW;
    xhi = min(xlo + a.RW, a.Wo) - 1;
  }
  int live = 0;
  if (ulo <= uhi && xlo <= xhi) {
    const int y_lo = max(0, ulo * a.stride - a.pad), y_hi = min(a.H - 1, uhi * a.stride - a.pad + a.kh - 1);
    const int x_lo = max(0, xlo * a.stride - a.pad), x_hi = min(a.W - 1, xhi * a.stride - a.pad + a.kw - 1);
    if (y_lo <= y_hi && x_lo <= x_hi) {
      const int ra = fdiv(y_lo, d.th), nr = fdiv(y_hi, d.th) - ra + 1;
      const int ca = fdiv(x_lo, d.tw), nc = fdiv(x_hi, d.tw) - ca + 1;
      const uint8_t* fa = a.fany + (int64_t)s * d.GHi * d.GWi + ra * d.GWi + ca;
      if (nr * nc <= 32) {
        const FDiv dn = fdiv_of(nc);
        const int e = (int)(threadIdx.x & 31);
        if (e < nr * nc) {
          const int r = fdiv(e, dn);
          live = fa[r * d.GWi + e - r * nc];
        }
      } else {
        for (int r = 0; r < nr; ++r)
          for (int c = (int)(threadIdx.x & 31); c < nc; c += 32) live |= fa[r * d.GWi + c];
      }
    }
  }
  return __any_sync(0xffffffffu, live) != 0;
}

// epilogue warps of the persistent kernel: 8 (two per TMEM lane quarter, each taking half of
// the channel block) when one CTA owns the SM, 4 when two co-reside (BN = 16)
template <int BN>
__host__ __device__ constexpr int persist_epi_warps() { return BN >= 32 ? 8 : 4; }
template <int BN>
__host__ __device__ constexpr int persist_threads() { return (4 + persist_epi_warps<BN>()) * 32; }

// PK: packed row mode (a.row == 2) -- a separate instantiation, so each epilogue gets its own
// register allocation
template <int BN, bool PK>
__global__ void __launch_bounds__(persist_threads<BN>(), (BN <= 16 ? 2 : 1)) k_conv_persist(const __grid_constant__ CUtensorMap tmap,
                                                                              const __grid_constant__ Args a) {
  // SS (BN = 128): TMEM = [main_0 | main_1 | small_0 | small_1] -- the hi.hi segments alternate between
  // the main blocks (promotion), the small terms hi.lo + lo.hi of a whole item go to small_(item & 1), so
  // the next item's MMAs start while the epilogue still drains the previous one (512 columns).
  constexpr bool SS = BN >= 128;
  constexpr int BUF = SS ? BN : (BN <= 32 ? 6 * BN : 3 * BN);  // packed: 3 taps x [A.B_hi | A.B_lo]; CAT: [hi.hi | hi.lo | lo.hi]
  constexpr int TMEM_COLS = SS ? 4 * BN : (2 * BUF <= 128 ? 128 : (2 * BUF <= 256 ? 256 : 512));
  constexpr uint32_t IDESC_BASE = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BM >> 4) << 24);
  constexpr uint32_t IDESC = IDESC_BASE | ((uint32_t)(BN >> 3) << 17);
  constexpr uint32_t IDESC2 = IDESC_BASE | ((uint32_t)((2 * BN) >> 3) << 17);
  constexpr int MAXNS = 4;
  constexpr int EPI = persist_epi_warps<BN>(), NH = EPI / 4;  // epilogue warps, channel halves
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int R = a.R, nb = (a.c_out + BN - 1) / BN;
  const int n_items = a.S * R * nb;
  const int NS = a.ns, STAGE = a.stage, nk = a.nkb;
  const uint32_t A_HALF = (uint32_t)a.a_half, B_BYTES = (uint32_t)a.b_bytes;
  const uint32_t A_TX = a.row ? (uint32_t)(BM + a.kw - 1) * 128u : (uint32_t)BM * 128u;
  constexpr bool packed = PK;
  // promotion: K-blocks per TMEM accumulation segment, segments per item
  // (balanced: GS = round(nk / drain) segments of DS K-blocks; a short item stays one segment)
  const int GS0 = a.drain > 0 ? max(1, (nk + a.drain / 2) / a.drain) : 1, DS = (nk + GS0 - 1) / GS0;
  const int GS = (nk + DS - 1) / DS;  // the MMA issuer closes a segment every DS K-blocks

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * STAGE);  // full[4], empty[4], tfull[2], tempty[2], sfull[2], sempty[2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * MAXNS + 8);
  const uint32_t sb = su32(smem), b0 = su32(bars);
  auto full_bar = [&](int i) { return b0 + 8u * i; };
  auto empty_bar = [&](int i) { return b0 + 8u * (MAXNS + i); };
  auto tfull_bar = [&](int i) { return b0 + 8u * (2 * MAXNS + i); };
  auto tempty_bar = [&](int i) { return b0 + 8u * (2 * MAXNS + 2 + i); };
  auto sfull_bar = [&](int i) { return b0 + 8u * (2 * MAXNS + 4 + i); };
  auto sempty_bar = [&](int i) { return b0 + 8u * (2 * MAXNS + 6 + i); };

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      bar_init(full_bar(i), 1);
      bar_init(empty_bar(i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(tfull_bar(i), 1);
      bar_init(tempty_bar(i), 32 * EPI);
      bar_init(sfull_bar(i), 1);
      bar_init(sempty_bar(i), 32 * EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_trigger();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();

  if (warp == 0) {  // ---------------------------------------------------------- TMA producer
#if EVC_TMA_WARP
#define ARRIVE_TX_ bar_arrive_tx_w
#define BULK_ bulk_load_w
#define TMA3_ tma_load_3d_w
#define TMA4_ tma_load_4d_w
#else
#define ARRIVE_TX_ bar_arrive_tx
#define BULK_ bulk_load
#define TMA3_ tma_load_3d
#define TMA4_ tma_load_4d
#endif
    int g = 0;  // global stage counter
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int nblk = item % nb, reg = item / nb, s = reg / R, rr = reg % R;
      if (!region_live_warp(a, s, rr)) continue;
      if (EVC_TMA_WARP || lane == 0) {
        const char* wsrc = reinterpret_cast<const char*>(a.wpack) + (int64_t)nblk * a.nkb * B_BYTES;
        int ulo = 0, xlo = 0;
        if (!a.row) {
          ulo = (rr / a.RWn) * a.RH;
          xlo = (rr % a.RWn) * a.RW;
        }
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const int st = g % NS;
          if (g >= NS) bar_spin(empty_bar(st), ((g / NS) & 1) ^ 1);
          const uint32_t abuf = sb + st * STAGE;
          ARRIVE_TX_(full_bar(st), 2 * A_TX + B_BYTES);
          BULK_(abuf + 2 * A_HALF, wsrc + (int64_t)kb * B_BYTES, B_BYTES, full_bar(st));
          if (a.row) {
            const int r = kb / a.cchunks, c0 = (kb % a.cchunks) * 32;
            const int i0 = rr * a.VM + r * a.P;
            TMA3_(abuf, &tmap, 2 * c0, i0, s, full_bar(st));
            TMA3_(abuf + A_HALF, &tmap, 2 * c0 + 32, i0, s, full_bar(st));
          } else {
            const int tap = kb / a.cchunks, c0 = (kb % a.cchunks) * 32;
            const int r = tap / a.kw, qq = tap % a.kw;
            const int xs = xlo * a.stride + qq, ys = ulo * a.stride + r;
            TMA4_(abuf, &tmap, 2 * c0, xs, ys, s, full_bar(st));
            TMA4_(abuf + A_HALF, &tmap, 2 * c0 + 32, xs, ys, s, full_bar(st));
          }
        }
      } else {
        g += nk;
      }
      __syncwarp();
    }
#undef ARRIVE_TX_
#undef BULK_
#undef TMA3_
#undef TMA4_
  } else if (warp == 1) {  // --------------------------------------------------- MMA issuer
#if EVC_MMA_WARP
#define MMA_ mma_w
#define COMMIT_ commit_w
#else
#define MMA_ mma
#define COMMIT_ commit
#endif
    // TMEM buffer use = one accumulation segment of DS K-blocks (the whole item when a.drain == 0);
    // segment gs fills buffer gs & 1 while the epilogue promotes segment gs - 1 into registers
    int g = 0, gs = 0, it = 0;  // it: live items so far (small block it & 1 when SS)
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int reg = item / nb, s = reg / R, rr = reg % R;
      if (!region_live_warp(a, s, rr)) continue;
      if (EVC_MMA_WARP || lane == 0) {  // (warp-wide issue: every lane walks the loop, one elected lane issues)
        uint32_t tb = tmem;
        int ab = 0;
        const uint32_t tsm = tmem + (uint32_t)(2 * BN + (it & 1) * BN);
        if (SS && it >= 2) bar_spin(sempty_bar(it & 1), ((it >> 1) & 1) ^ 1);
        fence_after();
        for (int kb = 0; kb < nk; ++kb, ++g) {
          const bool seg0 = kb % DS == 0;
          if (seg0) {
            ab = gs & 1;
            if (gs >= 2) bar_spin(tempty_bar(ab), ((gs >> 1) & 1) ^ 1);
            fence_after();
            tb = tmem + (uint32_t)(ab * BUF);
          }
          const int st = g % NS;
          bar_spin(full_bar(st), (g / NS) & 1);
          fence_after();
          const uint32_t ah = sb + st * STAGE, al = ah + A_HALF, bb = ah + 2 * A_HALF;
          const int c0k = (kb % a.cchunks) * 32, nkk = min(4, (a.c_in - c0k + 7) >> 3);
          if (packed) {
            const uint32_t idp = IDESC_BASE | ((uint32_t)((a.kw * 2 * BN) >> 3) << 17);
            const uint64_t dl = desc_k(al), dh = desc_k(ah), db = desc_k(bb);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (kk >= nkk) break;
              MMA_(tb, dl + 2 * kk, db + 2 * kk, idp, (!seg0 || kk) ? 1u : 0u);
              MMA_(tb, dh + 2 * kk, db + 2 * kk, idp, 1u);
            }
          } else {
            const int taps = a.row ? a.kw : 1;
            for (int t = 0; t < taps; ++t) {
              const uint64_t da = desc_k(ah + t * 128), dl = desc_k(al + t * 128), db = desc_k(bb + t * 2 * BN * 128);
              const bool first = seg0 && t == 0;
              if constexpr (SS) {
                const uint64_t dbl = desc_k(bb + BN * 128);  // B_lo rows of the [B_hi | B_lo] tile
                const bool firsts = kb == 0 && t == 0;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  if (kk >= nkk) break;
                  MMA_(tb, da + 2 * kk, db + 2 * kk, IDESC, (!first || kk) ? 1u : 0u);      // hi.hi
                  MMA_(tsm, da + 2 * kk, dbl + 2 * kk, IDESC, (!firsts || kk) ? 1u : 0u);  // hi.lo
                  MMA_(tsm, dl + 2 * kk, db + 2 * kk, IDESC, 1u);                           // lo.hi
                }
              } else {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                  if (kk >= nkk) break;
                  MMA_(tb, da + 2 * kk, db + 2 * kk, IDESC2, (!first || kk) ? 1u : 0u);           // hi.[hi|lo]
                  MMA_(tb + 2 * BN, dl + 2 * kk, db + 2 * kk, IDESC, (!first || kk) ? 1u : 0u);  // lo.hi
                }
              }
            }
          }
          COMMIT_(empty_bar(st));
          if (kb % DS == DS - 1 || kb == nk - 1) {
            COMMIT_(tfull_bar(ab));
            ++gs;
          }
        }
        if (SS) COMMIT_(sfull_bar(it & 1));
      } else {
        g += nk;
      }
      ++it;
      __syncwarp();
    }
#undef MMA_
#undef COMMIT_
  } else if (warp < 4) {  // ---------------------------------------------------- flags + meter
    if (!a.dense) {
      const int Qs = R * nb;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int nblk = item % nb, reg = item / nb, s = reg / R, rr = reg % R;
        side_work(a, s, nblk * R + rr, Qs, threadIdx.x - 64);
      }
    }
  } else {  // -------------------------------------------------------------------- epilogue
    __shared__ float s_xch[NH][4][3][3][8];
    __shared__ double s_red[EPI];
    const int q4 = warp & 3, m = 32 * q4 + lane;
    const int half = NH > 1 ? (warp - 4) >> 2 : 0;  // channel half of the block (NH = 2) or 0
    // named barrier of this half's four warps: id 2 (half 0) or 4 (half 1)
    const int Qs = R * nb;
    int gs = 0, it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int nblk = item % nb, reg = item / nb, s = reg / R, rr = reg % R;
      const int64_t rs_idx = (int64_t)reg * nb + nblk;
      const bool live = region_live_warp(a, s, rr);
      int u, x;
      site_of(a, rr, m, u, x);
      double ssq = 0.0;
      const int prev = a.dense ? 0 : a.rstate[rs_idx];
      if (!live) {
        if (prev) {  // computed last step, dead now: restore exact zeros
          const int n0 = nblk * BN, nn = min(BN, a.c_out - n0);
          if (u < a.Ho && x < a.Wo)
            for (int n = n0 + half; n < n0 + nn; n += NH) zero_site(a, s, u, x, n);
        }
      } else {
        const int sl = sub_live_of(a, s, u, x);
        prefetch_acc(a, s, u, x, nblk * BN + half * (BN / NH), BN / NH);
        if (packed) {
          // per segment and 8-channel chunk: v_s = A.B_lo + A.B_hi of tap s, out[m] = sum_s v_s[m + s]
          // (shifts by s rows = shuffles inside the warp, the next warp's first rows through shared
          // memory), accumulated over the segments
          const int KW = a.kw;
          constexpr int PB = BN <= 32 ? BN : 8;  // (packed mode only runs with BN <= 32)
          constexpr int CH = PB / NH < 8 ? 8 : PB / NH;  // channels of this half (BN = 64: never packed)
          float O[CH];
#pragma unroll 1
          for (int sg = 0; sg < GS; ++sg, ++gs) {
            const int ab = gs & 1;
            bar_wait(tfull_bar(ab), (gs >> 1) & 1);
            fence_after();
            const uint32_t trow = tmem + (uint32_t)(ab * BUF) + ((uint32_t)(32 * q4) << 16);
#pragma unroll
            for (int cc = 0; cc < CH; cc += 8) {
              const int c0 = half * CH + cc;
              float v[3][8];
              {
                uint32_t r4[3][2][8];
#pragma unroll
                for (int s2 = 0; s2 < 3; ++s2)
                  if (s2 < KW) {
                    const uint32_t cb = (uint32_t)(s2 * 2 * BN + c0);
                    tmem_ld8_issue(trow + cb + BN, r4[s2][0]);
                    tmem_ld8_issue(trow + cb, r4[s2][1]);
                  }
                tmem_wait_ld();
#pragma unroll
                for (int s2 = 0; s2 < 3; ++s2)
#pragma unroll
                  for (int j = 0; j < 2; ++j)
#pragma unroll
                    for (int e = 0; e < 8; ++e) asm volatile("" : "+r"(r4[s2][j][e]));
#pragma unroll
                for (int s2 = 0; s2 < 3; ++s2)
#pragma unroll
                  for (int e = 0; e < 8; ++e)
                    v[s2][e] = s2 < KW ? __fadd_rn(__uint_as_float(r4[s2][0][e]), __uint_as_float(r4[s2][1][e])) : 0.0f;
              }
              if (cc + 8 >= CH) {  // this thread's last TMEM read of the buffer
                fence_before();
                bar_arrive(tempty_bar(ab));
              }
#pragma unroll
              for (int s2 = 1; s2 < 3; ++s2)
                if (s2 < KW && lane < s2) {
#pragma unroll
                  for (int e = 0; e < 8; ++e) s_xch[half][q4][s2][lane][e] = v[s2][e];
                }
              if (half == 0)
                asm volatile("bar.sync 2, 128;" ::: "memory");
              else
                asm volatile("bar.sync 4, 128;" ::: "memory");
              float o[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = v[0][e];
#pragma unroll
              for (int s2 = 1; s2 < 3; ++s2) {
                if (s2 >= KW) break;
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  float t = __shfl_down_sync(0xffffffffu, v[s2][e], s2);
                  if (lane >= 32 - s2) t = q4 < 3 ? s_xch[half][q4 + 1][s2][lane + s2 - 32][e] : 0.0f;
                  o[e] = __fadd_rn(o[e], t);
                }
              }
              if (half == 0)
                asm volatile("bar.sync 2, 128;" ::: "memory");
              else
                asm volatile("bar.sync 4, 128;" ::: "memory");
#pragma unroll
              for (int e = 0; e < 8; ++e) O[cc + e] = sg ? __fadd_rn(O[cc + e], o[e]) : o[e];
            }
          }
          const int n0 = nblk * BN;
#pragma unroll
          for (int cc = 0; cc < CH; cc += 8) {
            const int c0 = half * CH + cc;
            ssq += emit<8>(a, s, u, x, n0 + c0, 1, min(8, a.c_out - n0 - c0), O + cc, sl);
          }
        } else {
          constexpr int CB = BN / NH;  // channels of this half
          float acc[CB];               // (lo.hi + hi.lo) + hi.hi, summed over the segments
#pragma unroll 1
          for (int sg = 0; sg < GS; ++sg, ++gs) {
            const int ab = gs & 1;
            bar_wait(tfull_bar(ab), (gs >> 1) & 1);
            fence_after();
            const uint32_t trow = tmem + (uint32_t)(ab * BUF) + ((uint32_t)(32 * q4) << 16);
            if constexpr (SS) {
#pragma unroll
              for (int cc = 0; cc < CB; cc += 32) {  // hi . hi of this segment
                const int c0 = half * CB + cc;
                uint32_t r[2][16];
                tmem_ld16_issue(trow + (uint32_t)c0, r[0]);
                tmem_ld16_issue(trow + (uint32_t)(c0 + 16), r[1]);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 2; ++j)
#pragma unroll
                  for (int e = 0; e < 16; ++e) {
                    asm volatile("" : "+r"(r[j][e]));
                    const float v = __uint_as_float(r[j][e]);
                    acc[cc + 16 * j + e] = sg ? __fadd_rn(acc[cc + 16 * j + e], v) : v;
                  }
              }
            } else {
#pragma unroll
              for (int cc = 0; cc < CB; cc += 16) {
                const int c0 = half * CB + cc;
                uint32_t r[3][16];
                tmem_ld16_issue(trow + (uint32_t)(2 * BN + c0), r[0]);  // lo . hi
                tmem_ld16_issue(trow + (uint32_t)(BN + c0), r[1]);      // hi . lo
                tmem_ld16_issue(trow + (uint32_t)c0, r[2]);             // hi . hi
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 3; ++j)
#pragma unroll
                  for (int e = 0; e < 16; ++e) asm volatile("" : "+r"(r[j][e]));
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  const float v = __fadd_rn(__fadd_rn(__uint_as_float(r[0][e]), __uint_as_float(r[1][e])),
                                            __uint_as_float(r[2][e]));
                  acc[cc + e] = sg ? __fadd_rn(acc[cc + e], v) : v;
                }
              }
            }
            fence_before();
            bar_arrive(tempty_bar(ab));
          }
          if constexpr (SS) {  // + the item's small terms (hi.lo + lo.hi, one chain over the whole K range)
            bar_wait(sfull_bar(it & 1), (it >> 1) & 1);
            fence_after();
            const uint32_t srow = tmem + (uint32_t)(2 * BN + (it & 1) * BN) + ((uint32_t)(32 * q4) << 16);
#pragma unroll
            for (int cc = 0; cc < CB; cc += 32) {
              const int c0 = half * CB + cc;
              uint32_t r[2][16];
              tmem_ld16_issue(srow + (uint32_t)c0, r[0]);
              tmem_ld16_issue(srow + (uint32_t)(c0 + 16), r[1]);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 2; ++j)
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                  asm volatile("" : "+r"(r[j][e]));
                  acc[cc + 16 * j + e] = __fadd_rn(__uint_as_float(r[j][e]), acc[cc + 16 * j + e]);
                }
            }
            fence_before();
            bar_arrive(sempty_bar(it & 1));
          }
#pragma unroll
          for (int cc = 0; cc < CB; cc += 16) {
            const int n0 = nblk * BN + half * CB + cc;
            ssq += emit<16, (BN >= 64 && !PK)>(a, s, u, x, n0, 1, min(16, a.c_out - n0), acc + cc, sl);
          }
        }
        ++it;
      }
      // per-item bookkeeping: region state, sum of squares of the fused sparsify
      if (a.sp_part) {
        const double w = warp_sum_d(ssq);
        if (lane == 0) s_red[warp - 4] = w;
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * EPI) : "memory");
      if (threadIdx.x == 128) {
        double tot = 0.0;
#pragma unroll
        for (int w = 0; w < EPI; ++w) tot += s_red[w];
        if (a.sp_part) a.sp_part[(int64_t)s * Qs + nblk * R + rr] = tot;
        if (!a.dense && live != (prev != 0)) a.rstate[rs_idx] = live ? 1 : 0;
      }
      asm volatile("bar.sync 3, %0;" ::"n"(32 * EPI) : "memory");
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// CUDA-core path for thin convs (C_in <= 8 or C_out <= 8, C_out <= 32): the prediction heads
// (1x1, C_out = 2) and the 4-channel input layer waste most of a 128-row tensor-core tile and
// all of its 32-channel K-blocks.  Same regions, region test, flags / meter side work and fused
// epilogue as k_conv_fused; the values are exact fp32 FFMA sums over the hi/lo shadow
// (head + tail = the float32 input exactly).  One thread per output site, weights in shared
// memory as [tap][c_in][c_out].
constexpr int THIN_THREADS = BM;

// acc[n] += x * w[n] for CO weights in shared memory (16-byte broadcast reads when CO % 4 == 0)
template <int CO>
__device__ __forceinline__ void thin_fma(float* acc, float x, const float* w) {
  if (CO % 4 == 0) {
#pragma unroll
    for (int n = 0; n < CO; n += 4) {
      const float4 w4 = *reinterpret_cast<const float4*>(w + n);
      acc[n] = __fmaf_rn(x, w4.x, acc[n]);
      acc[n + 1] = __fmaf_rn(x, w4.y, acc[n + 1]);
      acc[n + 2] = __fmaf_rn(x, w4.z, acc[n + 2]);
      acc[n + 3] = __fmaf_rn(x, w4.w, acc[n + 3]);
    }
  } else {
#pragma unroll
    for (int n = 0; n < CO; ++n) acc[n] = __fmaf_rn(x, w[n], acc[n]);
  }
}

// output channels padded to CO (2, 4, 8, 16, 32); weights [tap][c_in][CO]; F32: fp32 shadow (cp < 0)
template <int CO, bool F32 = false>
#ifndef EVC_THIN_MINB32
#define EVC_THIN_MINB32 6
#endif
#ifndef EVC_THIN_MINB
#define EVC_THIN_MINB 8
#endif
__global__ void __launch_bounds__(THIN_THREADS, (CO >= 32 ? EVC_THIN_MINB32 : EVC_THIN_MINB)) k_conv_thin(const float* __restrict__ in_hwc, int64_t hwc_stride,
                                                            const __grid_constant__ Args a) {
  extern __shared__ float s_w[];
  __shared__ int s_flag[2];
  __shared__ double s_red[THIN_THREADS / 32];
  const int R = a.R;
  const int reg = blockIdx.x, s = reg / R, rr = reg % R;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = a.kh * a.kw * a.c_in * CO;
  for (int e = threadIdx.x; e < nw; e += THIN_THREADS) s_w[e] = a.wpack[e];
  pdl_trigger();
  pdl_wait();
  const int ulo = (rr / a.RWn) * a.RH, uhi = min(ulo + a.RH, a.Ho) - 1;
  const int xlo = (rr % a.RWn) * a.RW, xhi = min(xlo + a.RW, a.Wo) - 1;
  if (warp == 0) {
    int live = 1;
    if (!a.dense) {
      live = 0;
      const int y_lo = max(0, ulo * a.stride - a.pad), y_hi = min(a.H - 1, uhi * a.stride - a.pad + a.kh - 1);
      const int x_lo = max(0, xlo * a.stride - a.pad), x_hi = min(a.W - 1, xhi * a.stride - a.pad + a.kw - 1);
      if (y_lo <= y_hi && x_lo <= x_hi) {
        const int GWi = (a.W + a.tw - 1) / a.tw, GHi = (a.H + a.th - 1) / a.th;
        const int ra = y_lo / a.th, nr = y_hi / a.th - ra + 1, ca = x_lo / a.tw, nc = x_hi / a.tw - ca + 1;
        const uint8_t* fa = a.fany + (int64_t)s * GHi * GWi;
        for (int e = lane; e < nr * nc; e += 32) live |= fa[(ra + e / nc) * GWi + ca + e % nc];
      }
      live = __any_sync(0xffffffffu, live);
    }
    if (lane == 0) {
      s_flag[0] = live;
      s_flag[1] = a.dense ? 0 : a.rstate[reg];
    }
  }
  __syncthreads();
  const int Qs = R, q = rr;
  if (!a.dense && warp < 2) side_work(a, s, q, Qs, threadIdx.x);
  int u, x;
  site_of(a, rr, threadIdx.x, u, x);
  const bool valid = u < a.Ho && x < a.Wo;
  double ssq = 0.0;
  if (!s_flag[0]) {
    if (!a.dense && s_flag[1]) {  // computed last step, dead now: restore exact zeros
      for (int n = 0; n < a.c_out && valid; ++n) {
        const int64_t off = (int64_t)n * a.Ho * a.Wo + (int64_t)u * a.Wo + x;
        if (a.out) a.out[(int64_t)s * a.ovs + off] = 0.0f;
        if (a.yact) a.yact[(int64_t)s * a.yvs + off] = 0.0f;
        if (a.sp_hwc) hwc_store(a.sp_hwc + (int64_t)s * a.sp_hs + ((int64_t)u * a.sp_pitch + x) * hwc_px(a.sp_cp), a.sp_cp, n, 0.0f);
      }
      if (threadIdx.x == 0) a.rstate[reg] = 0;
    }
  } else {
    if (!a.dense && threadIdx.x == 0 && !s_flag[1]) a.rstate[reg] = 1;
    if (valid) prefetch_acc(a, s, u, x, 0, a.c_out);
    float acc[CO];
#pragma unroll
    for (int n = 0; n < CO; ++n) acc[n] = 0.0f;
    if (valid) {
      const float* base = in_hwc + (int64_t)s * hwc_stride;
      constexpr bool f32 = F32;
      for (int r = 0; r < a.kh; ++r)
        for (int q2 = 0; q2 < a.kw; ++q2) {
          const float* px = base + ((int64_t)(u * a.stride + r) * a.P + x * a.stride + q2) * hwc_px(a.cp);
          const float* wt = s_w + (r * a.kw + q2) * a.c_in * CO;
          // four channel values at c (16 bytes of an fp32 shadow, or head + tail runs)
          auto ld4 = [&](int c) -> float4 {
            if (f32) return *reinterpret_cast<const float4*>(px + c);
            const float4 h = *reinterpret_cast<const float4*>(px + hwc_head(a.cp, c));
            const float4 l = *reinterpret_cast<const float4*>(px + hwc_head(a.cp, c) + hwc_unit(a.cp));
            return make_float4(__fadd_rn(h.x, l.x), __fadd_rn(h.y, l.y), __fadd_rn(h.z, l.z), __fadd_rn(h.w, l.w));
          };
          int c = 0;
          if ((a.c_in & 3) == 0) {  // 8 channels per round: 16-byte loads in flight
            for (; c + 8 <= a.c_in; c += 8) {
              const float4 v0 = ld4(c), v1 = ld4(c + 4);
              const float xv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
              for (int k = 0; k < 8; ++k) thin_fma<CO>(acc, xv[k], wt + (c + k) * CO);
            }
            for (; c + 4 <= a.c_in; c += 4) {
              const float4 v0 = ld4(c);
              thin_fma<CO>(acc, v0.x, wt + c * CO);
              thin_fma<CO>(acc, v0.y, wt + (c + 1) * CO);
              thin_fma<CO>(acc, v0.z, wt + (c + 2) * CO);
              thin_fma<CO>(acc, v0.w, wt + (c + 3) * CO);
            }
          }
          for (; c < a.c_in; ++c)  // head + tail
            thin_fma<CO>(acc, f32 ? px[c] : __fadd_rn(px[hwc_head(a.cp, c)], px[hwc_head(a.cp, c) + hwc_unit(a.cp)]),
                         wt + c * CO);
        }
    }
    constexpr int E = CO < 16 ? CO : 16;
    ssq += emit<E>(a, s, u, x, 0, 1, min(E, a.c_out), acc);
    if (CO > 16) ssq += emit<E>(a, s, u, x, 16, 1, a.c_out - 16, acc + (CO > 16 ? 16 : 0));
  }
  if (a.sp_part) {
    double v = warp_sum_d(ssq);
    if (lane == 0) s_red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < THIN_THREADS / 32; ++w) t += s_red[w];
      a.sp_part[(int64_t)s * Qs + q] = t;
    }
  }
}

static int thin_co(int c_out) { return c_out <= 2 ? 2 : (c_out <= 4 ? 4 : (c_out <= 8 ? 8 : (c_out <= 16 ? 16 : 32))); }

// any-channel tile map: fany[s][t] = OR_c flags[s][c][t]
__global__ void k_tile_any(TView x, uint8_t* __restrict__ fany) {
  pdl_wait();
  pdl_trigger();
  const int Ti = x.GH * x.GW;
  const int s = blockIdx.y;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < Ti; t += gridDim.x * blockDim.x) {
    int any = 0;
    for (int c0 = 0; c0 < x.C && !any; c0 += 8) {  // eight independent loads in flight per test
      uint8_t f[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = c0 + k < x.C ? x.fplane(s, c0 + k)[t] : 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) any |= f[k];
    }
    fany[(int64_t)s * Ti + t] = any != 0;
  }
}

// End-of-step bookkeeping (graph.py:617-636), one launch.  Block (l, s) < n*S resolves meter
// node l of session s: a fused conv sums its per-CTA partials (live input flags, weighted term;
// integer, so exact in any order) and applies the reference's all-false / all-true shortcuts
// (increment_ops.py:148-154); other nodes already hold `performed`.  Then perf_cum and the
// false-tile fraction.  Block n*S + j folds sparsify node j's per-CTA sums of squares into
// norm_ema / k (sparsify.py:72-76) in a fixed order; k is first read by the NEXT step's
// sparsify of that node, so folding at the end of the step is the reference's sequence.
__global__ void __launch_bounds__(256) k_meter_step(const evc_meter_node* __restrict__ nodes, int n, int S,
                                                    int32_t* in_true, long long* perf_step, long long* perf_cum,
                                                    double* ff_last, double* ff_sum,
                                                    const evc_sp_node* __restrict__ sp) {
  pdl_wait();
  pdl_trigger();
  if ((int)blockIdx.x >= n * S) {  // one (sparsify node, session) per block: its partials in fixed order
    const int b = blockIdx.x - n * S, j = b / S, s = b % S;
    const evc_sp_node nd = sp[j];
    sparsify_finalize_all(nd.partials, nd.n, nd.norm_ema, nd.k, nd.tp, nd.decay, 0, s + 1, s);
    return;
  }
  const int l = blockIdx.x / S, s = blockIdx.x % S, e = l * S + s;
  const evc_meter_node nd = nodes[l];
  long long cnt, p;
  if (nd.part) {
    long long c = 0, w = 0;
    const long long* mp = reinterpret_cast<const long long*>(nd.part) + (int64_t)s * nd.n * 2;
    for (int64_t i = threadIdx.x; i < nd.n; i += blockDim.x) {
      c += mp[2 * i];
      w += mp[2 * i + 1];
    }
    c = block_sum<long long>(c, [](long long v) { return warp_sum_ll(v); });
    __syncthreads();
    w = block_sum<long long>(w, [](long long v) { return warp_sum_ll(v); });
    if (threadIdx.x != 0) return;
    cnt = c;
    in_true[e] = (int32_t)c;
    p = cnt == 0 ? 0LL : (cnt == nd.nflags ? nd.dense : 2LL * nd.c_out * w);
    perf_step[e] = p;
  } else {
    if (threadIdx.x != 0) return;
    cnt = in_true[e];
    p = perf_step[e];
  }
  perf_cum[e] += p;
  const double ff = __dsub_rn(1.0, __ddiv_rn((double)cnt, (double)nd.nflags));
  ff_last[e] = ff;
  ff_sum[e] = __dadd_rn(ff_sum[e], ff);
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}

template <int BN>
static cudaError_t launch(const CUtensorMap& m, const Args& a, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(a.S * a.R), (unsigned)((a.c_out + BN - 1) / BN), (unsigned)a.splits);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = (size_t)a.ns * a.stage + 1024 + 256;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (a.splits > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = 1;
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = (unsigned)a.splits;
    ++na;
  }
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k_conv_fused<BN>, m, a);
}

constexpr int SMEM_MAX = 227 * 1024;
constexpr int STAGE_BUDGET = SMEM_MAX - 1024 - 256 - 2048;

template <int BN, bool PK>
static int attr_persist1() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_conv_persist<BN, PK>) != cudaSuccess) return 1;
  return cudaFuncSetAttribute(k_conv_persist<BN, PK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              SMEM_MAX - (int)fa.sharedSizeBytes) == cudaSuccess
             ? 0
             : 1;
}
template <int BN>
static int attr_persist() {
  return attr_persist1<BN, false>() | (BN <= 32 ? attr_persist1<BN, true>() : 0);
}

template <int BN>
static cudaError_t launch_persist(const CUtensorMap& m, const Args& a, int grid, cudaStream_t st) {
  const size_t smem = (size_t)a.ns * a.stage + 1024 + 256;
  if (BN <= 32 && a.row == 2)
    return launch_pdl(k_conv_persist<BN, (BN <= 32)>, dim3((unsigned)grid), dim3(persist_threads<BN>()), smem, st, m, a);
  return launch_pdl(k_conv_persist<BN, false>, dim3((unsigned)grid), dim3(persist_threads<BN>()), smem, st, m, a);
}

template <int BN>
static int attr() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_conv_fused<BN>) != cudaSuccess) return 1;
  if (cudaFuncSetAttribute(k_conv_fused<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           SMEM_MAX - (int)fa.sharedSizeBytes) != cudaSuccess)
    return 1;
  return cudaFuncSetAttribute(k_conv_fused<BN>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess
             ? 0
             : 1;
}

static bool valid_bn(int bn) { return bn == 16 || bn == 32 || bn == 64 || bn == 128 || bn == 256; }

// Pipeline layout of one configuration: stage = [A heads | A tails | B], A halves 1 KiB aligned.
struct Layout {
  int ns, stage, a_half, b_bytes, R, nkb, cchunks, VM = BM;
};

static Layout layout_of(const evc_conv_geom* g, const evc_conv_cfg* cfg) {
  Layout L;
  L.cchunks = (g->c_in + 31) / 32;
  if (cfg->thin) {
    L.R = ((g->Ho + cfg->rh - 1) / cfg->rh) * ((g->Wo + cfg->rw - 1) / cfg->rw);
    L.nkb = 1;
    L.ns = 1;
    L.a_half = L.b_bytes = 0;
    L.stage = g->kh * g->kw * g->c_in * thin_co(g->c_out) * 4;  // weights in shared memory
    return L;
  }
  if (cfg->row) {
    L.a_half = ((BM + g->kw - 1 + 7) / 8) * 8 * 128;
    L.b_bytes = g->kw * 2 * cfg->bn * 128;
    L.nkb = g->kh * L.cchunks;
    const int P = g->W + 2 * g->pad;
    L.VM = cfg->row == 2 ? BM - (g->kw - 1) : BM;
    L.R = (int)(((int64_t)g->Ho * P + L.VM - 1) / L.VM);
  } else {
    L.a_half = BM * 128;
    L.b_bytes = 2 * cfg->bn * 128;
    L.nkb = g->kh * g->kw * L.cchunks;
    L.R = ((g->Ho + cfg->rh - 1) / cfg->rh) * ((g->Wo + cfg->rw - 1) / cfg->rw);
  }
  L.a_half = (L.a_half + 1023) / 1024 * 1024;
  L.stage = 2 * L.a_half + L.b_bytes;
  L.stage = (L.stage + 1023) / 1024 * 1024;
  L.ns = std::max(1, std::min(4, STAGE_BUDGET / L.stage));
  // two co-resident CTAs per SM when two stages of each fit and the accumulators fit half of TMEM:
  // one CTA's prologue / epilogue then overlaps the other's MMA stream
  const int bn = cfg->bn, na = bn >= 128 ? 1 : (bn >= 32 ? 3 : 4);
  int need = bn <= 128 ? na * 2 * bn + bn : 2 * bn;
  if (bn <= 32) need = std::max(need, 6 * bn);  // the kernel sizes TMEM for the packed mode too
  if (need <= 256 && 2 * (2 * L.stage + 1024 + 256 + 1024) <= SMEM_MAX && !getenv("EVC_NO_OCC2")) L.ns = 2;
  return L;
}

static int split_count(int nkb, int splits) {
  int sp = std::max(1, std::min(splits, nkb));
  const int kbps = (nkb + sp - 1) / sp;
  return (nkb + kbps - 1) / kbps;
}

}  // namespace fz

int init_conv_fused() {
  int rc = fz::attr<16>() | fz::attr<32>() | fz::attr<64>() | fz::attr<128>() | fz::attr<256>();
  rc |= fz::attr_persist<16>() | fz::attr_persist<32>() | fz::attr_persist<64>() | fz::attr_persist<128>();
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, fz::k_tile_any) != cudaSuccess) rc = 1;
  if (cudaFuncGetAttributes(&fa, fz::k_meter_step) != cudaSuccess) rc = 1;
  if (cudaFuncGetAttributes(&fa, fz::k_conv_thin<2>) != cudaSuccess) rc = 1;
  if (cudaFuncGetAttributes(&fa, fz::k_conv_thin<4>) != cudaSuccess) rc = 1;
  if (cudaFuncGetAttributes(&fa, fz::k_conv_thin<8>) != cudaSuccess) rc = 1;
  if (cudaFuncGetAttributes(&fa, fz::k_conv_thin<16>) != cudaSuccess) rc = 1;
  if (cudaFuncGetAttributes(&fa, fz::k_conv_thin<32>) != cudaSuccess) rc = 1;
  return rc ? EVC_ECUDA : EVC_OK;
}

}  // namespace evc

using namespace evc;

extern "C" {

int evc_conv_fused_supported(const evc_conv_geom* g) {
  if (!g) return 0;
  // pad >= K: the all-true shortcut (increment_ops.py:150-154) can mark tiles whose
  // box holds only padding -- the unfused path keeps that corner exact.
  return g->stride >= 1 && g->stride <= 8 && g->stride * 32 <= 256 && g->pad < g->kh && g->pad < g->kw &&
         fz::encoder() != nullptr;
}

int evc_conv_fused_config(const evc_conv_geom* g, int32_t S, int32_t max_splits, evc_conv_cfg* cfg) {
  EVC_CHECK_ARG(g && cfg && S > 0, "conv_fused_config: null argument");
  cfg->drain = 0;
  // stride 1: row mode (halo rows loaded once for all kw taps); else tap mode over RH x RW regions
  cfg->thin = ((g->c_in <= 8 || g->c_out <= 8) && g->c_out <= 32 &&
               (int64_t)g->kh * g->kw * g->c_in * g->c_out * 4 <= 48 * 1024)
                  ? 1
                  : 0;
  // row mode caps BN at 64 (kw taps of weights per stage); with C_out >= 128 the wider channel
  // block of tap mode wins (fewer MMA cycles per output, the A tile read once per 128+ outputs;
  // measured: res 256->256 @16x16 96 vs 128 us, dec0 512->128 @32x32 268 vs 306 us at 32 streams;
  // with few streams the row mode's shorter per-region latency wins)
  cfg->row = (!cfg->thin && g->stride == 1 && g->kw <= 9 && g->Wo == g->W + 2 * g->pad - g->kw + 1 &&
              (g->c_out <= 64 || S < 8) && std::getenv("EVC_NO_ROW") == nullptr)
                 ? 1
                 : 0;
  if (cfg->thin) {
    cfg->rw = g->Wo > 16 ? 32 : (g->Wo > 8 ? 16 : 8);
    cfg->rh = fz::BM / cfg->rw;
    cfg->bn = 16;
    cfg->splits = 1;
    return EVC_OK;
  }
  if (cfg->row) {
    cfg->rh = 1;
    cfg->rw = fz::BM;
  } else {
    cfg->rw = g->Wo > 16 ? 32 : (g->Wo > 8 ? 16 : 8);
    if (const char* fr = std::getenv("EVC_FORCE_RW")) cfg->rw = std::max(8, std::min(atoi(fr), 32));
    cfg->rh = fz::BM / cfg->rw;
  }
  // BN <= 128 with many streams: N = 256 (hi.[hi|lo]) + N = 128 (lo.hi) per K8 step and twice the
  // CTAs of BN = 256 (measured at 32 streams: enc3 59 vs 75 us, res 85 vs 96 us)
  int bn = 16;
  while (bn < g->c_out && bn < (S >= 8 ? 128 : 256)) bn *= 2;
  if (cfg->row && bn > 64) bn = 64;  // kw taps of B per stage: keep >= 2 stages
  if (const char* fb = std::getenv("EVC_FORCE_BN")) bn = std::max(16, std::min(atoi(fb), cfg->row ? 64 : 256));
  cfg->bn = bn;
  // packed row mode: all kw taps of a K-block in ONE MMA along N (tcgen05.mma costs the same for
  // any N <= 128), shifted and summed in the epilogue: kw x fewer MMA instructions for thin C_out
  if (cfg->row && bn <= 32 && g->kw <= 3 && 2 * g->kw * bn <= 256 && std::getenv("EVC_NO_PACK") == nullptr)
    cfg->row = 2;
  const int msp = std::max(1, std::min<int>(max_splits > 0 ? max_splits : 8, 16));
  fz::Layout L = fz::layout_of(g, cfg);
  const int64_t regions = (int64_t)S * L.R;
  while (bn > 64 && regions * ((g->c_out + bn - 1) / bn) * msp < 148) {
    bn /= 2;
    cfg->bn = bn;
  }
  L = fz::layout_of(g, cfg);
  const int64_t ctas = regions * ((g->c_out + bn - 1) / bn);
  // split-K only for short grids: from ~2/3 of the SMs on, the extra partial traffic and the
  // cluster reduce cost more than the idle SMs (res 128 CTAs: 79 vs 85 us, enc3 54 vs 59 us)
  // short grids: about 96 CTAs in one wave (more ranks cost more in the cluster reduce than
  // they win; measured at one stream: dec0 / dec1 best at 4-5 ranks, res / enc3 at 8)
  int sp = ctas >= 96 ? 1
                      : (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)msp, (96 + ctas / 2) / ctas, 148 / ctas}));
  if (const char* fs = std::getenv("EVC_FORCE_SPLITS")) sp = std::max(1, std::min(atoi(fs), 16));
  if (cfg->row == 2) sp = 1;  // the packed epilogue sums shifted rows of one CTA's accumulators
  cfg->splits = fz::split_count(L.nkb, sp);
  // Promotion: the TMEM partial sums are added into fp32 registers every K-block (row mode: kw taps per
  // K-block) or every two (tap mode, packed row mode).  The tensor core's accumulate truncates, and an
  // unpromoted chain drifts with its length (dec0 unsplit: 576 K8 steps, ~1e-5 relative per layer --
  // enough to break 1e-4 at the network output); segments of <= 12 K8 steps keep fp32-level accuracy.
  // Segment lengths (measured at 32 streams, C1 over 32 increments: 4.7e-5 max error, 1 % slower than
  // 8-K-block segments at 8.5e-5): tap / packed mode 4 K-blocks (16 K8 steps), row mode 2 (one-shot,
  // 24) or 3 (persistent, 36).  The dense pass uses 1 / 2 (evc_conv_fused).
  if (cfg->bn <= 128) cfg->drain = cfg->row == 1 ? ((cfg->bn > 64 || cfg->splits > 1) ? 2 : 3) : 4;
  if (const char* d = std::getenv("EVC_DRAIN")) cfg->drain = std::max(0, atoi(d));
  return EVC_OK;
}

int64_t evc_conv_fused_pack_len(const evc_conv_geom* g, const evc_conv_cfg* cfg) {
  if (!g || !cfg || !fz::valid_bn(cfg->bn)) return -1;
  if (cfg->thin) return (int64_t)g->kh * g->kw * g->c_in * fz::thin_co(g->c_out);
  const int64_t nb = (g->c_out + cfg->bn - 1) / cfg->bn, nkb = (int64_t)g->kh * g->kw * ((g->c_in + 31) / 32);
  return nb * nkb * 2 * cfg->bn * 32;
}

int evc_conv_fused_pack(const float* w, const evc_conv_geom* g, const evc_conv_cfg* cfg, float* out) {
  EVC_CHECK_ARG(w && g && cfg && out && fz::valid_bn(cfg->bn), "conv_fused_pack: bad argument");
  const int bn = cfg->bn, c_out = g->c_out, c_in = g->c_in, kh = g->kh, kw = g->kw;
  if (cfg->thin) {  // plain fp32 [tap][c_in][CO], output channels zero-padded to CO
    const int co = fz::thin_co(c_out);
    for (int r = 0; r < kh; ++r)
      for (int q = 0; q < kw; ++q)
        for (int c = 0; c < c_in; ++c)
          for (int n = 0; n < co; ++n)
            out[(((int64_t)r * kw + q) * c_in + c) * co + n] =
                n < c_out ? w[(((int64_t)n * c_in + c) * kh + r) * kw + q] : 0.0f;
    return EVC_OK;
  }
  const int cch = (c_in + 31) / 32;
  const int64_t nb = (c_out + bn - 1) / bn, nkb = (int64_t)kh * kw * cch;
  for (int64_t b = 0; b < nb; ++b)
    for (int r = 0; r < kh; ++r)
      for (int q = 0; q < kw; ++q)
        for (int ch = 0; ch < cch; ++ch) {
          // tap mode: K-block (tap, chunk); row mode: K-block (kernel row, chunk) holding its kw taps
          const int64_t blk = cfg->row ? ((int64_t)r * cch + ch) * kw + q : ((int64_t)r * kw + q) * cch + ch;
          float* hi = out + ((b * nkb + blk) * 2) * bn * 32;
          float* lo = hi + (int64_t)bn * 32;
          const int c0 = ch * 32;
          for (int row = 0; row < bn; ++row)
            for (int e = 0; e < 32; ++e) {
              const int64_t n = b * bn + row;
              const int c = c0 + e;
              const float x = (n < c_out && c < c_in) ? w[((n * c_in + c) * kh + r) * kw + q] : 0.0f;
              uint32_t bits;
              memcpy(&bits, &x, 4);
              bits = (bits + 0x1000u) & 0xFFFFE000u;  // round to nearest TF32 (as tf32_head, common.cuh)
              float hv;
              memcpy(&hv, &bits, 4);
              // 128B swizzle: 16-byte chunk j of row `row` lives at chunk (j ^ (row & 7))
              const int j = e / 4, sub = e % 4;
              const int64_t pos = (int64_t)row * 32 + ((j ^ (row & 7)) * 4) + sub;
              hi[pos] = hv;
              lo[pos] = x - hv;
            }
        }
  return EVC_OK;
}

int64_t evc_conv_fused_ctas(const evc_conv_geom* g, const evc_conv_cfg* cfg) {
  if (!g || !cfg || !fz::valid_bn(cfg->bn)) return -1;
  const fz::Layout L = fz::layout_of(g, cfg);
  if (cfg->thin) return L.R;
  return (int64_t)L.R * ((g->c_out + cfg->bn - 1) / cfg->bn) * fz::split_count(L.nkb, cfg->splits);
}

int64_t evc_conv_fused_state_len(const evc_conv_geom* g, const evc_conv_cfg* cfg, int32_t S) {
  if (!g || !cfg || !fz::valid_bn(cfg->bn)) return -1;
  const fz::Layout L = fz::layout_of(g, cfg);
  if (cfg->thin) return (int64_t)S * L.R;
  return (int64_t)S * L.R * ((g->c_out + cfg->bn - 1) / cfg->bn);
}

static int conv_fused_impl(const evc_conv_geom* g, const evc_conv_cfg* cfg_in, const float* in_hwc, int32_t cp,
                           int64_t hwc_stride, const float* wpack, const float* bias, const evc_tensor* in,
                           const uint8_t* fany, const int32_t* table, uint8_t* rstate, int64_t* meter_part,
                           const evc_tensor* out, int32_t act, float alpha, float* acc, int64_t acc_stride,
                           const evc_tensor* act_out, const evc_conv_sparsify* sp, const evc_conv_subpixel* sub,
                           int32_t dense, int32_t S, void* stream) {
  EVC_CHECK_ARG(g && cfg_in && in_hwc && wpack && S > 0 && fz::valid_bn(cfg_in->bn), "conv_fused: null argument");
  // The dense pass (full-magnitude values, not increments) always runs promoted (K-segments of one
  // K-block in row mode, two otherwise), so its accumulation chains stay as short as fp32 needs.
  evc_conv_cfg cfg_local = *cfg_in;
  if (dense && !cfg_local.thin && cfg_local.bn <= 128) cfg_local.drain = cfg_local.row == 1 ? 1 : 2;
  const evc_conv_cfg* cfg = &cfg_local;
  EVC_CHECK_ARG(evc_conv_fused_supported(g), "conv_fused: unsupported geometry");
  EVC_CHECK_ARG(cfg->row ? (g->stride == 1 && cfg->bn <= 128 && g->kw <= 9 &&
                            (cfg->row == 1 || (cfg->bn <= 32 && g->kw <= 3 && cfg->splits == 1)))
                         : (cfg->rh * cfg->rw == fz::BM && (cfg->rw == 32 || cfg->rw == 16 || cfg->rw == 8) &&
                            cfg->rw * g->stride <= 256 && cfg->rh * g->stride <= 256),
                "conv_fused: bad region shape");
  EVC_CHECK_ARG(cfg->splits >= 1 && cfg->splits <= 16, "conv_fused: splits must lie in [1, 16]");
  const int Hp = g->H + 2 * g->pad, Wp = g->W + 2 * g->pad;
  const int acp = cp < 0 ? -cp : cp;  // cp < 0: fp32 shadow, CUDA-core path only
  EVC_CHECK_ARG((cp > 0 || cfg->thin) && acp % (cfg->thin ? 4 : 32) == 0 && acp >= g->c_in && hwc_stride % 4 == 0 &&
                    hwc_stride >= (int64_t)Hp * Wp * hwc_px(cp),
                "conv_fused: shadow layout (cp % 32, thin path +-cp % 4; (H + 2 pad) x (W + 2 pad) pixels per session)");
  EVC_CHECK_ARG(act < 0 || (act <= 3 && act_out && (act_out->vals || sp) && (acc || dense)), "conv_fused: activation");
  EVC_CHECK_ARG(out || (act >= 0 && act_out->vals) || sp, "conv_fused: no output");
  EVC_CHECK_ARG(!sub || (sub->c_out > 0 && sub->c_out % 4 == 0 && g->c_out == 4 * sub->c_out && g->th % 2 == 0 &&
                         g->tw % 2 == 0 && g->kh == 3 &&
                         g->kw == 3 && g->stride == 1 && g->pad == 1 && sub->Ho == 2 * g->Ho && sub->Wo == 2 * g->Wo &&
                         !cfg->thin && sub->border && (dense || sub->fany_in)),
                "conv_fused_subpixel: needs a 3x3 stride-1 pad-1 geometry with 4 x c_out (c_out % 4 == 0), even tiles, "
                "composed channels, the border correction and the high-res any-channel map");
  EVC_CHECK_ARG(!sub || (cfg->bn >= 64 && cfg->row != 2),
                "conv_fused_subpixel: needs a channel block of >= 64 composed channels, not packed");
  const int eHo = sub ? sub->Ho : g->Ho, eWo = sub ? sub->Wo : g->Wo, oc = sub ? sub->c_out : g->c_out;
  EVC_CHECK_ARG(!sp || (sp->hwc && sp->cp % 4 == 0 && std::abs(sp->cp) >= oc && sp->hwc_stride % 4 == 0 &&
                        sp->pitch >= eWo && sp->flags && sp->fany && sp->partials),
                "conv_fused: fused sparsify needs the shadow, flags, fany and partials");
  EVC_CHECK_ARG(dense || (in && in->flags && fany && table && rstate && meter_part &&
                          ((act >= 0 ? act_out->flags : (out ? out->flags : nullptr)) != nullptr)),
                "conv_fused: incremental mode needs masks, fany, table, rstate and counters");
  const fz::Layout L = fz::layout_of(g, cfg);
  fz::EncodeTiled enc = fz::encoder();
  CUtensorMap map;
  CUresult r = CUDA_SUCCESS;
  if (cfg->thin) {
    // no tensor map: the CUDA-core path reads the shadow directly
  } else if (cfg->row) {  // (channels, flattened padded pixels, session)
    const cuuint64_t dims[3] = {(cuuint64_t)(2 * cp), (cuuint64_t)Hp * Wp, (cuuint64_t)S};
    const cuuint64_t strides[2] = {(cuuint64_t)cp * 8, (cuuint64_t)hwc_stride * 4};
    const cuuint32_t box[3] = {32, (cuuint32_t)(fz::BM + g->kw - 1), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(in_hwc), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {  // (channels, padded x, padded y, session), traversal stride = conv stride
    const cuuint64_t dims[4] = {(cuuint64_t)(2 * cp), (cuuint64_t)Wp, (cuuint64_t)Hp, (cuuint64_t)S};
    const cuuint64_t strides[3] = {(cuuint64_t)cp * 8, (cuuint64_t)Wp * cp * 8, (cuuint64_t)hwc_stride * 4};
    const cuuint32_t box[4] = {32, (cuuint32_t)(cfg->rw * g->stride), (cuuint32_t)(cfg->rh * g->stride), 1};
    const cuuint32_t estr[4] = {1, (cuuint32_t)g->stride, (cuuint32_t)g->stride, 1};
    r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(in_hwc), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    set_error("evc: conv_fused: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return EVC_ECUDA;
  }
  fz::Args a;
  memset(&a, 0, sizeof(a));
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.kh = g->kh;
  a.kw = g->kw;
  a.stride = g->stride;
  a.pad = g->pad;
  a.H = g->H;
  a.W = g->W;
  a.Ho = g->Ho;
  a.Wo = g->Wo;
  a.S = S;
  a.RH = cfg->rh;
  a.RW = cfg->rw;
  a.RHn = (g->Ho + cfg->rh - 1) / cfg->rh;
  a.RWn = (g->Wo + cfg->rw - 1) / cfg->rw;
  a.row = cfg->row;
  a.P = Wp;
  a.R = L.R;
  a.VM = L.VM;
  a.ns = L.ns;
  a.stage = L.stage;
  a.a_half = L.a_half;
  a.b_bytes = L.b_bytes;
  a.drain = cfg->bn <= 128 ? std::max(0, cfg->drain) : 0;
  a.cchunks = L.cchunks;
  a.nkb = L.nkb;
  a.splits = fz::split_count(a.nkb, cfg->splits);
  a.kb_per_split = (a.nkb + a.splits - 1) / a.splits;
  a.bn = cfg->bn;
  a.th = g->th;
  a.tw = g->tw;
  a.cp = cp;
  a.wpack = wpack;
  a.bias = bias;
  a.dense = dense != 0;
  a.trace = fz::g_trace;
  a.pf = std::getenv("EVC_ACC_PREFETCH") != nullptr ? 1 : 0;  // opt-in: measured neutral
  a.eHo = eHo;
  a.eWo = eWo;
  a.oc = oc;
  a.fany_side = fany;
  if (sub) {
    a.sub = 1;
    a.fany_side = sub->fany_in;
    a.border = sub->border;
  }
  if (!a.dense) {
    const TView vin = view_of(*in);
    a.fany = fany;
    a.in_f = vin.f;
    a.in_fs = vin.fs;
    a.tab = table;
    const evc_tensor* fo = act >= 0 ? act_out : out;
    a.oflags = fo->flags;
    a.ofs = fo->fstride;
    a.rstate = rstate;
    a.mpart = reinterpret_cast<long long*>(meter_part);
  }
  a.out = out ? out->vals : nullptr;
  a.ovs = out ? out->vstride : 0;
  a.act = act;
  a.alpha = alpha;
  a.acc = acc;
  a.accs = acc_stride;
  a.yact = act >= 0 ? act_out->vals : nullptr;
  a.yvs = act >= 0 ? act_out->vstride : 0;
  if (sp) {
    a.sp_hwc = sp->hwc;
    a.sp_hs = sp->hwc_stride;
    a.sp_cp = sp->cp;
    a.sp_pitch = sp->pitch;
    a.sp_GH = (eHo + g->th - 1) / g->th;
    a.sp_GW = (eWo + g->tw - 1) / g->tw;
    a.sp_flags = sp->flags;
    a.sp_fs = sp->fstride;
    a.sp_fany = sp->fany;
    a.sp_part = sp->partials;
  }
  cudaStream_t st = as_stream(stream);
  cudaError_t e;
  if (cfg->thin) {
    EVC_CHECK_ARG(g->c_out <= 32 && L.stage <= 48 * 1024, "conv_fused: thin path needs C_out <= 32, small weights");
    a.splits = 1;
    const dim3 tg((unsigned)(S * L.R)), tb(fz::THIN_THREADS);
    const bool f32 = cp < 0;
    switch (fz::thin_co(g->c_out)) {
      case 2: e = launch_pdl((f32 ? fz::k_conv_thin<2, true> : fz::k_conv_thin<2, false>), tg, tb, (size_t)L.stage, st, in_hwc, hwc_stride, a); break;
      case 4: e = launch_pdl((f32 ? fz::k_conv_thin<4, true> : fz::k_conv_thin<4, false>), tg, tb, (size_t)L.stage, st, in_hwc, hwc_stride, a); break;
      case 8: e = launch_pdl((f32 ? fz::k_conv_thin<8, true> : fz::k_conv_thin<8, false>), tg, tb, (size_t)L.stage, st, in_hwc, hwc_stride, a); break;
      case 16: e = launch_pdl((f32 ? fz::k_conv_thin<16, true> : fz::k_conv_thin<16, false>), tg, tb, (size_t)L.stage, st, in_hwc, hwc_stride, a); break;
      default: e = launch_pdl((f32 ? fz::k_conv_thin<32, true> : fz::k_conv_thin<32, false>), tg, tb, (size_t)L.stage, st, in_hwc, hwc_stride, a); break;
    }
    if (e != cudaSuccess) {
      set_error(std::string("evc: conv_fused (thin) launch: ") + cudaGetErrorString(e));
      return EVC_ECUDA;
    }
    EVC_LAUNCH_CHECK("conv_fused_thin");
    return EVC_OK;
  }
  // BN = 128 (tap mode), opt-in (EVC_PERSIST128=1): persistent with the split-small TMEM layout, the next
  // item's mainloop overlapping the previous item's epilogue.  Measured slower at 32 streams (enc2 93 vs
  // 75 us, dec0 384 vs 313 us: these layers are bound by L2 operand traffic, ~8.7 TB/s for dec0, not
  // by the epilogue), so the one-shot kernel stays the default
  const bool p128 = cfg->bn == 128 && !cfg->row && (int64_t)S * L.R * ((g->c_out + 127) / 128) > 148 &&
                    std::getenv("EVC_PERSIST128") != nullptr;
  if (a.splits == 1 && (cfg->bn <= 64 || p128) && std::getenv("EVC_NO_PERSIST") == nullptr) {
    // persistent CTAs: one or two per SM (BN = 16 fits two), each walking work items
    const int occ = (cfg->bn <= 16 && 2 * ((int)L.ns * L.stage + 1024 + 256 + 2048) <= fz::SMEM_MAX) ? 2 : 1;
    const int items = S * L.R * ((g->c_out + cfg->bn - 1) / cfg->bn);
    const int grid = std::max(1, std::min(items, occ * 148));
    switch (cfg->bn) {
      case 16: e = fz::launch_persist<16>(map, a, grid, st); break;
      case 32: e = fz::launch_persist<32>(map, a, grid, st); break;
      case 128: e = fz::launch_persist<128>(map, a, grid, st); break;
      default: e = fz::launch_persist<64>(map, a, grid, st); break;
    }
    if (e != cudaSuccess) {
      set_error(std::string("evc: conv_fused (persistent) launch: ") + cudaGetErrorString(e));
      return EVC_ECUDA;
    }
    EVC_LAUNCH_CHECK("conv_fused_persist");
    return EVC_OK;
  }
  switch (cfg->bn) {
    case 16: e = fz::launch<16>(map, a, st); break;
    case 32: e = fz::launch<32>(map, a, st); break;
    case 64: e = fz::launch<64>(map, a, st); break;
    case 128: e = fz::launch<128>(map, a, st); break;
    default: e = fz::launch<256>(map, a, st); break;
  }
  if (e != cudaSuccess) {
    set_error(std::string("evc: conv_fused launch: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  EVC_LAUNCH_CHECK("conv_fused");
  return EVC_OK;
}

int evc_conv_fused(const evc_conv_geom* g, const evc_conv_cfg* cfg, const float* in_hwc, int32_t cp,
                   int64_t hwc_stride, const float* wpack, const float* bias, const evc_tensor* in,
                   const uint8_t* fany, const int32_t* table, uint8_t* rstate, int64_t* meter_part,
                   const evc_tensor* out, int32_t act, float alpha, float* acc, int64_t acc_stride,
                   const evc_tensor* act_out, const evc_conv_sparsify* sp, int32_t dense, int32_t S,
                   void* stream) {
  return conv_fused_impl(g, cfg, in_hwc, cp, hwc_stride, wpack, bias, in, fany, table, rstate, meter_part, out, act,
                         alpha, acc, acc_stride, act_out, sp, nullptr, dense, S, stream);
}

int evc_conv_fused_subpixel(const evc_conv_geom* g, const evc_conv_cfg* cfg, const float* in_hwc, int32_t cp,
                            int64_t hwc_stride, const float* wpack, const float* bias, const evc_tensor* in,
                            const uint8_t* fany, const int32_t* table, uint8_t* rstate, int64_t* meter_part,
                            const evc_tensor* out, int32_t act, float alpha, float* acc, int64_t acc_stride,
                            const evc_tensor* act_out, const evc_conv_sparsify* sp, const evc_conv_subpixel* sub,
                            int32_t dense, int32_t S, void* stream) {
  EVC_CHECK_ARG(sub, "conv_fused_subpixel: null sub-pixel descriptor");
  return conv_fused_impl(g, cfg, in_hwc, cp, hwc_stride, wpack, bias, in, fany, table, rstate, meter_part, out, act,
                         alpha, acc, acc_stride, act_out, sp, sub, dense, S, stream);
}

int evc_conv_trace(void* buf) {
  fz::g_trace = reinterpret_cast<unsigned long long*>(buf);
  return EVC_OK;
}

int evc_tile_any(const evc_tensor* x, uint8_t* fany, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && x->flags && fany && S > 0, "tile_any: null argument");
  TView v = view_of(*x);
  const int Ti = v.GH * v.GW;
  launch_pdl(fz::k_tile_any, dim3(dim3(cdiv(Ti, 128), S)), dim3(128), 0, as_stream(stream), v, fany);
  EVC_LAUNCH_CHECK("tile_any");
  return EVC_OK;
}

int evc_meter_step(const evc_meter_node* nodes, int32_t n, int32_t S, int32_t* in_true, int64_t* perf_step,
                   int64_t* perf_cum, double* ff_last, double* ff_sum, const evc_sp_node* sp_nodes, int32_t n_sp,
                   void* stream) {
  EVC_CHECK_ARG(nodes && n > 0 && S > 0 && in_true && perf_step && perf_cum && ff_last && ff_sum && n_sp >= 0 &&
                    (n_sp == 0 || sp_nodes),
                "meter_step: null argument");
  launch_pdl(fz::k_meter_step, dim3((unsigned)(n * S + n_sp * S)), dim3(256), 0, as_stream(stream), nodes, n, S, in_true,
             reinterpret_cast<long long*>(perf_step), reinterpret_cast<long long*>(perf_cum), ff_last, ff_sum,
             sp_nodes);
  EVC_LAUNCH_CHECK("meter_step");
  return EVC_OK;
}

}  // extern "C"
