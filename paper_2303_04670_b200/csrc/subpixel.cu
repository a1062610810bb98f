// Sub-pixel form of the decoder pattern "2x bilinear upsample -> sparsify(t_p = 0) -> 3x3 conv"
// (increment_ops.py:271-285, sparsify.py:54-78, increment_ops.py:126-194).
//
// A 3x3 stride-1 pad-1 conv of a 2x bilinear upsample U(x) is, per output phase (a, b) -- output
// site (2i + a, 2j + b) -- a 3x3 conv of the LOW-RES input x with composed weights
//   W'_ab[dy][dx] = sum_{kh, kw} C_a[dy][kh] C_b[dx][kw] W[kh][kw]
// (C_0 / C_1: the half-pixel bilinear taps 1/4, 3/4), evaluated here as ONE conv with 4 x C_out
// output channels on x padded by replicating its edge (the upsample clamps its source index, so
// the replicated ring reproduces U on every high-res row / column, including the first and last).
// Only the high-res conv's own zero padding differs: the composed conv sees U(clamp(p)) where the
// reference sees 0, on the taps that leave the high-res image -- evc_subpixel_border computes that
// difference for the four border lines and the conv epilogue adds it.  The conv then reads the
// low-res input (4x fewer shadow bytes than the upsampled one) and never materialises U.
//
//  k_subpix_prep:   the low-res hi/lo shadow (interior + replicated ring) and the low-res any-channel
//                   tile map (region liveness of the composed conv; OR-accumulated), one pass over x
//  k_subpix_border: border correction [S][2 (Ho + Wo)][C_out] = - sum over the off-image taps of
//                   W . U(clamped site), U evaluated with dense_upsample's float32 op order

#include <algorithm>

#include "common.cuh"

namespace evc {

constexpr int SP_THREADS = 256, SP_MAXC = 32;

// CTA = (session, low-res tile row, column block of CW = tw * floor(32 / tw) columns x one 32-channel
// chunk).  Thread (channel, row) reads its row run of the channel-planar input (all loads in flight),
// the CTA then writes 256-byte [32 heads | 32 tails] runs per pixel (lane = channel): both sides
// coalesced.  fany (zeroed per step) is OR-accumulated per tile (benign race: every writer stores 1).
__global__ void __launch_bounds__(SP_THREADS) k_subpix_prep(TView x, float* __restrict__ hwc, int64_t hs, int cp,
                                                             int pitch, uint8_t* __restrict__ fany, int CW, int nJB) {
  pdl_wait();
  pdl_trigger();
  __shared__ float t[SP_MAXC][8 * 33 + 1];  // [channel][row * 33 + col] (odd channel stride)
  __shared__ int s_any[8];
  const int s = blockIdx.z, ti = blockIdx.y, jb = blockIdx.x % nJB, k0 = (blockIdx.x / nJB) * 32;
  const int r0 = ti * x.th, nrow = min(x.th, x.H - r0);
  const int c0 = jb * CW, ncol = min(CW, x.W - c0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ntile = (ncol + x.tw - 1) / x.tw;
  if (threadIdx.x < 8) s_any[threadIdx.x] = 0;
  __syncthreads();
  {  // thread (channel ch, row) loads columns 0..ncol-1 of its row: independent loads, one wait
    const int ch = threadIdx.x >> 3, row = threadIdx.x & 7, c = k0 + ch;
    const bool ok = row < nrow && c < x.C;
    const float* src = ok ? x.plane(s, c) + (int64_t)(r0 + row) * x.W + c0 : nullptr;
    float v[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) v[q] = (ok && q < ncol) ? __ldg(src + q) : 0.0f;
    if (row < 8) {
      uint32_t nz = 0;
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        t[ch][row * 33 + q] = v[q];
        nz |= __float_as_uint(v[q]) & 0x7fffffffu;
      }
      if (ok && nz) {  // per tile of the row
        for (int tj = 0; tj < ntile; ++tj) {
          uint32_t z = 0;
          for (int q = tj * x.tw; q < min(ncol, (tj + 1) * x.tw); ++q) z |= __float_as_uint(t[ch][row * 33 + q]) & 0x7fffffffu;
          if (z) s_any[tj] = 1;
        }
      }
    }
  }
  __syncthreads();
  if (fany && threadIdx.x < ntile && s_any[threadIdx.x]) fany[((int64_t)s * x.GH + ti) * x.GW + c0 / x.tw + threadIdx.x] = 1;
  // output pixel rows / columns incl. the replicated ring at the image edges
  const int ra = r0 - (ti == 0 ? 1 : 0), rb = r0 + nrow + (r0 + nrow == x.H ? 1 : 0);
  const int ca = c0 - (c0 == 0 ? 1 : 0), cb = c0 + ncol + (c0 + ncol == x.W ? 1 : 0);
  const int nr = rb - ra, nc = cb - ca;
  float* base = hwc + (int64_t)s * hs + 2 * k0 + lane;
  for (int p = warp; p < nr * nc; p += SP_THREADS / 32) {  // warp per pixel, lane = channel
    const int pr = ra + p / nc, pc = ca + p % nc;
    const int sr = min(max(pr, 0), x.H - 1) - r0, sc = min(max(pc, 0), x.W - 1) - c0;
    const float v = t[lane][sr * 33 + sc];
    const float h = tf32_head(v);
    float* d = base + ((int64_t)pr * pitch + pc) * (2 * cp);
    d[0] = h;
    d[32] = __fsub_rn(v, h);
  }
}

// U(y, x) of the 2x bilinear upsample of plane xv (H x W low-res), dense_upsample's op order.
__device__ __forceinline__ float up2(const float* xv, int H, int W, int y, int x) {
  return upsample_at(xv, H, W, y, x, 2, 1);
}

// Border correction, a small GEMM per (session, line): out[pos][o] = - sum_{c, k} Wl[o][c][k] U[c][pos - 1 + k]
// over the 3 taps that leave the image across the line (Wl = W[:, :, 0 or 2, :] on a row line, W[:, :, :,
// 0 or 2] on a column line), plus, at the two ends of a row line (the corners), the taps that leave
// through the column with in-image rows.  Line 0 / 1 = output row 0 / Ho - 1 (index X), line 2 / 3 =
// output column 0 / Wo - 1 (index Y).  CTA = (32 positions, 32 output channels) of one line of one
// session; 256 threads = 32 positions x 8 groups of 4 channels; the channel (K) loop stages 32 input
// channels at a time: U of the 34 line positions + the 2 corner sites, and the weights [c][tap][o]
// (float4 per thread; w is laid out [C][9][c_out] so the staging reads are coalesced).  Fixed
// summation order: deterministic.
constexpr int SB_C = 32;

__global__ void __launch_bounds__(SP_THREADS) k_subpix_border(TView x, const float* __restrict__ w, int co,
                                                               float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ float sU[SB_C][36];               // [c][34 line positions | 2 corner sites]
  __shared__ __align__(16) float sW[SB_C][9][32];  // [c][tap][o]
  const int s = blockIdx.z, L = blockIdx.y % 4, oc0 = (blockIdx.y / 4) * 32, p0 = blockIdx.x * 32;
  const int Ho = 2 * x.H, Wo = 2 * x.W, C = x.C;
  const bool rowline = L < 2;
  const int len = rowline ? Wo : Ho;
  if (p0 >= len) return;
  const int fixed = L == 0 ? 0 : (L == 1 ? Ho - 1 : (L == 2 ? 0 : Wo - 1));
  const int other = L == 0 ? 1 : Ho - 2;  // row lines: the corner column's other in-image row
  const int kout = (L == 0 || L == 2) ? 0 : 2;
  const int pl = threadIdx.x & 31, og = threadIdx.x >> 5, pos = p0 + pl;
  const int no = min(32, co - oc0);
  const bool corner = rowline && (pos == 0 || pos == Wo - 1);
  float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  for (int c0 = 0; c0 < C; c0 += SB_C) {
    const int nc = min(SB_C, C - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < SB_C * 36; e += SP_THREADS) {
      const int c = e / 36, q = e % 36;
      float v = 0.0f;
      if (c < nc) {
        const float* xv = x.plane(s, c0 + c);
        if (q < 34) {
          const int pp = min(max(p0 - 1 + q, 0), len - 1);
          v = rowline ? up2(xv, x.H, x.W, fixed, pp) : up2(xv, x.H, x.W, pp, fixed);
        } else if (rowline && Ho > 1) {
          v = up2(xv, x.H, x.W, other, q == 34 ? 0 : Wo - 1);
        }
      }
      sU[c][q] = v;
    }
    for (int e = threadIdx.x; e < SB_C * 9 * 32; e += SP_THREADS) {
      const int o = e & 31, rest = e >> 5, tap = rest % 9, c = rest / 9;
      sW[c][tap][o] = (c < nc && o < no) ? w[((int64_t)(c0 + c) * 9 + tap) * co + oc0 + o] : 0.0f;
    }
    __syncthreads();
    if (pos < len && 4 * og < no) {
      for (int c = 0; c < nc; ++c) {
        const float u0 = sU[c][pl], u1 = sU[c][pl + 1], u2 = sU[c][pl + 2];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const float uk = k == 0 ? u0 : (k == 1 ? u1 : u2);
          const int tap = rowline ? kout * 3 + k : k * 3 + kout;
          const float4 wv = *reinterpret_cast<const float4*>(&sW[c][tap][4 * og]);
          acc[0] = __fmaf_rn(wv.x, uk, acc[0]);
          acc[1] = __fmaf_rn(wv.y, uk, acc[1]);
          acc[2] = __fmaf_rn(wv.z, uk, acc[2]);
          acc[3] = __fmaf_rn(wv.w, uk, acc[3]);
        }
        if (corner) {  // taps (kh, kc) leaving through the column: rows fixed (line value) and `other`
          const int kc = pos == 0 ? 0 : 2;
#pragma unroll
          for (int kh = 0; kh < 3; ++kh) {
            const int yy = fixed + kh - 1;
            if (yy < 0 || yy >= Ho) continue;  // (counted on the row line)
            const float uk = yy == fixed ? sU[c][pl + 1] : sU[c][pos == 0 ? 34 : 35];
            const float4 wv = *reinterpret_cast<const float4*>(&sW[c][kh * 3 + kc][4 * og]);
            acc[0] = __fmaf_rn(wv.x, uk, acc[0]);
            acc[1] = __fmaf_rn(wv.y, uk, acc[1]);
            acc[2] = __fmaf_rn(wv.z, uk, acc[2]);
            acc[3] = __fmaf_rn(wv.w, uk, acc[3]);
          }
        }
      }
    }
  }
  if (pos < len) {
    const int li = L == 0 ? pos : (L == 1 ? Wo + pos : (L == 2 ? 2 * Wo + pos : 2 * Wo + Ho + pos));
    float* o = out + ((int64_t)s * 2 * (Ho + Wo) + li) * co + oc0 + 4 * og;
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (4 * og + j < no) o[j] = -acc[j];
  }
}

int init_subpixel() { return EVC_OK; }

}  // namespace evc

using namespace evc;

extern "C" {

int evc_subpixel_prep(const evc_tensor* x, float* hwc, int32_t cp, int64_t hwc_stride, int32_t pitch, uint8_t* fany,
                      int32_t S, void* stream) {
  EVC_CHECK_ARG(x && hwc && S > 0, "subpixel_prep: null argument");
  EVC_CHECK_ARG(cp >= x->C && cp % 32 == 0 && pitch >= x->W + 2 && x->th <= 8 && x->tw <= 32,
                "subpixel_prep: shadow channels (multiple of 32 >= C), pitch >= W + 2, tiles <= 8 x 32");
  const TView v = view_of(*x);
  const int CW = v.tw * (32 / v.tw), nJB = (v.W + CW - 1) / CW;
  const dim3 grid((unsigned)(nJB * (cp / 32)), (unsigned)v.GH, (unsigned)S);
  launch_pdl(k_subpix_prep, grid, dim3(SP_THREADS), 0, as_stream(stream), v, hwc, hwc_stride, (int)cp, (int)pitch,
             fany, CW, nJB);
  EVC_LAUNCH_CHECK("subpixel_prep");
  return EVC_OK;
}

int evc_subpixel_border(const evc_tensor* x, const float* w, int32_t c_out, float* out, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && w && out && c_out > 0 && c_out % 4 == 0 && S > 0, "subpixel_border: null argument");
  const TView v = view_of(*x);
  const int len = 2 * std::max(v.H, v.W);
  const dim3 grid((unsigned)((len + 31) / 32), (unsigned)(4 * ((c_out + 31) / 32)), (unsigned)S);
  launch_pdl(k_subpix_border, grid, dim3(SP_THREADS), 0, as_stream(stream), v, w, (int)c_out, out);
  EVC_LAUNCH_CHECK("subpixel_border");
  return EVC_OK;
}

}  // extern "C"
