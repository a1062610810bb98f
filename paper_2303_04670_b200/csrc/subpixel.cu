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
//  k_subpix_input:  one pass over x: the low-res hi/lo shadow (interior + replicated ring), the
//                   low-res tile map (region liveness of the composed conv), and the sparsify's
//                   high-res flags / any-map / norm partials from the (unstored) upsample
//  k_subpix_border: border correction [S][2 (Ho + Wo)][C_out] = - sum over the off-image taps of
//                   W . U(clamped site), U evaluated with dense_upsample's float32 op order

#include <algorithm>

#include "common.cuh"

namespace evc {

constexpr int SP_THREADS = 256;
constexpr int SI_CH = 40;  // channels per input-pass CTA: a chunk of 32, the last one takes a remainder <= 8

// Half-pixel 2x bilinear tap of output index o (tensors.py:259-266 for factor 2, the values
// bilinear_tap computes, in closed form): o = 2i -> (i - 1, i) with (1/4, 3/4), o = 2i + 1 -> (i, i + 1)
// with (3/4, 1/4), indices clamped to [0, n).
__device__ __forceinline__ Tap tap2(int o, int n) {
  Tap t;
  const int i = o >> 1;
  if (o & 1) {
    t.i0 = min(i, n - 1);
    t.i1 = min(i + 1, n - 1);
    t.w0 = 0.75f;
    t.w1 = 0.25f;
  } else {
    t.i0 = max(i - 1, 0);
    t.i1 = min(i, n - 1);
    t.w0 = 0.25f;
    t.w1 = 0.75f;
  }
  return t;
}

// U(y, x) of the 2x bilinear upsample of plane xv (H x W low-res), dense_upsample's op order.
__device__ __forceinline__ float up2(const float* xv, int H, int W, int y, int x) {
  const Tap tr = tap2(y, H), tc = tap2(x, W);
  const float* x0 = xv + (int64_t)tr.i0 * W;
  const float* x1 = xv + (int64_t)tr.i1 * W;
  const float ra = __fadd_rn(__fmul_rn(x0[tc.i0], tr.w0), __fmul_rn(x1[tc.i0], tr.w1));
  const float rb = __fadd_rn(__fmul_rn(x0[tc.i1], tr.w0), __fmul_rn(x1[tc.i1], tr.w1));
  return __fadd_rn(__fmul_rn(ra, tc.w0), __fmul_rn(rb, tc.w1));
}

// The sub-pixel conv's input pass (replaces upsample_sparsify's t_p = 0 fast path for that conv plus
// a low-res shadow copy): per CTA = (session, low-res tile row, CW low-res columns, 32 channels) --
// i.e. the high-res tiles 2 ti, 2 ti + 1 x (2 CW / tw) tile columns it owns (th, tw even):
//  * the low-res hi/lo shadow of its pixels (+ the replicated ring at the image edges),
//  * the low-res tile map (any channel flag; OR, zeroed per step) for the composed conv's regions,
//  * the sparsify output's flags of every owned high-res (channel, tile), recomputed from the values
//    of the upsample (sparsify.py:77-78), the high-res any-channel map (OR) and the sum of squares of
//    the owned values (norm partial, one per CTA, folded later by evc_meter_step).
// The footprint (rows r0 - 1 .. r0 + th, columns c0 - 1 .. c0 + CW, edge-clamped) is staged once in
// shared memory by coalesced row loads; the upsample runs lane = high-res column (taps per lane
// hoisted), channel loops over the CTA's real channels only, skipping channels without a flagged
// low-res tile in the support (their values are exact zeros).
constexpr int SI_R = 10, SI_C = 34;  // footprint rows (th + 2 <= 10) and columns (CW + 2 <= 34)

__device__ __forceinline__ void subpix_input_body(const TView& x, uint8_t* __restrict__ yf, int64_t yfs, int GHy,
                                                  int GWy, double* __restrict__ part, float* __restrict__ hwc,
                                                  int64_t hs, int cp, int pitch, uint8_t* __restrict__ fany_lo,
                                                  uint8_t* __restrict__ fany_hi, int CW, int nJB, int bx, int nx,
                                                  float* si_dyn) {
  float(*t)[SI_R * SI_C + 1] = reinterpret_cast<float(*)[SI_R * SI_C + 1]>(si_dyn);
  __shared__ double s_w[SP_THREADS / 32];
  __shared__ uint8_t s_fy[SI_CH][2][16];  // high-res flags of the owned tiles
  __shared__ int s_live[SI_CH];           // channel has a flagged low-res tile in the support box
  const int s = blockIdx.z, ti = blockIdx.y, jb = bx % nJB, k0 = (bx / nJB) * 32;
  const int r0 = ti * x.th, nrow = min(x.th, x.H - r0);
  const int c0 = jb * CW, ncol = min(CW, x.W - c0);
  // real channels of the chunk: 32, the last chunk also the remainder (<= 8) of C past a multiple of 32
  const int nch = (x.C - k0 <= SI_CH) ? x.C - k0 : 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int jt0 = c0 / x.tw, ntl = (ncol + x.tw - 1) / x.tw;
  const int Hy = 2 * x.H;
  const int T0r = 2 * ti, T0c = 2 * c0 / x.tw, ntc = (2 * ncol + x.tw - 1) / x.tw;
  if (threadIdx.x < SI_CH) s_live[threadIdx.x] = 0;
  for (int e = threadIdx.x; e < SI_CH * 2 * 16; e += SP_THREADS) (&s_fy[0][0][0])[e] = 0;
  __syncthreads();
  // 1) footprint rows (coalesced: lane = column), support flags, low-res tile map
  {
    const int q0 = min(max(c0 - 1 + lane, 0), x.W - 1), q1 = min(max(c0 + 31 + lane, 0), x.W - 1);
    const bool has1 = lane + 32 < ncol + 2, has0 = lane < ncol + 2;
    for (int ch = warp; ch < nch; ch += SP_THREADS / 32) {  // every row's loads in flight, then the stores
      const float* pl = x.plane(s, k0 + ch);
      float* dst = t[ch];
      float v0[SI_R], v1[SI_R];
#pragma unroll
      for (int fr = 0; fr < SI_R; ++fr) {
        const float* src = pl + (int64_t)min(max(r0 - 1 + fr, 0), x.H - 1) * x.W;
        const bool rok = fr < nrow + 2;
        v0[fr] = (rok && has0) ? __ldg(src + q0) : 0.0f;
        v1[fr] = (rok && has1) ? __ldg(src + q1) : 0.0f;
      }
#pragma unroll
      for (int fr = 0; fr < SI_R; ++fr) {
        dst[fr * SI_C + lane] = v0[fr];
        if (lane + 32 < SI_C) dst[fr * SI_C + lane + 32] = v1[fr];
      }
    }
  }
  for (int e = threadIdx.x; e < nch * 4 * 8; e += SP_THREADS) {
    const int ch = e >> 5, rr = (e >> 3) & 3, cc = e & 7;
    if (rr == 3) continue;
    const int a = ti - 1 + rr, b = jt0 - 1 + cc;
    if (a >= 0 && a < x.GH && b >= 0 && b < x.GW && cc < ntl + 2 && x.fplane(s, k0 + ch)[a * x.GW + b]) {
      s_live[ch] = 1;  // (benign: all store 1)
      if (rr == 1 && cc >= 1 && cc <= ntl && fany_lo) fany_lo[((int64_t)s * x.GH + ti) * x.GW + b] = 1;
    }
  }
  __syncthreads();
  // 2) low-res shadow: owned pixels + the ring, lane = channel (256-byte [heads | tails] runs)
  {
    const int ra = r0 - (ti == 0 ? 1 : 0), rb = r0 + nrow + (r0 + nrow == x.H ? 1 : 0);
    const int ca = c0 - (c0 == 0 ? 1 : 0), cb = c0 + ncol + (c0 + ncol == x.W ? 1 : 0);
    for (int cl = lane; cl < nch; cl += 32) {  // (a second pass for the remainder channels)
      float* base = hwc + (int64_t)s * hs + 2 * ((k0 + cl) & ~31) + ((k0 + cl) & 31);  // hwc_head layout
      for (int pr = ra + warp; pr < rb; pr += SP_THREADS / 32) {
        const float* tr = &t[cl][(min(max(pr, 0), x.H - 1) - r0 + 1) * SI_C - c0 + 1];
        float* d = base + (int64_t)pr * pitch * (2 * cp);
        for (int pc = ca; pc < cb; ++pc) {
          const float v = tr[min(max(pc, 0), x.W - 1)];
          const float h = tf32_head(v);
          d[pc * (2 * cp)] = h;
          d[pc * (2 * cp) + 32] = __fsub_rn(v, h);
        }
      }
    }
  }
  // 3) the upsample of the owned high-res block: rows 2 r0 .. 2 (r0 + nrow) - 1; lane = footprint
  //    column q (low-res column j = c0 - 1 + q): the row interpolation r(j) once per lane, the
  //    neighbours' by shuffles, then the two output columns 2j (taps j - 1, j: 1/4, 3/4) and 2j + 1
  //    (taps j, j + 1: 3/4, 1/4) -- dense_upsample's op order (rows, then columns), bit-exact
  float ss = 0.0f;
  const int Ya = 2 * r0, Yb = min(Hy, 2 * (r0 + nrow));
  const bool own = lane >= 1 && lane <= ncol;  // j = c0 + lane - 1 is an owned column
  const int tje = own ? (2 * (lane - 1)) / x.tw : 0, tjo = own ? (2 * (lane - 1) + 1) / x.tw : 0;
  // The footprint row fr holds x[clamp(r0 - 1 + fr)], so the clamped taps of tap2(Y) are footprint rows
  // k / 2 + {0, 1} (Y = 2 r0 + k even: 1/4, 3/4) and k / 2 + {1, 2} (odd: 3/4, 1/4): the column is read
  // into registers once per channel and the row loop is unrolled over compile-time indices.
  const int nk = Yb - Ya;  // 2 nrow <= 2 (SI_R - 2)
  for (int ch = warp; ch < nch; ch += SP_THREADS / 32) {
    if (!s_live[ch]) continue;  // no flagged support: every value is an exact zero (flags stay 0)
    const float* tc = t[ch] + min(lane, SI_C - 1);
    float col[SI_R];
#pragma unroll
    for (int fr = 0; fr < SI_R; ++fr) col[fr] = tc[fr * SI_C];
    uint32_t n00 = 0u, n01 = 0u, n10 = 0u, n11 = 0u;  // [tile row][even, odd column]: OR of magnitude bits
#pragma unroll
    for (int k = 0; k < 2 * (SI_R - 2); ++k) {
      if (k >= nk) break;
      const float r = (k & 1) ? __fadd_rn(__fmul_rn(col[k / 2 + 1], 0.75f), __fmul_rn(col[k / 2 + 2], 0.25f))
                              : __fadd_rn(__fmul_rn(col[k / 2], 0.25f), __fmul_rn(col[k / 2 + 1], 0.75f));
      const float rl = __shfl_up_sync(0xffffffffu, r, 1), rr = __shfl_down_sync(0xffffffffu, r, 1);
      // (the sparsify's "0 + y" only turns -0 into +0: neither the squares nor the magnitude bits see it)
      const float oe = __fadd_rn(__fmul_rn(rl, 0.25f), __fmul_rn(r, 0.75f));
      const float oo = __fadd_rn(__fmul_rn(r, 0.75f), __fmul_rn(rr, 0.25f));
      if (own) {
        ss = __fmaf_rn(oe, oe, ss);
        ss = __fmaf_rn(oo, oo, ss);
        const uint32_t be = __float_as_uint(oe), bo = __float_as_uint(oo);  // sign bits masked once below
        if (k >= x.th) {  // (two tile rows)
          n10 |= be;
          n11 |= bo;
        } else {
          n00 |= be;
          n01 |= bo;
        }
      }
    }
    n00 &= 0x7fffffffu;
    n01 &= 0x7fffffffu;
    n10 &= 0x7fffffffu;
    n11 &= 0x7fffffffu;
    if (n00) s_fy[ch][0][tje] = 1;  // (benign: all store 1)
    if (n01) s_fy[ch][0][tjo] = 1;
    if (n10) s_fy[ch][1][tje] = 1;
    if (n11) s_fy[ch][1][tjo] = 1;
  }
  const double w = (double)warp_sum(ss);
  if (lane == 0) s_w[warp] = w;
  __syncthreads();
  // 4) flags of every owned (channel, tile) -- written, not accumulated --, the any-map, the partial
  for (int e = threadIdx.x; e < nch * 2 * 16; e += SP_THREADS) {
    const int ch = e >> 5, r = (e >> 4) & 1, q = e & 15, Tr = T0r + r, Tc = T0c + q;
    if (q < ntc && Tr < GHy && Tc < GWy) yf[(int64_t)s * yfs + ((int64_t)(k0 + ch) * GHy + Tr) * GWy + Tc] = s_fy[ch][r][q];
  }
  if (threadIdx.x < 32 && fany_hi) {
    const int r = threadIdx.x / 16, q = threadIdx.x % 16, Tr = T0r + r, Tc = T0c + q;
    int any = 0;
    for (int ch = 0; ch < nch; ++ch) any |= s_fy[ch][r][q];
    if (q < ntc && Tr < GHy && Tc < GWy && any) fany_hi[((int64_t)s * GHy + Tr) * GWy + Tc] = 1;
  }
  if (threadIdx.x == 0) {
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < SP_THREADS / 32; ++k) tot += s_w[k];
    part[(int64_t)s * nx * gridDim.y + blockIdx.y * nx + bx] = tot;
  }
}

__global__ void __launch_bounds__(SP_THREADS) k_subpix_input(TView x, uint8_t* __restrict__ yf, int64_t yfs,
                                                              int GHy, int GWy, double* __restrict__ part,
                                                              float* __restrict__ hwc, int64_t hs, int cp, int pitch,
                                                              uint8_t* __restrict__ fany_lo,
                                                              uint8_t* __restrict__ fany_hi, int CW, int nJB) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float si_dyn[];  // [channel][row * SI_C + col] (odd channel stride)
  subpix_input_body(x, yf, yfs, GHy, GWy, part, hwc, hs, cp, pitch, fany_lo, fany_hi, CW, nJB, (int)blockIdx.x,
                    (int)gridDim.x, si_dyn);
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
constexpr int SB_C = 32, SB_SPB = 1;  // channels per K step, sessions per CTA (1: measured fastest)
constexpr int SB_WL = 20;             // low-res window along a line: 34 positions -> <= 19 columns

static_assert(SB_SPB == 1, "the split-channel reduction below assumes one session per CTA");
constexpr int SB_RED = 4 * 32 * 4;  // split mode: the second channel half's partial sums [og][pos][4]
constexpr int SB_SMEM_FLOATS = SB_C * 3 * 32 + SB_C * 2 * 3 * 32 + SB_C * 36 + SB_C * 2 * SB_WL + SB_RED;

// one CTA of the border GEMM: (bx = 32 positions, by = line + 32 output channels, bz = session group);
// shared memory carved from `sm` (16-byte aligned, SB_SMEM_FLOATS floats)
__device__ __forceinline__ void subpix_border_body(const TView& x, const float* __restrict__ w, int co, int S,
                                                   float* __restrict__ out, int bx, int by, int bz, float* sm) {
  float(*sW)[3][32] = reinterpret_cast<float(*)[3][32]>(sm);                       // [c][k][o]: the line's three off-image taps
  float(*sWc)[2][3][32] = reinterpret_cast<float(*)[2][3][32]>(sm + SB_C * 3 * 32);  // corners: [c][kc = 0 | 2][kh][o]
  float(*sU)[36] = reinterpret_cast<float(*)[36]>(sm + SB_C * 9 * 32);             // [c][34 line positions | 2 corners]
  float(*sL)[2][SB_WL] = reinterpret_cast<float(*)[2][SB_WL]>(sm + SB_C * 9 * 32 + SB_C * 36);  // [c][across][along]
  const int s0 = bz * SB_SPB, L = by % 4, oc0 = (by / 4) * 32, p0 = bx * 32;
  const int Ho = 2 * x.H, Wo = 2 * x.W, C = x.C;
  const bool rowline = L < 2;
  const int len = rowline ? Wo : Ho;
  if (p0 >= len) return;
  const int fixed = L == 0 ? 0 : (L == 1 ? Ho - 1 : (L == 2 ? 0 : Wo - 1));
  const int other = L == 0 ? 1 : Ho - 2;  // row lines: the corner column's other in-image row
  const int kout = (L == 0 || L == 2) ? 0 : 2;
  const int pl = threadIdx.x & 31, pos = p0 + pl;
  // C_out <= 16 (one 16-channel group): warps 4-7 would idle in the FMA loop, so the warps split the input
  // channels of every K step in two halves instead (fixed order: half 0's sum + half 1's sum)
  const bool split = co - (by / 4) * 32 <= 16;
  const int og = split ? (threadIdx.x >> 5) & 3 : threadIdx.x >> 5, hf = split ? (int)(threadIdx.x >> 7) : 0;
  const int no = min(32, co - oc0), nss = min(SB_SPB, S - s0);
  const bool corner = rowline && (pos == 0 || pos == Wo - 1);
  // the two low-res lines across the line (taps of the fixed coordinate) and the window along it
  const Tap tx = tap2(fixed, rowline ? x.H : x.W);
  const int ac0 = tx.i0, ac1 = tx.i1;
  const int wlo = tap2(max(p0 - 1, 0), rowline ? x.W : x.H).i0;
  float acc[SB_SPB][4] = {};
  for (int c0 = 0; c0 < C; c0 += SB_C) {
    const int nc = min(SB_C, C - c0);
    __syncthreads();
    {  // 96 (channel, tap) rows of 32 output channels: 12 per warp, every load in flight first
      const int o = threadIdx.x & 31;
      float wv[SB_C * 3 / (SP_THREADS / 32)];
#pragma unroll
      for (int i = 0; i < SB_C * 3 / (SP_THREADS / 32); ++i) {
        const int ct = (threadIdx.x >> 5) + i * (SP_THREADS / 32), c = ct / 3, k = ct - 3 * c;
        const int tap = rowline ? kout * 3 + k : k * 3 + kout;
        wv[i] = (c < nc && o < no) ? __ldg(w + ((int64_t)(c0 + c) * 9 + tap) * co + oc0 + o) : 0.0f;
      }
#pragma unroll
      for (int i = 0; i < SB_C * 3 / (SP_THREADS / 32); ++i) {
        const int ct = (threadIdx.x >> 5) + i * (SP_THREADS / 32), c = ct / 3, k = ct - 3 * c;
        sW[c][k][o] = wv[i];
      }
      if (rowline && (p0 == 0 || p0 + 32 >= len)) {  // the column taps of the corners
        for (int ct = threadIdx.x >> 5; ct < SB_C * 6; ct += SP_THREADS / 32) {
          const int c = ct / 6, r = ct - 6 * c, kcs = r / 3, kh = r - 3 * kcs;
          sWc[c][kcs][kh][o] = (c < nc && o < no) ? __ldg(w + ((int64_t)(c0 + c) * 9 + kh * 3 + 2 * kcs) * co + oc0 + o)
                                                  : 0.0f;
        }
      }
    }
#pragma unroll
    for (int sl = 0; sl < SB_SPB; ++sl) {
      if (sl >= nss) break;
      const int s = s0 + sl;
      __syncthreads();
      {  // the low-res window under the line (2 lines x <= 20 along it per channel), loads first
        float lv[SB_C * 2 * SB_WL / SP_THREADS];
#pragma unroll
        for (int i = 0; i < SB_C * 2 * SB_WL / SP_THREADS; ++i) {
          const int e = threadIdx.x + i * SP_THREADS, c = e / (2 * SB_WL), r = e - c * 2 * SB_WL;
          const int k = r / SB_WL, q = r - k * SB_WL;
          const int along = min(wlo + q, (rowline ? x.W : x.H) - 1);
          const int across = k ? ac1 : ac0;
          lv[i] = c < nc ? __ldg(x.plane(s, c0 + c) + (rowline ? (int64_t)across * x.W + along
                                                               : (int64_t)along * x.W + across))
                         : 0.0f;
        }
#pragma unroll
        for (int i = 0; i < SB_C * 2 * SB_WL / SP_THREADS; ++i) {
          const int e = threadIdx.x + i * SP_THREADS, c = e / (2 * SB_WL), r = e - c * 2 * SB_WL;
          sL[c][r / SB_WL][r % SB_WL] = lv[i];
        }
      }
      __syncthreads();
      // U along the line from the window (dense_upsample's op order: rows first, then columns); the
      // corners' other-row sites straight from global memory (2 per channel)
      for (int e = threadIdx.x; e < SB_C * 36; e += SP_THREADS) {
        const int c = e / 36, q = e - 36 * c;
        float v = 0.0f;
        if (c < nc) {
          if (q < 34) {
            const int pp = min(max(p0 - 1 + q, 0), len - 1);
            const Tap ta = tap2(pp, rowline ? x.W : x.H);  // along the line
            const float a0 = sL[c][0][ta.i0 - wlo], a1 = sL[c][1][ta.i0 - wlo];
            const float b0 = sL[c][0][ta.i1 - wlo], b1 = sL[c][1][ta.i1 - wlo];
            if (rowline) {  // rows (across) first: r(col) = x[ac0][col] w0 + x[ac1][col] w1, then columns
              const float ra = __fadd_rn(__fmul_rn(a0, tx.w0), __fmul_rn(a1, tx.w1));
              const float rb = __fadd_rn(__fmul_rn(b0, tx.w0), __fmul_rn(b1, tx.w1));
              v = __fadd_rn(__fmul_rn(ra, ta.w0), __fmul_rn(rb, ta.w1));
            } else {  // rows (along) first: r(col k) = x[row i0][k] w0 + x[row i1][k] w1, then the columns
              const float ra = __fadd_rn(__fmul_rn(a0, ta.w0), __fmul_rn(b0, ta.w1));
              const float rb = __fadd_rn(__fmul_rn(a1, ta.w0), __fmul_rn(b1, ta.w1));
              v = __fadd_rn(__fmul_rn(ra, tx.w0), __fmul_rn(rb, tx.w1));
            }
          } else if (rowline) {
            v = up2(x.plane(s, c0 + c), x.H, x.W, other, q == 34 ? 0 : Wo - 1);
          }
        }
        sU[c][q] = v;
      }
      __syncthreads();
      if (pos < len && 4 * og < no) {
        float a4[4] = {acc[sl][0], acc[sl][1], acc[sl][2], acc[sl][3]};
        const int ch0 = split ? hf * ((nc + 1) >> 1) : 0, ch1 = split && !hf ? (nc + 1) >> 1 : nc;
        for (int c = ch0; c < ch1; ++c) {
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            const float uk = sU[c][pl + k];
            const float4 wv = *reinterpret_cast<const float4*>(&sW[c][k][4 * og]);
            a4[0] = __fmaf_rn(wv.x, uk, a4[0]);
            a4[1] = __fmaf_rn(wv.y, uk, a4[1]);
            a4[2] = __fmaf_rn(wv.z, uk, a4[2]);
            a4[3] = __fmaf_rn(wv.w, uk, a4[3]);
          }
          if (corner) {  // taps (kh, kc) leaving through the column: rows fixed (line value) and `other`
            const int kc = pos == 0 ? 0 : 2;
#pragma unroll
            for (int kh = 0; kh < 3; ++kh) {
              const int yy = fixed + kh - 1;
              if (yy < 0 || yy >= Ho) continue;  // (counted on the row line)
              const float uk = yy == fixed ? sU[c][pl + 1] : sU[c][pos == 0 ? 34 : 35];
              const float4 wv = *reinterpret_cast<const float4*>(&sWc[c][kc >> 1][kh][4 * og]);
              a4[0] = __fmaf_rn(wv.x, uk, a4[0]);
              a4[1] = __fmaf_rn(wv.y, uk, a4[1]);
              a4[2] = __fmaf_rn(wv.z, uk, a4[2]);
              a4[3] = __fmaf_rn(wv.w, uk, a4[3]);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[sl][j] = a4[j];
      }
    }
  }
  if (split) {  // add the second half's partial sums (every thread reaches these barriers)
    float* red = sm + SB_C * 9 * 32 + SB_C * 36 + SB_C * 2 * SB_WL;  // [og][pos][4]
    __syncthreads();
    if (hf)
#pragma unroll
      for (int j = 0; j < 4; ++j) red[(og * 32 + pl) * 4 + j] = acc[0][j];
    __syncthreads();
    if (hf) return;
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[0][j] = __fadd_rn(acc[0][j], red[(og * 32 + pl) * 4 + j]);
  }
  if (pos < len) {
    const int li = L == 0 ? pos : (L == 1 ? Wo + pos : (L == 2 ? 2 * Wo + pos : 2 * Wo + Ho + pos));
#pragma unroll
    for (int sl = 0; sl < SB_SPB; ++sl) {
      if (sl >= nss) break;
      float* o = out + ((int64_t)(s0 + sl) * 2 * (Ho + Wo) + li) * co + oc0 + 4 * og;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (4 * og + j < no) o[j] = -acc[sl][j];
    }
  }
}

#ifndef EVC_SB_MINB
#define EVC_SB_MINB 4
#endif
__global__ void __launch_bounds__(SP_THREADS, EVC_SB_MINB) k_subpix_border(TView x, const float* __restrict__ w, int co, int S,
                                                               float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  __shared__ __align__(16) float sm[SB_SMEM_FLOATS];
  subpix_border_body(x, w, co, S, out, (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z, sm);
}

// Both passes in one launch (they only read x): grid (nx + nbb, GH, S); x blocks >= nx run the border
// GEMM, CTA b = (blockIdx.x - nx) * GH + blockIdx.y of its (nbx x nby) grid per session, so its
// latency-bound CTAs spread between the input pass's instead of forming a serial phase.
#ifndef EVC_SIB_MINB
#define EVC_SIB_MINB 4
#endif
__global__ void __launch_bounds__(SP_THREADS, EVC_SIB_MINB) k_subpix_input_border(
    TView x, uint8_t* __restrict__ yf, int64_t yfs, int GHy, int GWy, double* __restrict__ part,
    float* __restrict__ hwc, int64_t hs, int cp, int pitch, uint8_t* __restrict__ fany_lo,
    uint8_t* __restrict__ fany_hi, int CW, int nJB, int nx, const float* __restrict__ w, int co, float* __restrict__ bout,
    int nbx, int nby) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) float si_dyn[];
  if ((int)blockIdx.x >= nx) {
    const int b = ((int)blockIdx.x - nx) * (int)gridDim.y + (int)blockIdx.y;
    if (b >= nbx * nby) return;
    subpix_border_body(x, w, co, (int)gridDim.z, bout, b % nbx, b / nbx, (int)blockIdx.z, si_dyn);
    return;
  }
  subpix_input_body(x, yf, yfs, GHy, GWy, part, hwc, hs, cp, pitch, fany_lo, fany_hi, CW, nJB, (int)blockIdx.x, nx,
                    si_dyn);
}

constexpr size_t SI_SMEM = sizeof(float) * SI_CH * (SI_R * SI_C + 1);

int init_subpixel() {
  static_assert(SB_SMEM_FLOATS * sizeof(float) <= SI_SMEM, "border GEMM carve exceeds the input pass's shared memory");
  return (cudaFuncSetAttribute(k_subpix_input, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SI_SMEM) == cudaSuccess &&
          cudaFuncSetAttribute(k_subpix_input_border, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SI_SMEM) ==
              cudaSuccess)
             ? EVC_OK
             : EVC_ECUDA;
}

}  // namespace evc

using namespace evc;

extern "C" {

static void si_geom(const TView& v, int cp, int& CW, int& nJB, int& nx) {
  (void)cp;
  CW = v.tw * (32 / v.tw);
  nJB = (v.W + CW - 1) / CW;
  // channel chunks of 32; a remainder <= SI_CH - 32 joins the last full chunk
  const int full = v.C / 32, rem = v.C - 32 * full;
  const int nchunk = full == 0 ? 1 : (rem == 0 ? full : (rem <= SI_CH - 32 ? full : full + 1));
  nx = nJB * nchunk;
}

int64_t evc_subpixel_input_partials(const evc_tensor* x, int32_t cp) {
  if (!x) return -1;
  const TView v = view_of(*x);
  int CW, nJB, nx;
  si_geom(v, cp, CW, nJB, nx);
  return (int64_t)nx * v.GH;
}

int evc_subpixel_input(const evc_tensor* x, const evc_tensor* y, double* partials, float* hwc, int32_t cp,
                       int64_t hwc_stride, int32_t pitch, uint8_t* fany_lo, uint8_t* fany_hi, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && x->flags && y && y->flags && partials && hwc && S > 0, "subpixel_input: null argument");
  EVC_CHECK_ARG(y->C == x->C && y->H == 2 * x->H && y->W == 2 * x->W && y->th == x->th && y->tw == x->tw &&
                    x->th % 2 == 0 && x->tw % 2 == 0 && x->th <= 8 && x->tw >= 6 && x->tw <= 32,
                "subpixel_input: y must be the 2x upsample of x with the same even tiles (th <= 8, 6 <= tw <= 32)");
  EVC_CHECK_ARG(cp >= x->C && cp % 32 == 0 && pitch >= x->W + 2,
                "subpixel_input: shadow channels (multiple of 32 >= C), pitch >= W + 2");
  const TView v = view_of(*x);
  const TView vy = view_of(*y);
  int CW, nJB, nx;
  si_geom(v, cp, CW, nJB, nx);
  launch_pdl(k_subpix_input, dim3((unsigned)nx, (unsigned)v.GH, (unsigned)S), dim3(SP_THREADS), SI_SMEM,
             as_stream(stream), v, vy.f, vy.fs, vy.GH, vy.GW, partials, hwc, hwc_stride, (int)cp, (int)pitch, fany_lo,
             fany_hi, CW, nJB);
  EVC_LAUNCH_CHECK("subpixel_input");
  return EVC_OK;
}

int evc_subpixel_border(const evc_tensor* x, const float* w, int32_t c_out, float* out, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && w && out && c_out > 0 && c_out % 4 == 0 && S > 0, "subpixel_border: null argument");
  const TView v = view_of(*x);
  const int len = 2 * std::max(v.H, v.W);
  const dim3 grid((unsigned)((len + 31) / 32), (unsigned)(4 * ((c_out + 31) / 32)),
                  (unsigned)((S + SB_SPB - 1) / SB_SPB));
  launch_pdl(k_subpix_border, grid, dim3(SP_THREADS), 0, as_stream(stream), v, w, (int)c_out, (int)S, out);
  EVC_LAUNCH_CHECK("subpixel_border");
  return EVC_OK;
}

int evc_subpixel_input_border(const evc_tensor* x, const evc_tensor* y, double* partials, float* hwc, int32_t cp,
                              int64_t hwc_stride, int32_t pitch, uint8_t* fany_lo, uint8_t* fany_hi, const float* w,
                              int32_t c_out, float* border, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && x->flags && y && y->flags && partials && hwc && w && border && S > 0 && c_out > 0 &&
                    c_out % 4 == 0,
                "subpixel_input_border: null argument");
  EVC_CHECK_ARG(y->C == x->C && y->H == 2 * x->H && y->W == 2 * x->W && y->th == x->th && y->tw == x->tw &&
                    x->th % 2 == 0 && x->tw % 2 == 0 && x->th <= 8 && x->tw >= 6 && x->tw <= 32,
                "subpixel_input_border: y must be the 2x upsample of x with the same even tiles (th <= 8, 6 <= tw <= 32)");
  EVC_CHECK_ARG(cp >= x->C && cp % 32 == 0 && pitch >= x->W + 2,
                "subpixel_input_border: shadow channels (multiple of 32 >= C), pitch >= W + 2");
  const TView v = view_of(*x);
  const TView vy = view_of(*y);
  int CW, nJB, nx;
  si_geom(v, cp, CW, nJB, nx);
  const int len = 2 * std::max(v.H, v.W);
  const int nbx = (len + 31) / 32, nby = 4 * ((c_out + 31) / 32);
  const int nbb = (nbx * nby + v.GH - 1) / v.GH;  // extra x blocks holding the border CTAs
  launch_pdl(k_subpix_input_border, dim3((unsigned)(nx + nbb), (unsigned)v.GH, (unsigned)S), dim3(SP_THREADS),
             SI_SMEM, as_stream(stream), v, vy.f, vy.fs, vy.GH, vy.GW, partials, hwc, hwc_stride, (int)cp, (int)pitch,
             fany_lo, fany_hi, CW, nJB, nx, w, (int)c_out, border, nbx, nby);
  EVC_LAUNCH_CHECK("subpixel_input_border");
  return EVC_OK;
}

}  // extern "C"
