// Fused inc_upsample -> sparsify_step (the decoder pattern "upsample, then the
// conv's sparsify layer": increment_ops.py:271-285 followed by sparsify.py:54-78).
//
// The upsampled increment exists only in registers: each CTA (32 channels x one
// output tile row x a tile-aligned column chunk) evaluates the upsample of the
// small input on the fly (same float32 op order as dense_upsample), applies the
// error-feedback rounding, derives the output tile flags from the values, and
// writes the next conv's channels-innermost shadow directly.  A tile is
// processed when its upsample support is live, when it was live in the output
// last step, or when its residual is nonzero -- exactly the tiles the unfused
// pair could change.  Norm partials are folded by the last CTA (fixed order).

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace evc {

constexpr int US_C = 32, US_THREADS = 256, US_MAXJ = 32, US_MAXR = 32;

struct USArgs {
  TView x;         // upsample input (masked)
  TView y;         // sparsify output (flags; values when write_chw)
  float* delta;    // residual
  int64_t ds;
  uint8_t* dlive;
  double* k;
  double* norm_ema;
  double tp, decay;
  double* partials;
  int* ticket;
  float* hwc;
  int64_t hs;
  int hp;  // shadow row pitch (pixels)
  uint8_t* fany;  // optional any-channel tile map of y (OR-accumulated, zeroed per step)
  int cp, write_chw, delta_zero, f, mode;
  int XR, XC;  // staged input footprint (rows, cols) per CTA
  int fast;    // t_p = 0 into a shadow only: no output staging buffer (smaller CTA -> more per SM)
  int CW, nCG, nJC;
  int RT;       // output tile rows per CTA (2 on the fast path when they fit, else 1)
  int pstride;  // partial slots per session (the RT = 1 CTA count)
  int RS;       // fast path: channel stride of the row-interpolated buffer (odd)
};

__global__ void __launch_bounds__(US_THREADS, 4) k_up_sparsify(USArgs a) {
  pdl_wait();
  pdl_trigger();
  __shared__ uint8_t s_proc[US_C * US_MAXJ], s_ny[US_C * US_MAXJ], s_nd[US_C * US_MAXJ], s_fin[US_C * US_MAXJ];
  extern __shared__ float us_dyn[];
  float* s_y = us_dyn;                             // [(row * 32 + col) * 33 + channel] staged output
  float* s_x = us_dyn + (a.fast ? 0 : 8 * 32 * 33);  // [channel][XR][XC] input footprint of this CTA
  // static upsample taps of this CTA's output columns / rows (tensors.py:259-282)
  __shared__ int s_ci0[32], s_ci1[32], s_ri0[US_MAXR], s_ri1[US_MAXR], s_tj[32], s_ro0[US_MAXR], s_ro1[US_MAXR];
  __shared__ float s_cw0[32], s_cw1[32], s_rw0[US_MAXR], s_rw1[US_MAXR];
  const TView& y = a.y;
  const FDiv d_tw_y = fdiv_of(y.tw);
  const int rest = fdiv(blockIdx.x, fdiv_of(a.nJC)), jc = blockIdx.x - rest * a.nJC;
  const int ib = fdiv(rest, fdiv_of(a.nCG)), cg = rest - ib * a.nCG, s = blockIdx.y;
  const int c0 = cg * US_C, nc = min(US_C, y.C - c0);
  const int x0 = jc * a.CW, ncol = min(y.W, x0 + a.CW) - x0;
  const int j0 = fdiv(x0, d_tw_y), nj = fdiv(ncol + y.tw - 1, d_tw_y);
  const int i0 = ib * a.RT, nti = min(y.GH - i0, a.RT);  // tile rows of this CTA
  const int r0 = i0 * y.th, nrow = min(y.H, r0 + nti * y.th) - r0;
  const int NT = nti * nj;  // tiles per channel: t = channel * NT + tile row * nj + tile column
  // 1) taps of this CTA's output columns / rows
  if (threadIdx.x < ncol) {
    const int v = x0 + threadIdx.x;
    s_tj[threadIdx.x] = fdiv(threadIdx.x, d_tw_y);
    if (a.mode == 0) {
      s_ci0[threadIdx.x] = s_ci1[threadIdx.x] = v / a.f;
      s_cw0[threadIdx.x] = 1.0f;
      s_cw1[threadIdx.x] = 0.0f;
    } else {
      const Tap t = bilinear_tap(v, a.x.W, a.f);
      s_ci0[threadIdx.x] = t.i0;
      s_ci1[threadIdx.x] = t.i1;
      s_cw0[threadIdx.x] = t.w0;
      s_cw1[threadIdx.x] = t.w1;
    }
  } else if (threadIdx.x >= 32 && threadIdx.x < 32 + nrow) {
    const int r = threadIdx.x - 32, u = r0 + r;
    if (a.mode == 0) {
      s_ri0[r] = s_ri1[r] = u / a.f;
      s_rw0[r] = 1.0f;
      s_rw1[r] = 0.0f;
    } else {
      const Tap t = bilinear_tap(u, a.x.H, a.f);
      s_ri0[r] = t.i0;
      s_ri1[r] = t.i1;
      s_rw0[r] = t.w0;
      s_rw1[r] = t.w1;
    }
  }
  // the CTA's input box from the taps of its corner pixels (taps are monotone), computed by
  // every thread so the flag loads below need no barrier first
  // (integer form of bilinear_tap's floor((o + 0.5) / f - 0.5), exact for f in {2, 4}:
  // floor((2o + 1 - f) / 2f), with 2f a power of two and 2o + 1 - f >= -3)
  const int fsh = a.f == 2 ? 2 : 3;
  auto tap_fl = [&](int o) { const int q = 2 * o + 1 - a.f; return q >= 0 ? q >> fsh : -1; };
  auto tap_i0 = [&](int u, int n) { return a.mode == 0 ? u >> (fsh - 1) : min(max(tap_fl(u), 0), n - 1); };
  auto tap_i1 = [&](int u, int n) { return a.mode == 0 ? u >> (fsh - 1) : min(max(tap_fl(u) + 1, 0), n - 1); };
  const int rlo = tap_i0(r0, a.x.H), nr = tap_i1(r0 + nrow - 1, a.x.H) - rlo + 1;
  const int clo = tap_i0(x0, a.x.W), ncl = tap_i1(x0 + ncol - 1, a.x.W) - clo + 1;
  const FDiv d_th = fdiv_of(a.x.th), d_tw = fdiv_of(a.x.tw), d_NT = fdiv_of(NT), d_nj = fdiv_of(nj);
  const int alo = fdiv(rlo, d_th), ahi = fdiv(rlo + nr - 1, d_th);
  const int blo0 = fdiv(clo, d_tw), bhi0 = fdiv(clo + ncl - 1, d_tw);
  const int na_ = ahi - alo + 1, nb_ = bhi0 - blo0 + 1;
  const bool box_fits = na_ * nb_ <= US_MAXJ;
  // last step's output / residual flags and the input flags of the box (all channels):
  // every load in flight at once
  for (int t = threadIdx.x; t < nc * NT; t += US_THREADS) {
    const int cl = fdiv(t, d_NT), e = t - cl * NT, tr = fdiv(e, d_nj), jl = e - tr * nj;
    const int64_t fo = ((int64_t)(c0 + cl) * y.GH + i0 + tr) * y.GW + j0 + jl;
    // t_p = 0 (fast path): the residual and its live flags are identically 0 -- not read
    s_nd[t] = y.f[(int64_t)s * y.fs + fo] | (a.fast ? 0 : a.dlive[(int64_t)s * y.C * y.GH * y.GW + fo]);
    s_ny[t] = 0;
  }
  if (box_fits) {
    const FDiv d_box = fdiv_of(na_ * nb_), d_nb = fdiv_of(nb_);
    for (int t = threadIdx.x; t < nc * na_ * nb_; t += US_THREADS) {
      const int cl = fdiv(t, d_box), e = t - cl * na_ * nb_, ea = fdiv(e, d_nb);
      s_fin[t] = a.x.fplane(s, c0 + cl)[(alo + ea) * a.x.GW + blo0 + e - ea * nb_];
    }
  }
  __syncthreads();
  // 2) process a tile when its upsample support is live, or it was live / left a residual
  bool any = false;
  for (int t = threadIdx.x; t < nc * NT; t += US_THREADS) {
    const int cl = fdiv(t, d_NT), e = t - cl * NT, tr = fdiv(e, d_nj), jl = e - tr * nj;
    const int xa = jl * y.tw, xb = min(ncol, xa + y.tw) - 1;
    const int ya = tr * y.th, yb = min(nrow, ya + y.th) - 1;
    const int blo = fdiv(s_ci0[xa], d_tw), bhi = fdiv(s_ci1[xb], d_tw);
    const int alo_t = fdiv(s_ri0[ya], d_th), ahi_t = fdiv(s_ri1[yb], d_th);
    uint8_t live = 0;
    if (box_fits) {
      for (int aa = alo_t; aa <= ahi_t; ++aa)
        for (int bb = blo; bb <= bhi; ++bb) live |= s_fin[(cl * na_ + aa - alo) * nb_ + bb - blo0];
    } else {
      const uint8_t* F = a.x.fplane(s, c0 + cl);
      for (int aa = alo_t; aa <= ahi_t; ++aa)
        for (int bb = blo; bb <= bhi; ++bb) live |= F[aa * a.x.GW + bb];
    }
    s_proc[t] = (live | s_nd[t]) != 0;
    any |= s_proc[t] != 0;
    s_nd[t] = 0;  // same thread, same entry: from here on this step's residual flags
  }
  const bool active = __syncthreads_or(any) != 0;
  double ss = 0.0;
  const bool stage = a.hwc && nrow <= 8 && ncol <= 32;
  if (active) {
    const double kd = a.k[s];
    const bool use_k = kd > 0.0;
    const float k32 = __double2float_rn(kd);
    const int64_t HW = (int64_t)y.H * y.W;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // stage the CTA's input footprint (all channels of the group) in shared memory:
    // every global load is issued up front, the upsample then reads shared memory
    const int cs = (a.XR * a.XC) | 1;  // odd channel stride: lane-per-channel reads are bank-conflict free
    if (threadIdx.x < nrow) {  // staged row offsets of each output row's two taps
      s_ro0[threadIdx.x] = (s_ri0[threadIdx.x] - rlo) * a.XC;
      s_ro1[threadIdx.x] = (s_ri1[threadIdx.x] - rlo) * a.XC;
    }
    {  // eight threads per channel walk its rows; each copies every eighth column (32-byte runs)
      const int cl = threadIdx.x >> 3, sub = threadIdx.x & 7;
      if (cl < nc) {
        const float* xs = a.x.plane(s, c0 + cl) + (int64_t)rlo * a.x.W + clo;
        float* xd = s_x + cl * cs;
        for (int rr = 0; rr < nr; ++rr, xs += a.x.W, xd += a.XC)
          for (int cc = sub; cc < ncl; cc += 8) cp_async4(xd + cc, xs + cc);
      }
      cp_async_wait_all();
    }
    __syncthreads();
    const bool fast = a.fast;
    if (fast) {
      // t_p = 0 fast path, separable: (1) the row interpolation R[channel][row][input col]
      // once per input column, (2) the column interpolation + split per output pixel.
      // lane -> (channel cl = lane % nc, column phase q = lane / nc): a narrow remainder
      // group (the 2 flow channels of a decoder concat) still fills the warp.
      const int Q = 32 / nc, cl = lane % nc, q = lane / nc;
      const int RS = a.RS;
      float* s_r = s_x + US_C * cs;  // [channel][row][input col] row-interpolated input
      if (q < Q) {  // work items (row, column half): the per-row taps are read once per 8+ columns
        const float* xc = s_x + cl * cs;
        float* rc = s_r + cl * RS;
        const int half_c = (ncl + 1) >> 1;
        for (int it = warp; it < 2 * nrow; it += US_THREADS / 32) {
          const int r = it >> 1, c0 = (it & 1) * half_c, c1 = min(ncl, c0 + half_c);
          const float* xr0 = xc + s_ro0[r];
          const float* xr1 = xc + s_ro1[r];
          const float rw0 = s_rw0[r], rw1 = s_rw1[r];
          float* rr_ = rc + r * a.XC;
          if (Q == 1) {  // full channel group: unit stride, unrolled
#pragma unroll 4
            for (int c = c0; c < c1; ++c)
              rr_[c] = a.mode == 0 ? xr0[c] : __fadd_rn(__fmul_rn(xr0[c], rw0), __fmul_rn(xr1[c], rw1));
          } else {
            for (int c = c0 + q; c < c1; c += Q)
              rr_[c] = a.mode == 0 ? xr0[c] : __fadd_rn(__fmul_rn(xr0[c], rw0), __fmul_rn(xr1[c], rw1));
          }
        }
      }
      __syncthreads();
      if (q < Q) {
        const float* rc = s_r + cl * RS;
        // (no shadow: flags, any-map and norm partials only -- the sub-pixel conv reads the low-res input)
        const bool wr = a.hwc != nullptr;
        const int rstride = wr ? a.hp * hwc_px(a.cp) : 0;  // floats between shadow rows (< 2^31 per session)
        float* sbase = wr ? a.hwc + (int64_t)s * a.hs + hwc_head(a.cp, c0 + cl) : nullptr;
        const int tl = !wr ? 0 : (a.cp < 0 ? -1 : hwc_unit(a.cp));  // tail offset (32 floats: an immediate); -1: fp32
        const int obase = r0 * rstride + x0 * hwc_px(a.cp);
        float ssf = 0.0f;
        for (int xq = warp * Q + q; xq < ncol; xq += (US_THREADS / 32) * Q) {
        // the column's taps once (before any s_ny store of this column)
        const int tj = s_tj[xq], o0 = s_ci0[xq] - clo, o1 = s_ci1[xq] - clo;
        const float cw0 = s_cw0[xq], cw1 = s_cw1[xq];
        float* dcol = wr ? sbase + obase + xq * hwc_px(a.cp) : nullptr;
        for (int tr = 0; tr < nti; ++tr) {
          const int ti = cl * NT + tr * nj + tj;
          if (!s_proc[ti]) continue;  // not live now nor last step: the shadow already holds zeros
          const int ra = tr * y.th, rb = min(nrow, ra + y.th);
          const float* p0 = rc + ra * a.XC + o0;
          const float* p1 = rc + ra * a.XC + o1;
          float* d = wr ? dcol + ra * rstride : nullptr;
          uint32_t nzb = 0;  // OR of the value bits: some value != +-0 iff a magnitude bit is set
          // same float32 op order as upsample_at (rows first, then columns)
          auto row = [&](int k) {
            const float up = a.mode == 0 ? p0[k * a.XC]
                                         : __fadd_rn(__fmul_rn(p0[k * a.XC], cw0), __fmul_rn(p1[k * a.XC], cw1));
            const float ov = __fadd_rn(0.0f, up);
            float* dk = wr ? d + (int64_t)k * rstride : nullptr;
            if (!wr) {
            } else if (tl < 0) {  // fp32 shadow (hwc_px)
              dk[0] = ov;
            } else {
              const float h = tf32_head(ov);
              dk[0] = h;
              dk[tl] = __fsub_rn(ov, h);
            }
            ssf = __fmaf_rn(ov, ov, ssf);
            nzb |= __float_as_uint(ov);  // (sign bits masked once per tile below)
          };
          if (rb - ra == 6) {  // the 6-row tiles of the reference default: fully unrolled
#pragma unroll
            for (int k = 0; k < 6; ++k) row(k);
          } else {
            for (int k = 0; k < rb - ra; ++k) row(k);
          }
          if (nzb & 0x7fffffffu) s_ny[ti] = 1;
        }
        }
        ss += (double)ssf;
      }
    } else {
    // lane = output column (ncol <= 32); warp w owns channels w, w + 8, ...
    const bool col_ok = lane < ncol;
    const int xl = lane, jl_lane = lane / y.tw;
    const int ci0 = col_ok ? s_ci0[xl] - clo : 0, ci1 = col_ok ? s_ci1[xl] - clo : 0;
    const float cw0 = col_ok ? s_cw0[xl] : 0.0f, cw1 = col_ok ? s_cw1[xl] : 0.0f;
    for (int cl = warp; cl < nc; cl += US_THREADS / 32)
    for (int r = 0; r < nrow; ++r) {
      if (!col_ok) continue;
      const int ti = cl * NT + jl_lane;  // RT = 1 here: NT = nj
      if (!s_proc[ti]) {
        if (stage) s_y[(r * 32 + xl) * 33 + cl] = 0.0f;
        continue;
      }
      const int c = c0 + cl, u = r0 + r, v = x0 + xl;
      const float* xr0 = s_x + cl * cs + (s_ri0[r] - rlo) * a.XC;
      float up;
      if (a.mode == 0) {
        up = xr0[ci0];
      } else {  // same float32 op order as upsample_at (rows first, then columns)
        const float* xr1 = s_x + cl * cs + (s_ri1[r] - rlo) * a.XC;
        const float rw0 = s_rw0[r], rw1 = s_rw1[r];
        const float ra = __fadd_rn(__fmul_rn(xr0[ci0], rw0), __fmul_rn(xr1[ci0], rw1));
        const float rb = __fadd_rn(__fmul_rn(xr0[ci1], rw0), __fmul_rn(xr1[ci1], rw1));
        up = __fadd_rn(__fmul_rn(ra, cw0), __fmul_rn(rb, cw1));
      }
      const int64_t off = (int64_t)c * HW + (int64_t)u * y.W + v;
      float* dp = a.delta + (int64_t)s * a.ds + off;
      const float corr = a.delta_zero ? __fadd_rn(0.0f, up) : __fadd_rn(*dp, up);
      float o, nd;
      if (use_k) {
        o = __fmul_rn(k32, floorf(__fadd_rn(0.5f, __fdiv_rn(corr, k32))));
        nd = __fsub_rn(corr, o);
      } else {
        o = corr;
        nd = 0.0f;
      }
      if (a.write_chw) y.v[(int64_t)s * y.vs + off] = o;
      if (stage) {
        s_y[(r * 32 + xl) * 33 + cl] = o;
      } else if (a.hwc) {
        hwc_store(a.hwc + (int64_t)s * a.hs + ((int64_t)u * a.hp + v) * hwc_px(a.cp), a.cp, c, o);
      }
      if (!a.delta_zero) *dp = nd;
      ss += (double)corr * (double)corr;
      if (o != 0.0f) s_ny[ti] = 1;
      if (nd != 0.0f) s_nd[ti] = 1;
    }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < nc * NT; t += US_THREADS) {
      const int cl = fdiv(t, d_NT), e = t - cl * NT, tr = fdiv(e, d_nj), jl = e - tr * nj;
      const int64_t fo = ((int64_t)(c0 + cl) * y.GH + i0 + tr) * y.GW + j0 + jl;
      y.f[(int64_t)s * y.fs + fo] = s_ny[t];
      if (a.fany && s_ny[t]) a.fany[((int64_t)s * y.GH + i0 + tr) * y.GW + j0 + jl] = 1;  // benign race: all store 1
      if (!a.fast) a.dlive[(int64_t)s * y.C * y.GH * y.GW + fo] = s_nd[t];
    }
    if (stage && !fast && lane < nc) {  // lane = channel: 128-byte runs of heads and of tails per pixel
      float* dst = a.hwc + (int64_t)s * a.hs + (int64_t)r0 * a.hp * hwc_px(a.cp);
      for (int r = 0; r < nrow; ++r)
        for (int xq = warp; xq < ncol; xq += US_THREADS / 32)
          hwc_store(dst + ((int64_t)r * a.hp + x0 + xq) * hwc_px(a.cp), a.cp, c0 + lane, s_y[(r * 32 + xq) * 33 + lane]);
    }
  }
  {  // block sum: the t_p = 0 path's per-thread sums are fp32 already -> fp32 warp sums
    __shared__ double s_wsum[US_THREADS / 32];
    const double w = a.fast ? (double)warp_sum((float)ss) : warp_sum_d(ss);
    if ((threadIdx.x & 31) == 0) s_wsum[threadIdx.x >> 5] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < US_THREADS / 32; ++k) t += s_wsum[k];
      ss = t;
    }
  }
  if (threadIdx.x == 0) {
    a.partials[(int64_t)s * a.pstride + blockIdx.x] = ss;
    if (blockIdx.x + gridDim.x < (unsigned)a.pstride) a.partials[(int64_t)s * a.pstride + blockIdx.x + gridDim.x] = 0.0;
  }
  if (!a.ticket) return;  // norm / k folded later by evc_meter_step (one launch for every node)
  const int nblocks = gridDim.x * gridDim.y;
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(a.ticket, 1) == nblocks - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    sparsify_finalize_all(a.partials, a.pstride, a.norm_ema, a.k, a.tp, a.decay, 0, gridDim.y);
  }
}

int init_upsparsify() {
  return cudaFuncSetAttribute(k_up_sparsify, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024) == cudaSuccess
             ? EVC_OK
             : EVC_ECUDA;
}

static void us_grid(const TView& y, int& CW, int& nCG, int& nJC) {
  CW = y.tw >= 32 ? y.tw : y.tw * (32 / y.tw);
  nCG = (y.C + US_C - 1) / US_C;
  nJC = (y.W + CW - 1) / CW;
}

}  // namespace evc

using namespace evc;

extern "C" {

int64_t evc_upsample_sparsify_partials(const evc_tensor* y) {
  if (!y) return -1;
  int CW, nCG, nJC;
  const TView v = view_of(*y);
  us_grid(v, CW, nCG, nJC);
  return (int64_t)v.GH * nCG * nJC;
}

int evc_upsample_sparsify(const evc_tensor* x, int32_t factor, int32_t mode, float* delta, int64_t ds,
                          uint8_t* dlive, const evc_tensor* y, double* k, double* norm_ema, double tp,
                          double ema_decay, double* partials, int32_t* ticket, float* hwc, int32_t cp,
                          int64_t hwc_stride, int32_t hwc_pitch, uint8_t* fany, int32_t write_chw,
                          int32_t delta_zero, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && y && x->flags && y->flags && delta && dlive && k && norm_ema && partials && S > 0,
                "upsample_sparsify: null argument");
  EVC_CHECK_ARG(y->tw <= 32 && y->th <= 8, "upsample_sparsify: tiles wider than 32 or taller than 8");
  EVC_CHECK_ARG(factor == 2 || factor == 4, "upsample_sparsify: factor must be 2 or 4");
  EVC_CHECK_ARG(mode == 0 || mode == 1, "upsample_sparsify: unknown mode");
  EVC_CHECK_ARG(y->H == x->H * factor && y->W == x->W * factor && y->C == x->C, "upsample_sparsify: shape");
  EVC_CHECK_ARG(write_chw || hwc || (delta_zero && tp == 0.0 && fany),
                "upsample_sparsify: no output requested (flags-only needs t_p = 0, a zero residual and fany)");
  EVC_CHECK_ARG(!hwc || (std::abs(cp) >= y->C && cp % 4 == 0 && hwc_pitch >= y->W),
                "upsample_sparsify: shadow channel count must cover C (multiple of 32), pitch >= W");
  USArgs a;
  a.x = view_of(*x);
  a.y = view_of(*y);
  a.delta = delta;
  a.ds = ds;
  a.dlive = dlive;
  a.k = k;
  a.norm_ema = norm_ema;
  a.tp = tp;
  a.decay = ema_decay;
  a.partials = partials;
  a.ticket = ticket;
  a.hwc = hwc;
  a.hs = hwc_stride;
  a.hp = hwc_pitch;
  a.cp = cp;
  a.fany = fany;
  a.write_chw = write_chw;
  a.delta_zero = delta_zero;
  a.f = factor;
  a.mode = mode;
  us_grid(a.y, a.CW, a.nCG, a.nJC);
  a.fast = (delta_zero && tp == 0.0 && !write_chw) ? 1 : 0;
  // tile rows per CTA on the fast path (EVC_UP_RT, default 2, when the per-CTA flag tables and 96 KB
  // of staging hold them): measured on C1 at 32 streams, 4 rows (fewer, larger CTAs) cost 25 % more
  // than 2 -- half the CTAs per SM fit -- and 1 row 5 % more (scripts/gpu_iter3.sh)
  a.RT = 1;
  if (a.fast) {
    const char* ev = std::getenv("EVC_UP_RT");
    const int want = ev ? std::max(1, std::atoi(ev)) : 2;
    for (int rt = want; rt > 1 && a.RT == 1; --rt) {
      const size_t xr = rt * y->th / factor + 3, xc = a.CW / factor + 3;
      const size_t bytes = sizeof(float) * US_C * (((rt * y->th * xc) | 1) + ((xr * xc) | 1));
      if (rt * (a.CW / a.y.tw) <= US_MAXJ && rt * a.y.th <= US_MAXR && bytes <= 96 * 1024) a.RT = rt;
    }
  }
  a.pstride = a.y.GH * a.nCG * a.nJC;
  dim3 grid((unsigned)(((a.y.GH + a.RT - 1) / a.RT) * a.nCG * a.nJC), (unsigned)S);
  a.XR = a.RT * y->th / factor + 3;
  a.XC = a.CW / factor + 3;
  a.RS = (a.RT * y->th * a.XC) | 1;
  const size_t smem = sizeof(float) * ((a.fast ? (size_t)US_C * a.RS : 8 * 32 * 33) +
                                       (size_t)US_C * ((a.XR * a.XC) | 1));
  launch_pdl(k_up_sparsify, dim3(grid), dim3(US_THREADS), smem, as_stream(stream), a);
  EVC_LAUNCH_CHECK("upsample_sparsify");
  return EVC_OK;
}

}  // extern "C"
