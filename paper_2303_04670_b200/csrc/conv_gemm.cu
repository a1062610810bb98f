// Gather -> GEMM -> scatter of the incremental convolution over active
// output tiles (increment_ops.py:165-190, tensors.py:205-228).
//
// Values equal the bias-free convolution of the increment: the reference's
// per-channel skip only drops taps that read exact zeros (mask soundness), so
// computing every channel at every site of an active output tile gives the same
// sum up to float reassociation and exact zeros where the reference skips.
// The M dimension packs the sites of the active output tiles (tile list from
// evc_conv_mask); A rows are gathered im2col rows of the channel-planar input,
// B is the weight in the reference's (C_out, C_in*KH*KW) layout.

#include <algorithm>

#include "conv_common.cuh"

namespace evc {

// ---------------------------------------------------------------------------
// FFMA implicit GEMM over packed active sites
// ---------------------------------------------------------------------------
struct GemmArgs {
  TView in, out;
  const float* w;
  const float* bias;
  const int32_t* kdec;
  const int32_t* list;
  const int32_t* count;
  float* ws;
  int64_t mcap;  // capacity of packed sites (workspace row count)
  int c_in, c_out, kh, kw, stride, pad, K;
  int T, GWo, S;
  int splits, kchunk;
};

constexpr int BK = 8;

template <int BM, int BN, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN)) k_conv_gemm(GemmArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = (BN * BK + NT - 1) / NT;
  const int th = a.out.th, tw = a.out.tw, sites = th * tw;
  const int n_tiles = a.list ? *a.count : a.S * a.T;
  const int64_t M = (int64_t)n_tiles * sites;
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  if (m0 >= M) return;
  const int n0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const int kbeg = z * a.kchunk, kend = min(a.K, kbeg + a.kchunk);

  __shared__ __align__(16) float As[2][BK][BM];
  __shared__ __align__(16) float Bs[2][BK][BN];
  __shared__ int64_t s_in[BM];   // session offset + y0*W + x0 into input, or -1
  __shared__ int64_t s_out[BM];  // session offset + u*Wo + v into output, or -1
  __shared__ int s_y0[BM], s_x0[BM];

  const int H = a.in.H, W = a.in.W, Ho = a.out.H, Wo = a.out.W;
  for (int m = threadIdx.x; m < BM; m += NT) {
    const int64_t pm = m0 + m;
    int64_t oi = -1, ii = 0;
    int y0 = -1000000, x0 = -1000000;
    if (pm < M) {
      const int e = (int)(pm / sites), l = (int)(pm % sites);
      const int ent = a.list ? a.list[e] : e;
      const int s = ent / a.T, t = ent % a.T;
      const int u = (t / a.GWo) * th + l / tw, v = (t % a.GWo) * tw + l % tw;
      if (u < Ho && v < Wo) {
        oi = (int64_t)s * a.out.vs + (int64_t)u * Wo + v;
        y0 = u * a.stride - a.pad;
        x0 = v * a.stride - a.pad;
        ii = (int64_t)s * a.in.vs + (int64_t)y0 * W + x0;
      }
    }
    s_in[m] = ii;
    s_out[m] = oi;
    s_y0[m] = y0;
    s_x0[m] = x0;
  }
  __syncthreads();

  const int tm = threadIdx.x % (BM / TM), tn = threadIdx.x / (BM / TM);
  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  float ra[A_PER], rb[B_PER];
  auto load = [&](int k0) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      const int m = idx % BM, kk = idx / BM;
      const int k = k0 + kk;
      float v = 0.0f;
      if (k < kend) {
        const int off = __ldg(a.kdec + 2 * k), rq = __ldg(a.kdec + 2 * k + 1);
        const int iy = s_y0[m] + (rq >> 16), ix = s_x0[m] + (rq & 0xffff);
        if ((unsigned)iy < (unsigned)H && (unsigned)ix < (unsigned)W) v = __ldg(a.in.v + s_in[m] + off);
      }
      ra[e] = v;
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      float v = 0.0f;
      if (idx < BN * BK) {
        const int n = idx / BK, kk = idx % BK;
        const int k = k0 + kk;
        if (k < kend && n0 + n < a.c_out) v = __ldg(a.w + (int64_t)(n0 + n) * a.K + k);
      }
      rb[e] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < A_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      As[buf][idx / BM][idx % BM] = ra[e];
    }
#pragma unroll
    for (int e = 0; e < B_PER; ++e) {
      const int idx = threadIdx.x + e * NT;
      if (idx < BN * BK) Bs[buf][idx % BK][idx / BK] = rb[e];
    }
  };

  const int nk = (kend - kbeg + BK - 1) / BK;
  if (nk > 0) {
    load(kbeg);
    store(0);
    __syncthreads();
    for (int kt = 0; kt < nk; ++kt) {
      const int cur = kt & 1;
      if (kt + 1 < nk) load(kbeg + (kt + 1) * BK);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        float av[TM], bv[TN];
#pragma unroll
        for (int i = 0; i < TM; i += 4) {
          const float4 t4 = *reinterpret_cast<const float4*>(&As[cur][kk][tm * TM + i]);
          av[i] = t4.x; av[i + 1] = t4.y; av[i + 2] = t4.z; av[i + 3] = t4.w;
        }
        if constexpr (TN % 4 == 0) {
#pragma unroll
          for (int j = 0; j < TN; j += 4) {
            const float4 t4 = *reinterpret_cast<const float4*>(&Bs[cur][kk][tn * TN + j]);
            bv[j] = t4.x; bv[j + 1] = t4.y; bv[j + 2] = t4.z; bv[j + 3] = t4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < TN; ++j) bv[j] = Bs[cur][kk][tn * TN + j];
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
      }
      if (kt + 1 < nk) store(cur ^ 1);
      __syncthreads();
    }
  }

  const int64_t plane = (int64_t)Ho * Wo;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int m = tm * TM + i;
    const int64_t pm = m0 + m;
    if (pm >= M) continue;
    const int64_t oi = s_out[m];
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int n = n0 + tn * TN + j;
      if (n >= a.c_out) continue;
      if (a.splits == 1) {
        if (oi >= 0) a.out.v[oi + n * plane] = a.bias ? __fadd_rn(acc[i][j], __ldg(a.bias + n)) : acc[i][j];
      } else {
        a.ws[((int64_t)z * a.mcap + pm) * a.c_out + n] = acc[i][j];
      }
    }
  }
}

// deterministic split-K reduction + scatter
__global__ void k_conv_splitk_reduce(GemmArgs a) {
  pdl_wait();
  pdl_trigger();
  const int th = a.out.th, tw = a.out.tw, sites = th * tw;
  const int n_tiles = a.list ? *a.count : a.S * a.T;
  const int64_t M = (int64_t)n_tiles * sites;
  const int Ho = a.out.H, Wo = a.out.W;
  const int64_t plane = (int64_t)Ho * Wo;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < M * a.c_out;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pm = e / a.c_out;
    const int n = (int)(e % a.c_out);
    const int te = (int)(pm / sites), l = (int)(pm % sites);
    const int ent = a.list ? a.list[te] : te;
    const int s = ent / a.T, t = ent % a.T;
    const int u = (t / a.GWo) * th + l / tw, v = (t % a.GWo) * tw + l % tw;
    if (u >= Ho || v >= Wo) continue;
    float sum = 0.0f;
    for (int z = 0; z < a.splits; ++z) sum = __fadd_rn(sum, a.ws[((int64_t)z * a.mcap + pm) * a.c_out + n]);
    if (a.bias) sum = __fadd_rn(sum, a.bias[n]);
    a.out.v[(int64_t)s * a.out.vs + n * plane + (int64_t)u * Wo + v] = sum;
  }
}

template <int BM, int BN, int TM, int TN>
static int launch_gemm(const GemmArgs& a, int64_t max_m, cudaStream_t st) {
  dim3 grid((unsigned)cdiv64(max_m, BM), (unsigned)cdiv(a.c_out, BN), (unsigned)a.splits);
  launch_pdl(k_conv_gemm<BM, BN, TM, TN>, dim3(grid), dim3((BM / TM) * (BN / TN)), 0, st, a);
  return 0;
}

}  // namespace evc

using namespace evc;

extern "C" {

int64_t evc_conv_workspace(const evc_conv_geom* g, int64_t max_tiles, int32_t splits) {
  if (!g || splits <= 1) return 0;
  return (int64_t)splits * max_tiles * g->th * g->tw * g->c_out;
}

int evc_conv_gemm(const evc_conv_geom* g, const evc_tensor* in, const float* weight, const float* wpack,
                  const float* bias, const evc_tensor* out, const int32_t* table, const int32_t* tile_list,
                  const int32_t* tile_count, int32_t S, int32_t splits, float* workspace, void* stream) {
  EVC_CHECK_ARG(g && in && out && (weight || wpack) && table && S > 0 && splits >= 1, "conv_gemm: null argument");
  EVC_CHECK_ARG(!tile_list || tile_count, "conv_gemm: tile_count required with tile_list");
  EVC_CHECK_ARG(splits == 1 || workspace, "conv_gemm: workspace required for split-K");
  GemmArgs a;
  a.in = view_of(*in);
  a.out = view_of(*out);
  a.w = weight;
  a.bias = bias;
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.kh = g->kh;
  a.kw = g->kw;
  a.stride = g->stride;
  a.pad = g->pad;
  a.K = g->c_in * g->kh * g->kw;
  a.kdec = table + tab_layout(g).kdec;
  a.list = tile_list;
  a.count = tile_count;
  a.T = a.out.GH * a.out.GW;
  a.GWo = a.out.GW;
  a.S = S;
  a.splits = splits;
  a.kchunk = (int)(cdiv64(cdiv64(a.K, splits), BK) * BK);
  a.ws = workspace;
  const int64_t max_m = (int64_t)S * a.T * g->th * g->tw;
  a.mcap = max_m;
  cudaStream_t st = as_stream(stream);
  if (wpack) {  // tcgen05 3xTF32 path (conv_tc.cu)
    const int eff = conv_tc_launch(g, in, wpack, bias, out, table, tile_list, tile_count, S, splits, workspace, st);
    EVC_CHECK_ARG(eff >= 1, "conv_gemm: unsupported tensor-core geometry");
    a.splits = eff;
    EVC_LAUNCH_CHECK("conv_gemm_tc");
  } else if (g->c_out > 24 && g->c_out <= 32) {
    launch_gemm<128, 32, 8, 4>(a, max_m, st);
  } else if (g->c_out > 32) {
    launch_gemm<128, 64, 8, 4>(a, max_m, st);
  } else if (g->c_out > 4) {
    launch_gemm<256, 16, 8, 4>(a, max_m, st);
  } else {
    launch_gemm<256, 4, 4, 2>(a, max_m, st);
  }
  EVC_LAUNCH_CHECK("conv_gemm");
  if (a.splits > 1) {
    const int64_t work = max_m * g->c_out;
    const int blocks = (int)std::min<int64_t>(cdiv64(work, 256), 148 * 8);
    launch_pdl(k_conv_splitk_reduce, dim3(blocks), dim3(256), 0, st, a);
    EVC_LAUNCH_CHECK("conv_splitk_reduce");
  }
  return EVC_OK;
}

}  // extern "C"

namespace evc {
int init_conv() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_conv_splitk_reduce) != cudaSuccess) return EVC_ECUDA;
  int rc = init_conv_mask();
  if (!rc) rc = init_conv_tc();
  if (!rc) rc = init_conv_fused();
  if (!rc) rc = init_conv_scatter();
  return rc ? rc : init_subpixel();
}
}  // namespace evc
