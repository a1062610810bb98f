// tcgen05 (5th-gen tensor core) implicit-GEMM for the incremental convolution.
//
// D[m, n] = sum_k A[m, k] * B[n, k]   with   m = packed site of an active output
// tile (evc_conv_mask work list), k = (c, r, s) im2col index, B = the weight in
// the reference layout (C_out, C_in*KH*KW) (graph.py:457-467).
//
// fp32 accuracy on TF32 tensor cores (hard part 1): every
// operand is split x = hi + lo with hi = x with the low 13 mantissa bits cleared
// (exact in TF32) and lo = x - hi, and each K=8 step issues three
// tcgen05.mma.kind::tf32: hi*hi + hi*lo + lo*hi into one fp32 TMEM accumulator.
//
// CTA = 8 warps:
//   warps 0-3  producers: each thread owns one of the 128 tile rows, gathers its
//              32 k-values per K-block from the channel-planar input, splits them
//              and writes both halves into 128B-swizzled K-major SMEM; thread 0
//              also streams the pre-split, pre-swizzled weight block with
//              cp.async.bulk (mbarrier complete_tx).
//   warp 4     TMEM allocator + single-thread MMA issuer, then epilogue.
//   warps 4-7  epilogue: tcgen05.ld 32x32b rows of the accumulator -> scatter to
//              the (C,H,W) output (or the split-K workspace).
// Stages are an mbarrier ring: full[s] (128 producer arrivals + weight bytes),
// empty[s] (tcgen05.commit of the MMAs that read the stage).

#include <algorithm>

#include "conv_common.cuh"

namespace evc {

constexpr int TC_BM = 128;
constexpr int TC_BK = 32;  // tf32 elements per 128-byte swizzle row
constexpr int TC_THREADS = 256;

__host__ __device__ constexpr int tc_bn(int c_out) {
  return c_out >= 256 ? 256 : (c_out <= 16 ? 16 : ((c_out + 15) / 16) * 16);
}
__host__ __device__ constexpr int tc_stages(int bn) { return bn <= 64 ? 4 : (bn <= 128 ? 3 : 2); }
__host__ __device__ constexpr int tc_stage_bytes(int bn) { return 2 * TC_BM * 128 + 2 * bn * 128; }
static inline int tc_smem_bytes(int bn) { return tc_stages(bn) * tc_stage_bytes(bn) + 1024 + 256; }

// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "EVC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra EVC_WAIT;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// K-major, 128B-swizzled operand: 8-row core groups 1024 B apart (SBO), LBO unused (1),
// version 1 (sm_100), layout type 2 = SWIZZLE_128B.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// hi = x rounded to the nearest TF32 (ties away from zero), exactly representable
// in TF32; lo = x - hi is exact in fp32 and |lo| <= 2^-11 |x|.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------
struct TcArgs {
  TView in, out;
  const float* wpack;  // [n_blocks][nkb][hi|lo][BN][32] swizzled images
  const float* bias;
  const int32_t* kdec;
  const int32_t* list;
  const int32_t* count;
  float* ws;
  int64_t mcap;
  int c_in, c_out, stride, pad, K, nkb;
  int T, GWo, S;
  int splits, kb_per_split;
};

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1) k_conv_tc(TcArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int NS = tc_stages(BN);
  constexpr int STAGE = tc_stage_bytes(BN);
  constexpr int TMEM_COLS = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);

  const int th = a.out.th, tw = a.out.tw, sites = th * tw;
  const int n_tiles = a.list ? *a.count : a.S * a.T;
  const int64_t M = (int64_t)n_tiles * sites;
  const int64_t m0 = (int64_t)blockIdx.x * TC_BM;
  if (m0 >= M) return;
  const int nblk = blockIdx.y;
  const int z = blockIdx.z;
  const int kb0 = z * a.kb_per_split;
  const int kb1 = min(a.nkb, kb0 + a.kb_per_split);
  const int nk = kb1 - kb0;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * STAGE);  // full[NS], empty[NS], accf
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 1);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (NS + s); };
  const uint32_t acc_bar = bar0 + 8u * (2 * NS);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(full_bar(s), 128);
      mbar_init(empty_bar(s), 1);
    }
    mbar_init(acc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 4) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int H = a.in.H, W = a.in.W, Ho = a.out.H, Wo = a.out.W;
  // site of tile row `m` (producers: own row; epilogue: row 32*(warp%4)+lane)
  auto site = [&](int m, int64_t& in_off, int& y0, int& x0, int64_t& out_off) {
    const int64_t pm = m0 + m;
    in_off = 0;
    out_off = -1;
    y0 = -(1 << 20);
    x0 = -(1 << 20);
    if (pm >= M) return;
    const int e = (int)(pm / sites), l = (int)(pm % sites);
    const int ent = a.list ? a.list[e] : e;
    const int s = ent / a.T, t = ent % a.T;
    const int u = (t / a.GWo) * th + l / tw, v = (t % a.GWo) * tw + l % tw;
    if (u >= Ho || v >= Wo) return;
    out_off = (int64_t)s * a.out.vs + (int64_t)u * Wo + v;
    y0 = u * a.stride - a.pad;
    x0 = v * a.stride - a.pad;
    in_off = (int64_t)s * a.in.vs + (int64_t)y0 * W + x0;
  };

  if (warp < 4) {
    // ------------------------------------------------------------ producers
    const int m = threadIdx.x;
    int64_t in_off, out_off;
    int y0, x0;
    site(m, in_off, y0, x0, out_off);
    const float* src = a.in.v + in_off;
    const uint32_t row_off = (uint32_t)m * 128u;
    const uint32_t sw = (uint32_t)(m & 7);
    const char* wsrc = reinterpret_cast<const char*>(a.wpack) + ((int64_t)nblk * a.nkb) * (2 * BN * 128);
    for (int i = 0; i < nk; ++i) {
      const int st = i % NS;
      const uint32_t par = ((i / NS) & 1) ^ 1;
      mbar_wait(empty_bar(st), par);
      const uint32_t abase = sbase + st * STAGE;
      const int kb = kb0 + i;
      float v[TC_BK];
#pragma unroll
      for (int e = 0; e < TC_BK; ++e) {
        const int k = kb * TC_BK + e;
        float x = 0.0f;
        if (k < a.K) {
          const int off = __ldg(a.kdec + 2 * k), rq = __ldg(a.kdec + 2 * k + 1);
          const int iy = y0 + (rq >> 16), ix = x0 + (rq & 0xffff);
          if ((unsigned)iy < (unsigned)H && (unsigned)ix < (unsigned)W) x = __ldg(src + off);
        }
        v[e] = x;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 hi, lo;
        hi.x = tf32_hi(v[4 * j + 0]);
        hi.y = tf32_hi(v[4 * j + 1]);
        hi.z = tf32_hi(v[4 * j + 2]);
        hi.w = tf32_hi(v[4 * j + 3]);
        lo.x = __fsub_rn(v[4 * j + 0], hi.x);
        lo.y = __fsub_rn(v[4 * j + 1], hi.y);
        lo.z = __fsub_rn(v[4 * j + 2], hi.z);
        lo.w = __fsub_rn(v[4 * j + 3], hi.w);
        const uint32_t off = row_off + ((((uint32_t)j) ^ sw) << 4);
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(abase + off), "f"(hi.x), "f"(hi.y),
                     "f"(hi.z), "f"(hi.w)
                     : "memory");
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(abase + TC_BM * 128 + off), "f"(lo.x),
                     "f"(lo.y), "f"(lo.z), "f"(lo.w)
                     : "memory");
      }
      fence_async_smem();  // make the generic-proxy SMEM writes visible to the tensor core
      if (threadIdx.x == 0) {
        mbar_arrive_tx(full_bar(st), 2 * BN * 128);
        bulk_g2s(abase + 2 * TC_BM * 128, wsrc + (int64_t)kb * (2 * BN * 128), 2 * BN * 128, full_bar(st));
      } else {
        mbar_arrive(full_bar(st));
      }
    }
  } else {
    if (warp == 4 && lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      for (int i = 0; i < nk; ++i) {
        const int st = i % NS;
        mbar_wait(full_bar(st), (i / NS) & 1);
        tc_fence_after();
        const uint32_t abase = sbase + st * STAGE;
        const uint32_t a_hi = abase, a_lo = abase + TC_BM * 128;
        const uint32_t b_hi = abase + 2 * TC_BM * 128, b_lo = b_hi + BN * 128;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 8; ++kk) {
          const uint32_t ko = kk * 32;  // 8 tf32 = 32 bytes along K inside the swizzle atom
          mma_tf32(tmem, sdesc(a_hi + ko), sdesc(b_hi + ko), IDESC, (i | kk) ? 1u : 0u);
          mma_tf32(tmem, sdesc(a_hi + ko), sdesc(b_lo + ko), IDESC, 1u);
          mma_tf32(tmem, sdesc(a_lo + ko), sdesc(b_hi + ko), IDESC, 1u);
        }
        tc_commit(empty_bar(st));  // frees the stage once these MMAs have read it
      }
      tc_commit(acc_bar);
    }
    __syncwarp();
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3;
    const int m = 32 * q + lane;
    int64_t in_off, out_off;
    int y0, x0;
    site(m, in_off, y0, x0, out_off);
    mbar_wait(acc_bar, 0);
    tc_fence_after();
    const int64_t plane = (int64_t)Ho * Wo;
    const int n0 = nblk * BN;
    const int64_t pm = m0 + m;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)c0, v);
      if (pm < M) {
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          const int n = n0 + c0 + jj;
          if (n >= a.c_out) break;
          if (a.splits == 1) {
            if (out_off >= 0) a.out.v[out_off + n * plane] = a.bias ? __fadd_rn(v[jj], __ldg(a.bias + n)) : v[jj];
          } else {
            a.ws[((int64_t)z * a.mcap + pm) * a.c_out + n] = v[jj];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

template <int BN>
static int launch_tc(const TcArgs& a, int64_t max_m, int n_blocks, cudaStream_t st) {
  dim3 grid((unsigned)cdiv64(max_m, TC_BM), (unsigned)n_blocks, (unsigned)a.splits);
  launch_pdl(k_conv_tc<BN>, dim3(grid), dim3(TC_THREADS), tc_smem_bytes(BN), st, a);
  return 0;
}

template <int BN>
static int set_attr() {
  return cudaFuncSetAttribute(k_conv_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc_smem_bytes(BN)) ==
                 cudaSuccess
             ? 0
             : -1;
}

int init_conv_tc() {
  int rc = 0;
  rc |= set_attr<16>();
  rc |= set_attr<32>();
  rc |= set_attr<48>();
  rc |= set_attr<64>();
  rc |= set_attr<80>();
  rc |= set_attr<96>();
  rc |= set_attr<112>();
  rc |= set_attr<128>();
  rc |= set_attr<144>();
  rc |= set_attr<160>();
  rc |= set_attr<176>();
  rc |= set_attr<192>();
  rc |= set_attr<208>();
  rc |= set_attr<224>();
  rc |= set_attr<240>();
  rc |= set_attr<256>();
  return rc ? EVC_ECUDA : EVC_OK;
}

int conv_tc_launch(const evc_conv_geom* g, const evc_tensor* in, const float* wpack, const float* bias,
                   const evc_tensor* out, const int32_t* table, const int32_t* tile_list, const int32_t* tile_count,
                   int32_t S, int32_t splits, float* workspace, cudaStream_t st) {
  TcArgs a;
  a.in = view_of(*in);
  a.out = view_of(*out);
  a.wpack = wpack;
  a.bias = bias;
  a.kdec = table + tab_layout(g).kdec;
  a.list = tile_list;
  a.count = tile_count;
  a.ws = workspace;
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.stride = g->stride;
  a.pad = g->pad;
  a.K = g->c_in * g->kh * g->kw;
  a.nkb = (a.K + TC_BK - 1) / TC_BK;
  a.T = a.out.GH * a.out.GW;
  a.GWo = a.out.GW;
  a.S = S;
  a.splits = std::max(1, std::min<int>(splits, a.nkb));
  a.kb_per_split = (a.nkb + a.splits - 1) / a.splits;
  a.splits = (a.nkb + a.kb_per_split - 1) / a.kb_per_split;
  const int64_t max_m = (int64_t)S * a.T * g->th * g->tw;
  a.mcap = max_m;
  const int bn = tc_bn(g->c_out);
  const int nb = (g->c_out + bn - 1) / bn;
  switch (bn) {
#define EVC_TC_CASE(B) \
  case B:              \
    launch_tc<B>(a, max_m, nb, st); \
    break;
    EVC_TC_CASE(16) EVC_TC_CASE(32) EVC_TC_CASE(48) EVC_TC_CASE(64) EVC_TC_CASE(80) EVC_TC_CASE(96)
    EVC_TC_CASE(112) EVC_TC_CASE(128) EVC_TC_CASE(144) EVC_TC_CASE(160) EVC_TC_CASE(176) EVC_TC_CASE(192)
    EVC_TC_CASE(208) EVC_TC_CASE(224) EVC_TC_CASE(240) EVC_TC_CASE(256)
#undef EVC_TC_CASE
    default:
      return EVC_EINVAL;
  }
  return a.splits;
}

}  // namespace evc

using namespace evc;

extern "C" {

int64_t evc_conv_tc_pack_len(int32_t c_out, int64_t K) {
  const int bn = tc_bn(c_out);
  const int64_t nb = (c_out + bn - 1) / bn, nkb = (K + TC_BK - 1) / TC_BK;
  return nb * nkb * 2 * bn * TC_BK;
}

int evc_conv_tc_pack(const float* w, int32_t c_out, int64_t K, float* out) {
  EVC_CHECK_ARG(w && out && c_out > 0 && K > 0, "conv_tc_pack: bad argument");
  const int bn = tc_bn(c_out);
  const int64_t nb = (c_out + bn - 1) / bn, nkb = (K + TC_BK - 1) / TC_BK;
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t kb = 0; kb < nkb; ++kb) {
      float* hi = out + ((b * nkb + kb) * 2) * bn * TC_BK;
      float* lo = hi + (int64_t)bn * TC_BK;
      for (int r = 0; r < bn; ++r)
        for (int e = 0; e < TC_BK; ++e) {
          const int64_t n = b * bn + r, k = kb * TC_BK + e;
          const float x = (n < c_out && k < K) ? w[n * K + k] : 0.0f;
          uint32_t bits;
          memcpy(&bits, &x, 4);
          bits = (bits + 0x1000u) & 0xFFFFE000u;  // round to nearest TF32, as tf32_hi()
          float h;
          memcpy(&h, &bits, 4);
          // 128B swizzle: 16-byte chunk j of row r lives at chunk (j ^ (r & 7))
          const int j = e / 4, sub = e % 4;
          const int64_t pos = (int64_t)r * TC_BK + ((j ^ (r & 7)) * 4) + sub;
          hi[pos] = h;
          lo[pos] = x - h;
        }
    }
  return EVC_OK;
}

}  // extern "C"
