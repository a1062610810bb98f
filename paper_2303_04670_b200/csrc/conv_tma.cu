// TMA-fed tcgen05 implicit GEMM for the incremental / dense convolution.
//
// The conv input is mirrored into a channels-innermost ("HWC", channel count
// padded to a multiple of 4) shadow buffer by k_to_hwc.  M tile = a 4 x 32
// region of output pixels; one K-block = one tap (r, s) x 32 channels, and its
// A operand is exactly four TMA boxes of the shadow, one per output row:
//   box = [32 channels] x [32 pixels, traversal stride = conv stride] x [1 row] x [1 session]
// at (c0, x0*st - pad + s, (y0 + h)*st - pad + r, session).  TMA zero-fills
// out-of-range coordinates, which *is* the convolution's zero padding (and the
// channel tail).  With SWIZZLE_128B each box lands as 32 pixel rows of 128 B =
// the canonical K-major UMMA layout (8-row groups 1 KiB apart), so the four
// boxes form the 128 x 32 A tile directly: no gathers, no index tables.  (The
// channel start c0 is a multiple of 32, i.e. 128-byte aligned: TMA with a
// swizzle mode traps on an unaligned innermost start, which rules out the
// channel-planar layout for padded convs.)
//
// fp32 accuracy: 3xTF32 (hi*hi + hi*lo + lo*hi, fp32 TMEM accumulation); four
// "split" warps turn each landed box into hi (in place, rounded to TF32) and
// lo = x - hi (second buffer) with linear SMEM traffic -- the swizzle is
// layout-preserving.  Weights are pre-split, pre-swizzled K-major images
// streamed by cp.async.bulk.
//
// Roles (8 warps): warp 0 lane 0 = TMA producer; warp 1 = TMEM alloc + MMA
// issuer (lane 0); warps 4-7 = hi/lo split, then epilogue (TMEM lane quadrant =
// warp % 4 = output row of the region; lane = output column, so the CHW output
// stores are coalesced).

#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "conv_common.cuh"

namespace evc {

namespace tma {

constexpr int BM = 128;
constexpr int RH = 4, RW = 32;  // output region rows x cols
constexpr int THREADS = 256;

__host__ __device__ constexpr int bn_of(int c_out) {
  return c_out >= 256 ? 256 : (c_out <= 16 ? 16 : ((c_out + 15) / 16) * 16);
}
__host__ __device__ constexpr int stages_of(int bn) { return bn <= 64 ? 4 : (bn <= 128 ? 3 : 2); }
__host__ __device__ constexpr int stage_bytes(int bn) { return 2 * BM * 128 + 2 * bn * 128; }
static inline int smem_bytes(int bn) { return stages_of(bn) * stage_bytes(bn) + 1024 + 256; }

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void bar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bar_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "EVC_TW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra EVC_TW;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c, int x, int y, int n,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(x), "r"(y), "r"(n), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// K-major SWIZZLE_128B operand descriptor (sm_100 version 1, layout type 2, SBO 1 KiB).
__device__ __forceinline__ uint64_t desc_k(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
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
__device__ __forceinline__ float tf32_rn(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

struct Args {
  float* out;
  int64_t ovs;  // output session stride (floats)
  const float* wpack;
  const float* bias;
  const uint8_t* region_flags;  // [S][RHn*RWn], nullptr = every region (dense pass)
  float* ws;
  int64_t mcap;
  int c_in, c_out, kh, kw, stride, pad, cchunks, nkb;
  int Ho, Wo, RHn, RWn, S;
  int splits, kb_per_split;
};

template <int BN>
__global__ void __launch_bounds__(THREADS, 1) k_conv_tma(const __grid_constant__ CUtensorMap tmap, Args a) {
  constexpr int NS = stages_of(BN);
  constexpr int STAGE = stage_bytes(BN);
  // Accumulators: NA rotating "main" ones for hi*hi (one per K-block, round
  // robin) + one for the small hi*lo + lo*hi corrections, summed in fp32 (RN)
  // by the epilogue: every accumulator chain is NA-times (main) or ~2^11-times
  // (corrections) less exposed to the tensor core's accumulation rounding.
  constexpr int NA = BN >= 256 ? 1 : (BN >= 128 ? 3 : 4);
  constexpr int NEED = (NA + 1) * BN;
  constexpr int TMEM_COLS = NEED <= 32 ? 32 : (NEED <= 64 ? 64 : (NEED <= 128 ? 128 : (NEED <= 256 ? 256 : 512)));
  // kind::tf32, fp32 accumulate, A and B K-major, N = BN, M = 128
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
  constexpr uint32_t A_BYTES = BM * 128;  // 4 boxes of 32 pixels x 32 channels
  constexpr uint32_t B_BYTES = 2 * BN * 128;

  const int R = a.RHn * a.RWn;
  const int reg = blockIdx.x;  // s * R + region
  const int s = reg / R, rr = reg % R;
  if (a.region_flags && !a.region_flags[reg]) return;
  const int u0 = (rr / a.RWn) * RH, v0 = (rr % a.RWn) * RW;
  const int nblk = blockIdx.y, z = blockIdx.z;
  const int kb0 = z * a.kb_per_split, kb1 = min(a.nkb, kb0 + a.kb_per_split), nk = kb1 - kb0;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NS * STAGE);  // tma[NS], split[NS], empty[NS], acc
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3 * NS + 1);
  const uint32_t sb = su32(smem), b0 = su32(bars);
  auto tma_bar = [&](int i) { return b0 + 8u * i; };
  auto split_bar = [&](int i) { return b0 + 8u * (NS + i); };
  auto empty_bar = [&](int i) { return b0 + 8u * (2 * NS + i); };
  const uint32_t acc_bar = b0 + 8u * (3 * NS);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      bar_init(tma_bar(i), 1);
      bar_init(split_bar(i), 128);
      bar_init(empty_bar(i), 1);
    }
    bar_init(acc_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {  // ------------------------------------------------ TMA producer
      const char* wsrc = reinterpret_cast<const char*>(a.wpack) + (int64_t)nblk * a.nkb * B_BYTES;
      for (int i = 0; i < nk; ++i) {
        const int st = i % NS;
        bar_wait(empty_bar(st), ((i / NS) & 1) ^ 1);
        const int kb = kb0 + i;
        const int tap = kb / a.cchunks, c0 = (kb % a.cchunks) * 32;
        const int r = tap / a.kw, q = tap % a.kw;
        const uint32_t abuf = sb + st * STAGE;
        bar_arrive_tx(tma_bar(st), A_BYTES + B_BYTES);
#pragma unroll
        for (int h = 0; h < RH; ++h)
          tma_load_4d(abuf + h * 4096, &tmap, c0, v0 * a.stride - a.pad + q, (u0 + h) * a.stride - a.pad + r, s,
                      tma_bar(st));
        bulk_load(abuf + 2 * A_BYTES, wsrc + (int64_t)kb * B_BYTES, B_BYTES, tma_bar(st));
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------------ MMA issuer
      for (int i = 0; i < nk; ++i) {
        const int st = i % NS;
        bar_wait(split_bar(st), (i / NS) & 1);
        fence_after();
        const uint32_t ah = sb + st * STAGE, al = ah + A_BYTES;
        const uint32_t bh = ah + 2 * A_BYTES, bl = bh + BN * 128;
        const uint32_t tmain = tmem + (uint32_t)((i % NA) * BN), tcorr = tmem + (uint32_t)(NA * BN);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          const uint32_t ko = kk * 32;  // K=8 tf32 = 32 bytes inside the 128-byte swizzle row
          mma(tmain, desc_k(ah + ko), desc_k(bh + ko), IDESC, (i >= NA || kk) ? 1u : 0u);
          mma(tcorr, desc_k(ah + ko), desc_k(bl + ko), IDESC, (i | kk) ? 1u : 0u);
          mma(tcorr, desc_k(al + ko), desc_k(bh + ko), IDESC, 1u);
        }
        commit(empty_bar(st));
      }
      commit(acc_bar);
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ------------------------------------------------------------- hi/lo split
    const int t = threadIdx.x - 128;  // 0..127
    for (int i = 0; i < nk; ++i) {
      const int st = i % NS;
      bar_wait(tma_bar(st), (i / NS) & 1);
      float4* ah = reinterpret_cast<float4*>(smem + st * STAGE);
      float4* al = reinterpret_cast<float4*>(smem + st * STAGE + A_BYTES);
#pragma unroll
      for (int e = 0; e < (int)(A_BYTES / 16 / 128); ++e) {
        const int idx = t + e * 128;
        const float4 x = ah[idx];
        float4 h, l;
        h.x = tf32_rn(x.x);
        h.y = tf32_rn(x.y);
        h.z = tf32_rn(x.z);
        h.w = tf32_rn(x.w);
        l.x = __fsub_rn(x.x, h.x);
        l.y = __fsub_rn(x.y, h.y);
        l.z = __fsub_rn(x.z, h.z);
        l.w = __fsub_rn(x.w, h.w);
        ah[idx] = h;
        al[idx] = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(split_bar(st));
    }
    // ------------------------------------------------------------- epilogue
    const int qd = warp & 3;  // TMEM lanes 32*qd.. = region row qd
    const int u = u0 + qd, v = v0 + lane;
    bar_wait(acc_bar, 0);
    fence_after();
    const bool valid = u < a.Ho && v < a.Wo;
    const int64_t plane = (int64_t)a.Ho * a.Wo;
    const int64_t obase = (int64_t)s * a.ovs + (int64_t)u * a.Wo + v;
    const int64_t pm = (int64_t)reg * BM + qd * 32 + lane;
    const int n0 = nblk * BN;
    const int n_main = nk < NA ? nk : NA;
    const uint32_t trow = tmem + ((uint32_t)(32 * qd) << 16);
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float vals[16], part[16];
      tmem_ld16(trow + (uint32_t)(NA * BN + c0), vals);  // corrections
      for (int j = 0; j < n_main; ++j) {
        tmem_ld16(trow + (uint32_t)(j * BN + c0), part);
#pragma unroll
        for (int e = 0; e < 16; ++e) vals[e] = __fadd_rn(vals[e], part[e]);
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = n0 + c0 + j;
        if (n >= a.c_out) break;
        if (a.splits == 1) {
          if (valid) a.out[obase + n * plane] = a.bias ? __fadd_rn(vals[j], __ldg(a.bias + n)) : vals[j];
        } else {
          a.ws[((int64_t)z * a.mcap + pm) * a.c_out + n] = vals[j];
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

// split-K: sum the partials of each active region in a fixed order
__global__ void k_region_reduce(Args a) {
  const int R = a.RHn * a.RWn;
  const int64_t total = (int64_t)a.S * R * BM * a.c_out;
  const int64_t plane = (int64_t)a.Ho * a.Wo;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pm = e / a.c_out;
    const int n = (int)(e % a.c_out);
    const int reg = (int)(pm / BM), m = (int)(pm % BM);
    if (a.region_flags && !a.region_flags[reg]) continue;
    const int s = reg / R, rr = reg % R;
    const int u = (rr / a.RWn) * RH + m / 32, v = (rr % a.RWn) * RW + m % 32;
    if (u >= a.Ho || v >= a.Wo) continue;
    float sum = 0.0f;
    for (int zz = 0; zz < a.splits; ++zz) sum = __fadd_rn(sum, a.ws[((int64_t)zz * a.mcap + pm) * a.c_out + n]);
    if (a.bias) sum = __fadd_rn(sum, a.bias[n]);
    a.out[(int64_t)s * a.ovs + n * plane + (int64_t)u * a.Wo + v] = sum;
  }
}

// CHW -> channels-innermost shadow (channel stride cp), 32x32 tiles through SMEM
// so both the planar reads and the channel-contiguous writes are coalesced.
__global__ void __launch_bounds__(256) k_to_hwc(TView x, float* __restrict__ y, int64_t ys, int cp) {
  __shared__ float t[32][33];
  const int HW = x.H * x.W;
  const int p0 = blockIdx.x * 32, c0 = blockIdx.y * 32, s = blockIdx.z;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const float* src = x.v + (int64_t)s * x.vs;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = c0 + ty + 8 * k, p = p0 + tx;
    t[ty + 8 * k][tx] = (c < x.C && p < HW) ? src[(int64_t)c * HW + p] : 0.0f;
  }
  __syncthreads();
  float* dst = y + (int64_t)s * ys;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int p = p0 + ty + 8 * k, c = c0 + tx;
    if (p < HW && c < x.C) dst[(int64_t)p * cp + c] = t[tx][ty + 8 * k];
  }
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiled encoder() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}

template <int BN>
static void launch(const CUtensorMap& m, const Args& a, int nb, cudaStream_t st) {
  dim3 grid((unsigned)(a.S * a.RHn * a.RWn), (unsigned)nb, (unsigned)a.splits);
  k_conv_tma<BN><<<grid, THREADS, smem_bytes(BN), st>>>(m, a);
}

template <int BN>
static int attr() {
  return cudaFuncSetAttribute(k_conv_tma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes(BN)) ==
                 cudaSuccess
             ? 0
             : 1;
}

}  // namespace tma

int init_conv_tma() {
  int rc = 0;
  rc |= tma::attr<16>() | tma::attr<32>() | tma::attr<48>() | tma::attr<64>() | tma::attr<80>() | tma::attr<96>();
  rc |= tma::attr<112>() | tma::attr<128>() | tma::attr<144>() | tma::attr<160>() | tma::attr<176>();
  rc |= tma::attr<192>() | tma::attr<208>() | tma::attr<224>() | tma::attr<240>() | tma::attr<256>();
  return rc ? EVC_ECUDA : EVC_OK;
}

}  // namespace evc

using namespace evc;

extern "C" {

int32_t evc_hwc_channels(int32_t c) { return (c + 3) / 4 * 4; }

int evc_to_hwc(const evc_tensor* x, float* y, int64_t y_stride, int32_t cp, int32_t S, void* stream) {
  EVC_CHECK_ARG(x && x->vals && y && S > 0 && cp >= x->C, "to_hwc: bad argument");
  TView v = view_of(*x);
  dim3 grid(cdiv(v.H * v.W, 32), cdiv(v.C, 32), S);
  tma::k_to_hwc<<<grid, 256, 0, as_stream(stream)>>>(v, y, y_stride, cp);
  EVC_LAUNCH_CHECK("to_hwc");
  return EVC_OK;
}

int evc_conv_region_supported(const evc_conv_geom* g) {
  if (!g) return 0;
  return g->stride >= 1 && g->stride * tma::RW <= 256 && g->stride <= 8 && tma::encoder() != nullptr;
}

int evc_conv_region_grid(const evc_conv_geom* g, int32_t* rh, int32_t* rw) {
  EVC_CHECK_ARG(g && rh && rw, "conv_region_grid: null argument");
  *rh = (g->Ho + tma::RH - 1) / tma::RH;
  *rw = (g->Wo + tma::RW - 1) / tma::RW;
  return EVC_OK;
}

int64_t evc_conv_region_pack_len(int32_t c_out, int32_t c_in, int32_t kh, int32_t kw) {
  const int bn = tma::bn_of(c_out);
  const int64_t nb = (c_out + bn - 1) / bn, nkb = (int64_t)kh * kw * ((c_in + 31) / 32);
  return nb * nkb * 2 * bn * 32;
}

int evc_conv_region_pack(const float* w, int32_t c_out, int32_t c_in, int32_t kh, int32_t kw, float* out) {
  EVC_CHECK_ARG(w && out && c_out > 0 && c_in > 0, "conv_region_pack: bad argument");
  const int bn = tma::bn_of(c_out);
  const int cch = (c_in + 31) / 32;
  const int64_t nb = (c_out + bn - 1) / bn, nkb = (int64_t)kh * kw * cch;
  for (int64_t b = 0; b < nb; ++b)
    for (int64_t kb = 0; kb < nkb; ++kb) {
      const int tap = (int)(kb / cch), c0 = (int)(kb % cch) * 32;
      const int r = tap / kw, q = tap % kw;
      float* hi = out + ((b * nkb + kb) * 2) * bn * 32;
      float* lo = hi + (int64_t)bn * 32;
      for (int row = 0; row < bn; ++row)
        for (int e = 0; e < 32; ++e) {
          const int64_t n = b * bn + row;
          const int c = c0 + e;
          const float x = (n < c_out && c < c_in) ? w[((n * c_in + c) * kh + r) * kw + q] : 0.0f;
          uint32_t bits;
          memcpy(&bits, &x, 4);
          bits = (bits + 0x1000u) & 0xFFFFE000u;  // round to nearest TF32 (as tf32_rn)
          float h;
          memcpy(&h, &bits, 4);
          // 128B swizzle: 16-byte chunk j of row `row` lives at chunk (j ^ (row & 7))
          const int j = e / 4, sub = e % 4;
          const int64_t pos = (int64_t)row * 32 + ((j ^ (row & 7)) * 4) + sub;
          hi[pos] = h;
          lo[pos] = x - h;
        }
    }
  return EVC_OK;
}

int64_t evc_conv_region_workspace(const evc_conv_geom* g, int32_t S, int32_t splits) {
  if (!g || splits <= 1) return 0;
  const int64_t R = (int64_t)((g->Ho + tma::RH - 1) / tma::RH) * ((g->Wo + tma::RW - 1) / tma::RW);
  return (int64_t)splits * S * R * tma::BM * g->c_out;
}

int evc_conv_gemm_region(const evc_conv_geom* g, const float* in_hwc, int32_t cp, int64_t hwc_stride,
                         const float* wpack, const float* bias, const evc_tensor* out, const uint8_t* region_flags,
                         int32_t S, int32_t splits, float* workspace, void* stream) {
  EVC_CHECK_ARG(g && in_hwc && out && wpack && S > 0 && splits >= 1, "conv_gemm_region: null argument");
  EVC_CHECK_ARG(evc_conv_region_supported(g), "conv_gemm_region: unsupported geometry");
  EVC_CHECK_ARG(cp % 4 == 0 && cp >= g->c_in && hwc_stride % 4 == 0, "conv_gemm_region: shadow not 16B aligned");
  EVC_CHECK_ARG(splits == 1 || workspace, "conv_gemm_region: workspace required for split-K");
  tma::EncodeTiled enc = tma::encoder();
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)cp, (cuuint64_t)g->W, (cuuint64_t)g->H, (cuuint64_t)S};
  const cuuint64_t strides[3] = {(cuuint64_t)cp * 4, (cuuint64_t)g->W * cp * 4, (cuuint64_t)hwc_stride * 4};
  const cuuint32_t box[4] = {32, (cuuint32_t)(tma::RW * g->stride), 1, 1};
  const cuuint32_t estr[4] = {1, (cuuint32_t)g->stride, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(in_hwc), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("evc: conv_gemm_region: cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return EVC_ECUDA;
  }
  tma::Args a;
  a.out = out->vals;
  a.ovs = out->vstride;
  a.wpack = wpack;
  a.bias = bias;
  a.region_flags = region_flags;
  a.ws = workspace;
  a.c_in = g->c_in;
  a.c_out = g->c_out;
  a.kh = g->kh;
  a.kw = g->kw;
  a.stride = g->stride;
  a.pad = g->pad;
  a.cchunks = (g->c_in + 31) / 32;
  a.nkb = g->kh * g->kw * a.cchunks;
  a.Ho = g->Ho;
  a.Wo = g->Wo;
  a.RHn = (g->Ho + tma::RH - 1) / tma::RH;
  a.RWn = (g->Wo + tma::RW - 1) / tma::RW;
  a.S = S;
  a.splits = std::max(1, std::min<int>(splits, a.nkb));
  a.kb_per_split = (a.nkb + a.splits - 1) / a.splits;
  a.splits = (a.nkb + a.kb_per_split - 1) / a.kb_per_split;
  a.mcap = (int64_t)S * a.RHn * a.RWn * tma::BM;
  const int bn = tma::bn_of(g->c_out);
  const int nb = (g->c_out + bn - 1) / bn;
  cudaStream_t st = as_stream(stream);
  switch (bn) {
#define EVC_TMA_CASE(B) \
  case B:               \
    tma::launch<B>(map, a, nb, st); \
    break;
    EVC_TMA_CASE(16) EVC_TMA_CASE(32) EVC_TMA_CASE(48) EVC_TMA_CASE(64) EVC_TMA_CASE(80) EVC_TMA_CASE(96)
    EVC_TMA_CASE(112) EVC_TMA_CASE(128) EVC_TMA_CASE(144) EVC_TMA_CASE(160) EVC_TMA_CASE(176) EVC_TMA_CASE(192)
    EVC_TMA_CASE(208) EVC_TMA_CASE(224) EVC_TMA_CASE(240) EVC_TMA_CASE(256)
#undef EVC_TMA_CASE
    default:
      set_error("evc: conv_gemm_region: bad N tile");
      return EVC_EINVAL;
  }
  EVC_LAUNCH_CHECK("conv_gemm_region");
  if (a.splits > 1) {
    const int64_t work = a.mcap * g->c_out;
    const int blocks = (int)std::min<int64_t>(cdiv64(work, 256), 148 * 8);
    tma::k_region_reduce<<<blocks, 256, 0, st>>>(a);
    EVC_LAUNCH_CHECK("conv_region_reduce");
  }
  return EVC_OK;
}

}  // extern "C"
