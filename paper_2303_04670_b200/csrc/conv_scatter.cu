// Input-stationary incremental convolution: gather -> tcgen05 GEMM -> deterministic scatter-add.
//
// The fused conv (conv_fused.cu) is output-stationary: it computes whole 128-site output regions
// around every live input tile, so with a 3x3 kernel and 6x6 tiles an isolated live tile costs ~9
// tiles of output work and, at 20 % clustered density, ~87 % of the output regions are live.  The
// reference meter (increment_ops.py:156-194) charges only the live input tiles.  This path does the
// same amount of work as the meter:
//
//  1. live input tiles (any channel, evc_tile_any) are compacted (evc_compact: warp ballot + block
//     scan, ascending = np.flatnonzero) and a tile -> list index map is built;
//  2. k_conv_scatter: a unit = 3 live tiles x 16 output channels.  Producer warps gather each tile's
//     6x6 pixels x 32 input channels straight from the channel-planar increment, split them into
//     TF32 heads / tails and store them as a 128B-swizzled K-major A tile (40 rows per tile slot);
//     the weights of all kh x kw taps sit side by side along N (N = taps x 16 = 144), so ONE MMA per
//     K8 step computes every tap's contribution of every input site (3xTF32: hi.hi + hi.lo + lo.hi,
//     fp32 accumulate in TMEM, double-buffered across units).  The epilogue warps add the tap
//     columns of each site into an (th + kh - 1) x (tw + kw - 1) output patch in shared memory, tap
//     by tap (within a tap every site lands on a distinct position: no atomics), and store the patch;
//  3. k_scatter_gather: every output tile sums the patches of its (up to) 9 live neighbour input
//     tiles in a fixed order -- deterministic, no atomics -- and writes its 6x6 x C_out values; a
//     tile that was live last step and is dead now is written with exact zeros (TileMask soundness).
//
// Output flags and the FLOP meter are the unfused path's (evc_conv_mask), run by the caller.
// Geometry: stride 1, kh * 16 * kw <= 256, tiles th * tw <= 36 (th, tw <= 6 + ...).

#include <algorithm>

#include "conv_common.cuh"
#include "tcgen05.cuh"

#ifndef EVC_MMA_WARP
#define EVC_MMA_WARP 1  // as conv_fused.cu: the MMA warp walks its loop converged, one elected lane issues
#endif

namespace evc {
namespace sc {

using namespace fz;

constexpr int BNB = 16;      // output channels per unit
constexpr int SLOT = 40;     // A rows (TMEM lanes) per tile slot: th * tw <= 36 sites, five 8-row groups
constexpr int TPU = 3;       // tiles per group (120 of 128 rows)
constexpr int NS = 2;        // weight pipeline stages
constexpr int A_KB = 2 * 128 * 128;  // one K-block of the resident A tile: heads + tails, 128 rows x 128 B
constexpr int MAX_KB = 2;    // resident A: C_in <= 64
constexpr int THREADS = 448;  // warps 0-3 gather, 4-11 epilogue, 12 TMEM alloc + MMA issuer, 13 weight stream
constexpr int EPI = 256;      // epilogue threads (two warps per TMEM lane quarter)

struct ScArgs {
  const float* in;
  int64_t in_vs;
  int C, H, W, th, tw, GH, GW;
  int kh, kw, pad, taps;
  int c_out, nb, nkb, b_half;
  int PH, PW;
  const float* wpack;
  const int32_t* list;
  const int32_t* count;
  float* contrib;
};

__device__ __forceinline__ void sync_epi() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// One CTA walks tile groups (3 live input tiles); per group the gather warps stage the A tile of
// every K-block once (resident), and the MMA issuer runs all output-channel blocks over it, each
// into a double-buffered TMEM accumulator that the epilogue warps scatter into output patches.
template <int K, int T>
__global__ void __launch_bounds__(THREADS, 1) k_conv_scatter(const __grid_constant__ ScArgs a) {
  // compile-time geometry: every index decode below is shifts / multiplies
  constexpr int TAPS = K * K, PH = T + K - 1, PW = T + K - 1, SITES = T * T, PPT = PH * PW;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int N = TAPS * BNB;
  const uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int BSTAGE = (2 * a.b_half + 1023) / 1024 * 1024;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* bst = smem + a.nkb * A_KB;  // weight stages
  float* Dsm = reinterpret_cast<float*>(bst + NS * BSTAGE);  // accumulator stage [column][TMEM lane]
  constexpr int PSZ = PPT * BNB;  // floats per tile patch
  uint64_t* bars = reinterpret_cast<uint64_t*>(Dsm + 128 * N);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 2 * NS + 6);
  const uint32_t sA = su32(smem), sB = su32(bst), b0 = su32(bars);
  auto bfull = [&](int i) { return b0 + 8u * i; };
  auto bempty = [&](int i) { return b0 + 8u * (NS + i); };
  auto tfull = [&](int i) { return b0 + 8u * (2 * NS + i); };
  auto tempty = [&](int i) { return b0 + 8u * (2 * NS + 2 + i); };
  const uint32_t afull = b0 + 8u * (2 * NS + 4), aempty = b0 + 8u * (2 * NS + 5);

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      bar_init(bfull(i), 1);
      bar_init(bempty(i), 1);
    }
    for (int i = 0; i < 2; ++i) {
      bar_init(tfull(i), 1);
      bar_init(tempty(i), EPI);
    }
    bar_init(afull, 128);
    bar_init(aempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 12) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  pdl_trigger();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tslot;
  pdl_wait();
  const int n_live = *a.count;
  const int ngroups = (n_live + TPU - 1) / TPU;
  const int Ti = a.GH * a.GW;

  if (warp < 4) {  // ------------------------------------------------------------ A gather
    const int tid = threadIdx.x;
    constexpr int BATCH = 9;  // independent loads in flight per thread
    int q = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++q) {
      int tile_s[TPU], tile_y[TPU], tile_x[TPU];
#pragma unroll
      for (int j = 0; j < TPU; ++j) {
        const int li = g * TPU + j;
        tile_s[j] = -1;
        tile_y[j] = tile_x[j] = 0;
        if (li < n_live) {
          const int t = a.list[li];
          tile_s[j] = t / Ti;
          const int r = t - tile_s[j] * Ti;
          tile_y[j] = (r / a.GW) * T;
          tile_x[j] = (r % a.GW) * T;
        }
      }
      if (q >= 1) bar_wait(aempty, (q - 1) & 1);  // every MMA over the previous group's A is done
      // element e = ((j * 32 + c) * th + y) * tw + x  (x fastest: short coalesced runs)
      constexpr int per = TPU * 32 * SITES;
      for (int kb = 0; kb < a.nkb; ++kb) {
        float* Ah = reinterpret_cast<float*>(smem + kb * A_KB);
        float* Al = Ah + 128 * 32;
#pragma unroll 1
        for (int e0 = tid; e0 < per; e0 += 128 * BATCH) {
          float v[BATCH];
#pragma unroll
          for (int k = 0; k < BATCH; ++k) {
            const int e = e0 + 128 * k;
            v[k] = 0.0f;
            if (e < per) {
              const int x = e % T, y = (e / T) % T, c = (e / SITES) % 32, j = e / (32 * SITES);
              const int ch = kb * 32 + c, py = tile_y[j] + y, px = tile_x[j] + x;
              if (tile_s[j] >= 0 && ch < a.C && py < a.H && px < a.W)
                v[k] = __ldg(a.in + (int64_t)tile_s[j] * a.in_vs + ((int64_t)ch * a.H + py) * a.W + px);
            }
          }
#pragma unroll
          for (int k = 0; k < BATCH; ++k) {
            const int e = e0 + 128 * k;
            if (e < per) {
              const int x = e % T, y = (e / T) % T, c = (e / SITES) % 32, j = e / (32 * SITES);
              const int row = j * SLOT + y * T + x;
              const int off = row * 32 + (((c >> 2) ^ (row & 7)) << 2) + (c & 3);  // 128B swizzle (floats)
              const float hi = tf32_head(v[k]);
              Ah[off] = hi;
              Al[off] = __fsub_rn(v[k], hi);
            }
          }
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bar_arrive(afull);
    }
  } else if (warp == 13) {  // ---------------------------------------------------- weight stream
    if (lane == 0) {
      int it = 0;
      for (int g = blockIdx.x; g < ngroups; g += gridDim.x)
        for (int nb = 0; nb < a.nb; ++nb)
          for (int kb = 0; kb < a.nkb; ++kb, ++it) {
            const int st = it % NS;
            if (it >= NS) bar_spin(bempty(st), ((it / NS) & 1) ^ 1);
            bar_arrive_tx(bfull(st), 2u * a.b_half);
            bulk_load(sB + st * BSTAGE, reinterpret_cast<const char*>(a.wpack) + ((int64_t)nb * a.nkb + kb) * 2 * a.b_half,
                      2u * a.b_half, bfull(st));
          }
    }
    __syncwarp();
  } else if (warp == 12) {  // ------------------------------------------------------ MMA issuer
#if EVC_MMA_WARP
#define MMA_ mma_w
#define COMMIT_ commit_w
#else
#define MMA_ mma
#define COMMIT_ commit
#endif
    if (EVC_MMA_WARP || lane == 0) {  // (warp-wide: every lane walks the loop, one elected lane issues)
      int it = 0, u = 0, q = 0;
      for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++q) {
        bar_spin(afull, q & 1);
        fence_after();
        for (int nb = 0; nb < a.nb; ++nb, ++u) {
          const int ab = u & 1;
          if (u >= 2) bar_spin(tempty(ab), ((u >> 1) & 1) ^ 1);
          fence_after();
          const uint32_t d = tmem + (uint32_t)(ab * 256);
          for (int kb = 0; kb < a.nkb; ++kb, ++it) {
            const int st = it % NS;
            bar_spin(bfull(st), (it / NS) & 1);
            fence_after();
            const uint32_t ah = sA + kb * A_KB, al = ah + 128 * 128, bh = sB + st * BSTAGE, bl = bh + a.b_half;
            const uint64_t dah = desc_k(ah), dal = desc_k(al), dbh = desc_k(bh), dbl = desc_k(bl);
            const int nkk = min(4, (a.C - kb * 32 + 7) >> 3);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              if (kk >= nkk) break;
              MMA_(d, dah + 2 * kk, dbh + 2 * kk, IDESC, (kb || kk) ? 1u : 0u);  // hi.hi
              MMA_(d, dah + 2 * kk, dbl + 2 * kk, IDESC, 1u);                    // hi.lo
              MMA_(d, dal + 2 * kk, dbh + 2 * kk, IDESC, 1u);                    // lo.hi
            }
            COMMIT_(bempty(st));
          }
          COMMIT_(tfull(ab));
        }
        COMMIT_(aempty);  // the gather may overwrite A once these MMAs have completed
      }
    }
    __syncwarp();
#undef MMA_
#undef COMMIT_
  } else {  // ---------------------------------------------------------------------- epilogue
    // per unit: the accumulator (site x [tap][16 channels]) goes TMEM -> shared memory, then every
    // thread forms output patch points: patch point (py, px) of tile j, channel n sums, in tap
    // order, D[site (py + r - kh + 1, px + q - kw + 1)][tap (r, q)][n] -- a gather, no atomics
    const int etid = threadIdx.x - 128;
    const int m = 32 * (warp & 3) + lane;  // TMEM lane = A row
    const int half = (warp - 4) >> 2;      // the two warps of a lane quarter split the taps
    const uint32_t trow = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    int u = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
      const int ntile = min(TPU, n_live - g * TPU);
      for (int nb = 0; nb < a.nb; ++nb, ++u) {
        const int ab = u & 1;
        bar_wait(tfull(ab), (u >> 1) & 1);
        fence_after();
#pragma unroll
        for (int t0 = 0; t0 < TAPS; t0 += 3) {  // three taps per TMEM wait
          if (((t0 / 3) & 1) != half) continue;
          uint32_t r[3][16];
#pragma unroll
          for (int dt = 0; dt < 3; ++dt)
            if (t0 + dt < TAPS) tmem_ld16_issue(trow + (uint32_t)(ab * 256 + (t0 + dt) * BNB), r[dt]);
          tmem_wait_ld();
#pragma unroll
          for (int dt = 0; dt < 3; ++dt)
            if (t0 + dt < TAPS) {
#pragma unroll
              for (int e = 0; e < 16; ++e) Dsm[((t0 + dt) * BNB + e) * 128 + m] = __uint_as_float(r[dt][e]);
            }
        }
        fence_before();
        bar_arrive(tempty(ab));  // the accumulator buffer is free for the unit after next
        sync_epi();
        // contrib layout [list index][channel block][16][PH][PW]: consecutive items, consecutive floats
        const int items = ntile * BNB * PPT;
        float* cdst = a.contrib + ((int64_t)(g * TPU) * a.nb + nb) * PSZ;
#pragma unroll 2
        for (int i = etid; i < items; i += EPI) {
          const int px = i % PW, py = (i / PW) % PH, n = (i / PPT) % BNB, j = i / (BNB * PPT);
          const float* dcol = Dsm + n * 128 + j * SLOT;
          float sum = 0.0f;
#pragma unroll
          for (int t = 0; t < TAPS; ++t) {
            const int iy = py + t / K - K + 1, ix = px + t % K - K + 1;
            if (iy >= 0 && iy < T && ix >= 0 && ix < T) sum = __fadd_rn(sum, dcol[t * BNB * 128 + iy * T + ix]);
          }
          cdst[(int64_t)j * a.nb * PSZ + (i - j * BNB * PPT)] = sum;
        }
        sync_epi();
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 12) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

// map[t] = list index of live input tile t (map pre-filled with -1)
__global__ void k_scatter_map(const int32_t* __restrict__ list, const int32_t* __restrict__ count, int32_t* map) {
  pdl_wait();
  pdl_trigger();
  const int n = *count;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) map[list[i]] = i;
}

// One CTA per (session, strip of STRIP output tiles in a tile row): each output value sums, in a
// fixed neighbour order, the patch points of the (up to 4) live neighbour input tiles that cover it
// (contrib layout [li][nb][16][PH][PW]).  The covering list of every pixel is resolved once per CTA;
// a warp then writes 24-pixel row runs.  Tiles dead now but live last step are zeroed once;
// `live_prev` carries that state between steps.
constexpr int STRIP = 4;

template <int K, int T>
__global__ void __launch_bounds__(256) k_scatter_gather(const __grid_constant__ ScArgs a, const int32_t* __restrict__ map,
                                                        float* __restrict__ out, int64_t ovs, int Ho, int Wo,
                                                        uint8_t* live_prev) {
  constexpr int PH = T + K - 1, PW = T + K - 1, SITES = T * T, PPT = PH * PW, PSZ = PPT * BNB;
  constexpr int OFF = K - 1 - K / 2;  // patch origin offset ("same" padding K / 2)
  __shared__ int s_off[STRIP][SITES][4];
  __shared__ int s_cnt[STRIP][SITES];
  __shared__ int s_state[STRIP];  // bit 0: live now, bit 1: live last step
  pdl_wait();
  pdl_trigger();
  const int GHo = (Ho + T - 1) / T, GWo = (Wo + T - 1) / T, nstrip = (GWo + STRIP - 1) / STRIP;
  const int s = blockIdx.y, ty = blockIdx.x / nstrip, tx0 = (blockIdx.x % nstrip) * STRIP;
  const int32_t* mp = map + (int64_t)s * a.GH * a.GW;
  uint8_t* lp = live_prev + (int64_t)s * GHo * GWo + (int64_t)ty * GWo;
  if (threadIdx.x < STRIP * SITES) {
    const int q = threadIdx.x / SITES, p = threadIdx.x % SITES, tx = tx0 + q;
    const int ly = p / T, lx = p % T;
    int cnt = 0;
    bool live = false;
    if (tx < GWo) {
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        const int ny = ty + k / 3 - 1, nx = tx + k % 3 - 1;
        const int li = (ny >= 0 && ny < a.GH && nx >= 0 && nx < a.GW) ? __ldg(mp + ny * a.GW + nx) : -1;
        live |= li >= 0;
        const int py = ly - (k / 3 - 1) * T + OFF, px = lx - (k % 3 - 1) * T + OFF;  // in the neighbour's patch
        if (li >= 0 && py >= 0 && py < PH && px >= 0 && px < PW) s_off[q][p][cnt++] = li * a.nb * PSZ + py * PW + px;
      }
    }
    s_cnt[q][p] = cnt;
    if (p == 0) s_state[q] = tx < GWo ? ((live ? 1 : 0) | (lp[tx] ? 2 : 0)) : 0;
  }
  __syncthreads();
  if (!(s_state[0] | s_state[1] | s_state[2] | s_state[3])) return;  // nothing to write in this strip
  constexpr int RW = STRIP * T;  // strip row width (pixels)
  constexpr int U = 4;           // items per thread per pass: every load issued before any store
  const int total = a.c_out * T * RW;
  for (int i0 = threadIdx.x; i0 < total; i0 += U * 256) {
    float sum[U];
    int64_t dst[U];
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      const int i = i0 + uu * 256;
      sum[uu] = 0.0f;
      dst[uu] = -1;
      if (i >= total) continue;
      const int xx = i % RW, y = (i / RW) % T, n = i / (RW * T);
      const int q = xx / T, lx = xx % T, p = y * T + lx;
      const int st = s_state[q];
      const int oy = ty * T + y, ox = (tx0 + q) * T + lx;
      if (!st || oy >= Ho || ox >= Wo) continue;
      dst[uu] = (int64_t)s * ovs + ((int64_t)n * Ho + oy) * Wo + ox;
      if (st & 1) {
        const float* cb = a.contrib + (int64_t)(n / BNB) * PSZ + (n % BNB) * PPT;
        const int c = s_cnt[q][p];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (k < c) sum[uu] = __fadd_rn(sum[uu], __ldg(cb + s_off[q][p][k]));
      }
    }
#pragma unroll
    for (int uu = 0; uu < U; ++uu)
      if (dst[uu] >= 0) out[dst[uu]] = sum[uu];
  }
  __syncthreads();
  if (threadIdx.x < STRIP && tx0 + (int)threadIdx.x < GWo) lp[tx0 + threadIdx.x] = s_state[threadIdx.x] & 1;
}

}  // namespace sc

template <int K>
static int init_scatter_k() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, sc::k_conv_scatter<K, 6>) != cudaSuccess) return EVC_ECUDA;
  if (cudaFuncSetAttribute(sc::k_conv_scatter<K, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
      cudaSuccess)
    return EVC_ECUDA;
  if (cudaFuncGetAttributes(&fa, sc::k_scatter_gather<K, 6>) != cudaSuccess) return EVC_ECUDA;
  return EVC_OK;
}

int init_conv_scatter() { return init_scatter_k<1>() | init_scatter_k<3>(); }

}  // namespace evc

using namespace evc;

namespace {

struct ScGeo {
  int taps, nb, nkb, b_half, PH, PW, GH, GW, Ti, GHo, GWo;
};

ScGeo sc_geo(const evc_conv_geom* g) {
  ScGeo o;
  o.taps = g->kh * g->kw;
  o.nb = (g->c_out + sc::BNB - 1) / sc::BNB;
  o.nkb = (g->c_in + 31) / 32;
  o.b_half = o.taps * sc::BNB * 128;
  o.PH = g->th + g->kh - 1;
  o.PW = g->tw + g->kw - 1;
  o.GH = (g->H + g->th - 1) / g->th;
  o.GW = (g->W + g->tw - 1) / g->tw;
  o.Ti = o.GH * o.GW;
  o.GHo = (g->Ho + g->th - 1) / g->th;
  o.GWo = (g->Wo + g->tw - 1) / g->tw;
  return o;
}

// workspace layout (bytes, 256-aligned parts): fany u8 [S*Ti] | list i32 [S*Ti] | count i32 | map i32
// [S*Ti] | compact scratch | live_prev u8 [S*GHo*GWo] | contrib f32 [S*Ti][nb][PH*PW*16]
struct ScWs {
  size_t fany, list, count, map, scratch, prev, contrib, total;
};

size_t al256(size_t x) { return (x + 255) / 256 * 256; }

ScWs sc_ws(const evc_conv_geom* g, int S) {
  const ScGeo o = sc_geo(g);
  const int64_t n = (int64_t)S * o.Ti;
  ScWs w;
  w.fany = 0;
  w.list = al256(w.fany + n);
  w.count = al256(w.list + 4 * n);
  w.map = al256(w.count + 4);
  w.scratch = al256(w.map + 4 * n);
  w.prev = al256(w.scratch + 4 * (size_t)evc_compact_scratch(n));
  w.contrib = al256(w.prev + (size_t)S * o.GHo * o.GWo);
  w.total = al256(w.contrib + 4 * (size_t)n * o.nb * o.PH * o.PW * sc::BNB);
  return w;
}

}  // namespace

extern "C" {

int evc_conv_scatter_supported(const evc_conv_geom* g) {
  if (!g) return 0;
  return g->stride == 1 && g->kh == g->kw && (g->kh == 1 || g->kh == 3) && g->pad == g->kh / 2 && g->th == 6 &&
         g->tw == 6 && g->c_in <= 32 * sc::MAX_KB &&
         g->pad < g->kw && g->kh <= 3 && g->kw <= 3 && g->Ho == g->H + 2 * g->pad - g->kh + 1 &&
         g->Wo == g->W + 2 * g->pad - g->kw + 1 && (g->th + g->kh - 1) * (g->tw + g->kw - 1) * sc::BNB % 4 == 0;
}

int64_t evc_conv_scatter_pack_len(const evc_conv_geom* g) {
  if (!evc_conv_scatter_supported(g)) return -1;
  const ScGeo o = sc_geo(g);
  return (int64_t)o.nb * o.nkb * 2 * o.taps * sc::BNB * 32;
}

int evc_conv_scatter_pack(const float* w, const evc_conv_geom* g, float* out) {
  EVC_CHECK_ARG(w && out && evc_conv_scatter_supported(g), "conv_scatter_pack: bad argument");
  const ScGeo o = sc_geo(g);
  const int rows = o.taps * sc::BNB;
  for (int b = 0; b < o.nb; ++b)
    for (int kb = 0; kb < o.nkb; ++kb) {
      float* hi = out + ((int64_t)b * o.nkb + kb) * 2 * rows * 32;
      float* lo = hi + (int64_t)rows * 32;
      for (int row = 0; row < rows; ++row) {
        const int t = row / sc::BNB, n = b * sc::BNB + row % sc::BNB, r = t / g->kw, q = t % g->kw;
        for (int e = 0; e < 32; ++e) {
          const int c = kb * 32 + e;
          const float x = (n < g->c_out && c < g->c_in) ? w[(((int64_t)n * g->c_in + c) * g->kh + r) * g->kw + q] : 0.0f;
          uint32_t bits;
          memcpy(&bits, &x, 4);
          bits = (bits + 0x1000u) & 0xFFFFE000u;  // TF32 head (round to nearest, as tf32_head)
          float hv;
          memcpy(&hv, &bits, 4);
          const int64_t pos = (int64_t)row * 32 + (((e / 4) ^ (row & 7)) * 4) + e % 4;  // 128B swizzle
          hi[pos] = hv;
          lo[pos] = x - hv;
        }
      }
    }
  return EVC_OK;
}

int64_t evc_conv_scatter_workspace(const evc_conv_geom* g, int32_t S) {
  if (!evc_conv_scatter_supported(g) || S < 1) return -1;
  return (int64_t)sc_ws(g, S).total;
}

int evc_conv_scatter(const evc_conv_geom* g, const evc_tensor* in, const float* wpack, const evc_tensor* out,
                     void* workspace, int64_t ws_bytes, int32_t fresh_out, int32_t S, void* stream) {
  EVC_CHECK_ARG(g && in && in->vals && in->flags && wpack && out && out->vals && workspace && S > 0,
                "conv_scatter: null argument");
  EVC_CHECK_ARG(evc_conv_scatter_supported(g), "conv_scatter: unsupported geometry (stride 1, k <= 3, tiles <= 36)");
  EVC_CHECK_ARG(in->C == g->c_in && in->H == g->H && in->W == g->W && out->C == g->c_out && out->H == g->Ho &&
                    out->W == g->Wo,
                "conv_scatter: tensor shapes do not match the geometry");
  const ScWs w = sc_ws(g, S);
  EVC_CHECK_ARG(ws_bytes >= (int64_t)w.total, "conv_scatter: workspace too small");
  const ScGeo o = sc_geo(g);
  char* ws = static_cast<char*>(workspace);
  uint8_t* fany = reinterpret_cast<uint8_t*>(ws + w.fany);
  int32_t* list = reinterpret_cast<int32_t*>(ws + w.list);
  int32_t* count = reinterpret_cast<int32_t*>(ws + w.count);
  int32_t* map = reinterpret_cast<int32_t*>(ws + w.map);
  cudaStream_t st = as_stream(stream);
  int rc = evc_tile_any(in, fany, S, stream);
  if (rc) return rc;
  rc = evc_compact(fany, (int64_t)S * o.Ti, list, count, reinterpret_cast<int32_t*>(ws + w.scratch), stream);
  if (rc) return rc;
  cudaError_t e = cudaMemsetAsync(map, 0xFF, sizeof(int32_t) * (size_t)S * o.Ti, st);
  if (e == cudaSuccess && fresh_out)  // a zeroed output buffer: no tile holds values from an earlier call
    e = cudaMemsetAsync(ws + w.prev, 0, (size_t)S * o.GHo * o.GWo, st);
  if (e != cudaSuccess) {
    set_error(std::string("evc: conv_scatter memset: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  launch_pdl(sc::k_scatter_map, dim3(148), dim3(256), 0, st, list, count, map);
  EVC_LAUNCH_CHECK("scatter_map");
  const TView vin = view_of(*in);
  sc::ScArgs a;
  memset(&a, 0, sizeof(a));
  a.in = vin.v;
  a.in_vs = vin.vs;
  a.C = g->c_in;
  a.H = g->H;
  a.W = g->W;
  a.th = g->th;
  a.tw = g->tw;
  a.GH = o.GH;
  a.GW = o.GW;
  a.kh = g->kh;
  a.kw = g->kw;
  a.pad = g->pad;
  a.taps = o.taps;
  a.c_out = g->c_out;
  a.nb = o.nb;
  a.nkb = o.nkb;
  a.b_half = o.b_half;
  a.PH = o.PH;
  a.PW = o.PW;
  a.wpack = wpack;
  a.list = list;
  a.count = count;
  a.contrib = reinterpret_cast<float*>(ws + w.contrib);
  const int bstage = (2 * o.b_half + 1023) / 1024 * 1024;
  const size_t smem = (size_t)o.nkb * sc::A_KB + (size_t)sc::NS * bstage + 4 * (size_t)128 * o.taps * sc::BNB +
                      1024 + 256;
  EVC_CHECK_ARG(smem <= 227 * 1024, "conv_scatter: shared memory");
  const int grid = 148;
  e = g->kh == 3 ? launch_pdl(sc::k_conv_scatter<3, 6>, dim3(grid), dim3(sc::THREADS), smem, st, a)
                 : launch_pdl(sc::k_conv_scatter<1, 6>, dim3(grid), dim3(sc::THREADS), smem, st, a);
  if (e != cudaSuccess) {
    set_error(std::string("evc: conv_scatter launch: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  const TView vout = view_of(*out);
  auto gk = g->kh == 3 ? sc::k_scatter_gather<3, 6> : sc::k_scatter_gather<1, 6>;
  const int nstrip = (o.GWo + sc::STRIP - 1) / sc::STRIP;
  e = launch_pdl(gk, dim3(o.GHo * nstrip, S), dim3(256), 0, st, a, map, vout.v, vout.vs, (int)g->Ho, (int)g->Wo,
                 reinterpret_cast<uint8_t*>(ws + w.prev));
  if (e != cudaSuccess) {
    set_error(std::string("evc: scatter_gather launch: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  return EVC_OK;
}

}  // extern "C"
