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

namespace evc {
namespace sc {

using namespace fz;

constexpr int BNB = 16;      // output channels per unit
constexpr int SLOT = 40;     // A rows (TMEM lanes) per tile slot: th * tw <= 36 sites, five 8-row groups
constexpr int TPU = 3;       // tiles per group (120 of 128 rows)
constexpr int NS = 3;        // weight pipeline stages
constexpr int A_KB = 2 * 128 * 128;  // one K-block of the resident A tile: heads + tails, 128 rows x 128 B
constexpr int MAX_KB = 3;    // resident A: C_in <= 96
constexpr int THREADS = 320;  // warps 0-3 gather, 4-7 epilogue, 8 TMEM alloc + MMA issuer, 9 weight stream

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

__device__ __forceinline__ void sync_epi() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// One CTA walks tile groups (3 live input tiles); per group the gather warps stage the A tile of
// every K-block once (resident), and the MMA issuer runs all output-channel blocks over it, each
// into a double-buffered TMEM accumulator that the epilogue warps scatter into output patches.
__global__ void __launch_bounds__(THREADS, 1) k_conv_scatter(const __grid_constant__ ScArgs a) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int N = a.taps * BNB;
  const uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const int BSTAGE = (2 * a.b_half + 1023) / 1024 * 1024;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* bst = smem + a.nkb * A_KB;  // weight stages
  float* patch = reinterpret_cast<float*>(bst + NS * BSTAGE);
  const int PSZ = a.PH * a.PW * BNB;  // floats per tile patch
  uint64_t* bars = reinterpret_cast<uint64_t*>(patch + TPU * PSZ);
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
      bar_init(tempty(i), 128);
    }
    bar_init(afull, 128);
    bar_init(aempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
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
  const int sites = a.th * a.tw, Ti = a.GH * a.GW;

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
          tile_y[j] = (r / a.GW) * a.th;
          tile_x[j] = (r % a.GW) * a.tw;
        }
      }
      if (q >= 1) bar_wait(aempty, (q - 1) & 1);  // every MMA over the previous group's A is done
      // element e = ((j * 32 + c) * th + y) * tw + x  (x fastest: short coalesced runs)
      const int per = TPU * 32 * sites;
      for (int kb = 0; kb < a.nkb; ++kb) {
        float* Ah = reinterpret_cast<float*>(smem + kb * A_KB);
        float* Al = Ah + 128 * 32;
        for (int e0 = tid; e0 < per; e0 += 128 * BATCH) {
          float v[BATCH];
#pragma unroll
          for (int k = 0; k < BATCH; ++k) {
            const int e = e0 + 128 * k;
            v[k] = 0.0f;
            if (e < per) {
              const int x = e % a.tw, y = (e / a.tw) % a.th, c = (e / sites) % 32, j = e / (32 * sites);
              const int ch = kb * 32 + c, py = tile_y[j] + y, px = tile_x[j] + x;
              if (tile_s[j] >= 0 && ch < a.C && py < a.H && px < a.W)
                v[k] = __ldg(a.in + (int64_t)tile_s[j] * a.in_vs + ((int64_t)ch * a.H + py) * a.W + px);
            }
          }
#pragma unroll
          for (int k = 0; k < BATCH; ++k) {
            const int e = e0 + 128 * k;
            if (e < per) {
              const int x = e % a.tw, y = (e / a.tw) % a.th, c = (e / sites) % 32, j = e / (32 * sites);
              const int row = j * SLOT + y * a.tw + x;
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
  } else if (warp == 9) {  // ----------------------------------------------------- weight stream
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
  } else if (warp == 8) {  // ------------------------------------------------------- MMA issuer
    if (lane == 0) {
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
              mma(d, dah + 2 * kk, dbh + 2 * kk, IDESC, (kb || kk) ? 1u : 0u);  // hi.hi
              mma(d, dah + 2 * kk, dbl + 2 * kk, IDESC, 1u);                    // hi.lo
              mma(d, dal + 2 * kk, dbh + 2 * kk, IDESC, 1u);                    // lo.hi
            }
            commit(bempty(st));
          }
          commit(tfull(ab));
        }
        commit(aempty);  // the gather may overwrite A once these MMAs have completed
      }
    }
    __syncwarp();
  } else {  // ---------------------------------------------------------------------- epilogue
    const int etid = threadIdx.x - 128;
    const int m = 32 * (warp & 3) + lane;  // TMEM lane = A row
    const int j = m / SLOT, p = m % SLOT;
    const bool site = j < TPU && p < sites;
    const int iy = p / a.tw, ix = p % a.tw;
    const uint32_t trow = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    int u = 0;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
      const int ntile = min(TPU, n_live - g * TPU);
      for (int nb = 0; nb < a.nb; ++nb, ++u) {
        for (int i = etid; i < TPU * PSZ; i += 128) patch[i] = 0.0f;
        sync_epi();
        const int ab = u & 1;
        bar_wait(tfull(ab), (u >> 1) & 1);
        fence_after();
        for (int t0 = 0; t0 < a.taps; t0 += 3) {  // three taps per TMEM wait
          uint32_t r[3][16];
#pragma unroll
          for (int dt = 0; dt < 3; ++dt)
            if (t0 + dt < a.taps) tmem_ld16_issue(trow + (uint32_t)(ab * 256 + (t0 + dt) * BNB), r[dt]);
          tmem_wait_ld();
          if (t0 + 3 >= a.taps) {  // the accumulator buffer is free for the unit after next
            fence_before();
            bar_arrive(tempty(ab));
          }
#pragma unroll
          for (int dt = 0; dt < 3; ++dt) {
            const int t = t0 + dt;
            if (t < a.taps) {
              if (site && j < ntile) {
                const int rr = t / a.kw, qq = t % a.kw;
                const int py = iy - rr + a.kh - 1, px = ix - qq + a.kw - 1;  // patch coordinates
                float4* dst = reinterpret_cast<float4*>(patch + j * PSZ + (py * a.PW + px) * BNB);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  float4 w = dst[e];
                  w.x = __fadd_rn(w.x, __uint_as_float(r[dt][4 * e]));
                  w.y = __fadd_rn(w.y, __uint_as_float(r[dt][4 * e + 1]));
                  w.z = __fadd_rn(w.z, __uint_as_float(r[dt][4 * e + 2]));
                  w.w = __fadd_rn(w.w, __uint_as_float(r[dt][4 * e + 3]));
                  dst[e] = w;
                }
              }
              sync_epi();  // the next tap may hit the same positions from other sites
            }
          }
        }
        // patches of the group's live tiles -> contrib[list index][nb]
        const int q4 = PSZ / 4;
        for (int i = etid; i < ntile * q4; i += 128) {
          const int jj = i / q4, k = i - jj * q4;
          float4* dst = reinterpret_cast<float4*>(a.contrib + ((int64_t)(g * TPU + jj) * a.nb + nb) * PSZ);
          dst[k] = reinterpret_cast<const float4*>(patch + jj * PSZ)[k];
        }
        sync_epi();
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 8) {
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

// One CTA per (session, output tile): sum the patches of the live neighbour input tiles in a fixed
// order, stage the th x tw x C_out tile in shared memory, write it channel-planar.  Tiles dead now
// but live last step are zeroed once; `live_prev` carries the state between steps.
__global__ void __launch_bounds__(128) k_scatter_gather(const __grid_constant__ ScArgs a, const int32_t* __restrict__ map,
                                                        float* __restrict__ out, int64_t ovs, int Ho, int Wo,
                                                        uint8_t* live_prev) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float tile[];  // [sites][c_out + 1]
  const int GHo = (Ho + a.th - 1) / a.th, GWo = (Wo + a.tw - 1) / a.tw;
  const int s = blockIdx.y, T = blockIdx.x, ty = T / GWo, tx = T % GWo;
  const int Ti = a.GH * a.GW;
  const int32_t* mp = map + (int64_t)s * Ti;
  // neighbour input tiles whose patch reaches this output tile: input tile rows ny with
  // [ny th + pad - (kh - 1), ny th + th - 1 + pad] meeting [ty th, ty th + th - 1]
  int nbr[9];
  int nn = 0;
  bool live = false;
  for (int dy = -1; dy <= 1; ++dy)
    for (int dx = -1; dx <= 1; ++dx) {
      const int ny = ty + dy, nx = tx + dx;
      int li = -1;
      if (ny >= 0 && ny < a.GH && nx >= 0 && nx < a.GW) li = mp[ny * a.GW + nx];
      nbr[nn++] = li >= 0 ? (li << 4) | ((dy + 1) * 3 + (dx + 1)) : -1;
      live |= li >= 0;
    }
  uint8_t* lp = live_prev + (int64_t)s * GHo * GWo + T;
  const bool was = *lp != 0;
  if (!live && !was) return;
  const int sites = a.th * a.tw, CP = a.c_out + 1, PSZ = a.PH * a.PW * BNB;
  for (int i = threadIdx.x; i < sites * a.c_out; i += blockDim.x) {
    const int n = i % a.c_out, pidx = i / a.c_out;
    const int oy = ty * a.th + pidx / a.tw, ox = tx * a.tw + pidx % a.tw;
    float sum = 0.0f;
    if (live) {
#pragma unroll
      for (int k = 0; k < 9; ++k) {
        if (nbr[k] < 0) continue;
        const int li = nbr[k] >> 4, d = nbr[k] & 15, dy = d / 3 - 1, dx = d % 3 - 1;
        const int py = oy - ((ty + dy) * a.th + a.pad - (a.kh - 1)), px = ox - ((tx + dx) * a.tw + a.pad - (a.kw - 1));
        if (py < 0 || py >= a.PH || px < 0 || px >= a.PW) continue;
        sum = __fadd_rn(sum, a.contrib[((int64_t)li * a.nb + n / BNB) * PSZ + (py * a.PW + px) * BNB + n % BNB]);
      }
    }
    tile[pidx * CP + n] = sum;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < sites * a.c_out; i += blockDim.x) {
    const int pidx = i % sites, n = i / sites;
    const int oy = ty * a.th + pidx / a.tw, ox = tx * a.tw + pidx % a.tw;
    if (oy < Ho && ox < Wo) out[(int64_t)s * ovs + ((int64_t)n * Ho + oy) * Wo + ox] = tile[pidx * CP + n];
  }
  if (threadIdx.x == 0) *lp = live ? 1 : 0;
}

}  // namespace sc

int init_conv_scatter() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, sc::k_conv_scatter) != cudaSuccess) return EVC_ECUDA;
  if (cudaFuncSetAttribute(sc::k_conv_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) !=
      cudaSuccess)
    return EVC_ECUDA;
  if (cudaFuncSetAttribute(sc::k_scatter_gather, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024) !=
      cudaSuccess)
    return EVC_ECUDA;
  return EVC_OK;
}

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
  return g->stride == 1 && g->kh * g->kw * sc::BNB <= 256 && g->th * g->tw <= 36 && g->pad < g->kh &&
         g->c_in <= 32 * sc::MAX_KB &&
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
  const size_t smem = (size_t)o.nkb * sc::A_KB + (size_t)sc::NS * bstage +
                      4 * (size_t)sc::TPU * o.PH * o.PW * sc::BNB + 1024 + 256;
  EVC_CHECK_ARG(smem <= 227 * 1024, "conv_scatter: shared memory");
  const int grid = 148;
  e = launch_pdl(sc::k_conv_scatter, dim3(grid), dim3(sc::THREADS), smem, st, a);
  if (e != cudaSuccess) {
    set_error(std::string("evc: conv_scatter launch: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  const TView vout = view_of(*out);
  const size_t gsm = 4 * (size_t)g->th * g->tw * (g->c_out + 1);
  EVC_CHECK_ARG(gsm <= 96 * 1024, "conv_scatter: too many output channels for the gather tile");
  e = launch_pdl(sc::k_scatter_gather, dim3(o.GHo * o.GWo, S), dim3(128), gsm, st, a, map, vout.v, vout.vs,
                 (int)g->Ho, (int)g->Wo, reinterpret_cast<uint8_t*>(ws + w.prev));
  if (e != cudaSuccess) {
    set_error(std::string("evc: scatter_gather launch: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  return EVC_OK;
}

}  // extern "C"
