// Tile-mask kernels: step_increment diff+mask, make_tile_mask, ordered
// compaction, flag counts, integrate, masked/dense copies, drift.
//
// Layout: channel-planar (C,H,W) per session, exactly the reference layout
// (tensors.py:1-6).  "Band" kernels give one CTA a (session, channel,
// tile-row) band: th rows x W columns, contiguous in memory, so loads are
// coalesced along W and a tile's any() is a CTA-local shared-memory OR.

#include <mutex>

#include "common.cuh"

namespace evc {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static bool g_pdl = false;
bool pdl_enabled() { return g_pdl; }

// ---------------------------------------------------------------------------
// step_increment + make_tile_mask  (events.py:295-302, tensors.py:93-107)
// ---------------------------------------------------------------------------
__global__ void k_diff_mask(const float* __restrict__ prev, const float* __restrict__ cur,
                            int64_t in_stride, TView o) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t s_nz[];
  const int i = blockIdx.x, c = blockIdx.y, s = blockIdx.z;
  for (int j = threadIdx.x; j < o.GW; j += blockDim.x) s_nz[j] = 0;
  __syncthreads();
  const int64_t base = (int64_t)s * in_stride + (int64_t)c * o.H * o.W;
  float* out = o.plane(s, c);
  const int r0 = i * o.th, r1 = min(o.H, r0 + o.th);
  for (int x = threadIdx.x; x < o.W; x += blockDim.x) {
    bool nz = false;
    for (int r = r0; r < r1; ++r) {
      const int64_t e = (int64_t)r * o.W + x;
      const float d = __fsub_rn(cur[base + e], prev[base + e]);
      out[e] = d;
      nz |= (d != 0.0f);  // -0.0 counts as zero (tensors.py:105)
    }
    if (nz) s_nz[x / o.tw] = 1;
  }
  __syncthreads();
  uint8_t* f = o.fplane(s, c) + (int64_t)i * o.GW;
  for (int j = threadIdx.x; j < o.GW; j += blockDim.x) f[j] = s_nz[j];
}

__global__ void k_make_mask(TView o) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t s_nz[];
  const int i = blockIdx.x, c = blockIdx.y, s = blockIdx.z;
  for (int j = threadIdx.x; j < o.GW; j += blockDim.x) s_nz[j] = 0;
  __syncthreads();
  const float* in = o.plane(s, c);
  const int r0 = i * o.th, r1 = min(o.H, r0 + o.th);
  for (int x = threadIdx.x; x < o.W; x += blockDim.x) {
    bool nz = false;
    for (int r = r0; r < r1; ++r) nz |= (in[(int64_t)r * o.W + x] != 0.0f);
    if (nz) s_nz[x / o.tw] = 1;
  }
  __syncthreads();
  uint8_t* f = o.fplane(s, c) + (int64_t)i * o.GW;
  for (int j = threadIdx.x; j < o.GW; j += blockDim.x) f[j] = s_nz[j];
}

// ---------------------------------------------------------------------------
// Ordered compaction (np.flatnonzero) -- two deterministic launches.
// ---------------------------------------------------------------------------
constexpr int kCompactThreads = 1024;
constexpr int kCompactPer = 4;  // flags per thread
constexpr int kCompactChunk = kCompactThreads * kCompactPer;

__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int w = lane < (blockDim.x >> 5) ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    s_warp[lane] = w;  // inclusive prefix of warp totals
  }
  __syncthreads();
  const int warp_off = wid ? s_warp[wid - 1] : 0;
  *total = s_warp[(blockDim.x >> 5) - 1];
  return warp_off + x - v;
}

__global__ void k_compact_count(const uint8_t* __restrict__ flags, int64_t n, int32_t* counts) {
  pdl_wait();
  pdl_trigger();
  const int64_t base = (int64_t)blockIdx.x * kCompactChunk;
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < kCompactPer; ++k) {
    const int64_t e = base + (int64_t)k * kCompactThreads + threadIdx.x;
    cnt += (e < n && flags[e] != 0);
  }
  __shared__ int s_w[32];
  int tot;
  (void)block_excl_scan(cnt, s_w, &tot);
  if (threadIdx.x == 0) counts[blockIdx.x] = tot;
}

__global__ void k_compact_write(const uint8_t* __restrict__ flags, int64_t n, const int32_t* counts,
                                int32_t* idx, int32_t* count) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_w[32];
  __shared__ int s_off;
  // offset = sum of counts of previous blocks (deterministic order)
  int part = 0;
  for (int b = threadIdx.x; b < (int)blockIdx.x; b += blockDim.x) part += counts[b];
  int tot0;
  (void)block_excl_scan(part, s_w, &tot0);
  if (threadIdx.x == 0) s_off = tot0;
  __syncthreads();
  int off = s_off;
  const int64_t base = (int64_t)blockIdx.x * kCompactChunk;
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < kCompactPer; ++k) {
    // elements of this sub-chunk are contiguous across threads -> ascending order
    const int64_t e = base + (int64_t)k * kCompactThreads + threadIdx.x;
    const bool on = e < n && flags[e] != 0;
    const unsigned bal = __ballot_sync(0xffffffffu, on);  // warp ballot
    if (lane == 0) s_w[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {  // prefix over warp totals
      int w = lane < nw ? s_w[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    const int woff = wid ? s_w[wid - 1] : 0;
    if (on) idx[off + woff + __popc(bal & ((1u << lane) - 1u))] = (int32_t)e;
    off += s_w[nw - 1];
    __syncthreads();
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) *count = off;
}

// ---------------------------------------------------------------------------
// counts of True flags per session
// ---------------------------------------------------------------------------
__global__ void k_count_flags(TView t, int32_t* counts) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  const int64_t n = (int64_t)t.C * t.GH * t.GW;
  const uint8_t* f = t.f + (int64_t)s * t.fs;
  int cnt = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    cnt += f[e] != 0;
  __shared__ int s_w[32];
  int tot;
  (void)block_excl_scan(cnt, s_w, &tot);
  if (threadIdx.x == 0 && tot) atomicAdd(counts + s, tot);
}

__global__ void k_copy_dense(const float* __restrict__ a, int64_t as, float* __restrict__ b, int64_t bs,
                             int64_t n) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    b[(int64_t)s * bs + e] = a[(int64_t)s * as + e];
}

__global__ void k_max_abs_diff(const float* __restrict__ a, int64_t as, const float* __restrict__ b, int64_t bs,
                               int64_t n, float* out) {
  pdl_wait();
  pdl_trigger();
  const int s = blockIdx.y;
  float m = 0.0f;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(__fsub_rn(a[(int64_t)s * as + e], b[(int64_t)s * bs + e])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0f)
    atomicMax(reinterpret_cast<unsigned int*>(out + s), __float_as_uint(m));
}

static int band_threads(int W) { return W >= 192 ? 256 : (W >= 96 ? 128 : (W >= 48 ? 64 : 32)); }

}  // namespace evc

using namespace evc;

extern "C" {

int evc_version(void) { return EVC_ABI_VERSION; }

const char* evc_last_error(void) { return g_err.c_str(); }

int evc_diff_mask(const float* prev, const float* cur, int64_t in_stride, const evc_tensor* out, int32_t S,
                  void* stream) {
  EVC_CHECK_ARG(out && out->vals && out->flags && prev && cur && S > 0, "diff_mask: null argument");
  TView o = view_of(*out);
  dim3 grid(o.GH, o.C, S);
  launch_pdl(k_diff_mask, dim3(grid), dim3(band_threads(o.W)), o.GW, as_stream(stream), prev, cur, in_stride, o);
  EVC_LAUNCH_CHECK("diff_mask");
  return EVC_OK;
}

int evc_make_tile_mask(const evc_tensor* t, int32_t S, void* stream) {
  EVC_CHECK_ARG(t && t->vals && t->flags && S > 0, "make_tile_mask: null argument");
  TView o = view_of(*t);
  dim3 grid(o.GH, o.C, S);
  launch_pdl(k_make_mask, dim3(grid), dim3(band_threads(o.W)), o.GW, as_stream(stream), o);
  EVC_LAUNCH_CHECK("make_tile_mask");
  return EVC_OK;
}

int64_t evc_compact_scratch(int64_t n) { return cdiv64(n > 0 ? n : 1, kCompactChunk); }

int evc_compact(const uint8_t* flags, int64_t n, int32_t* idx, int32_t* count, int32_t* scratch, void* stream) {
  EVC_CHECK_ARG(flags && idx && count && scratch && n >= 0, "compact: null argument");
  const int nb = (int)evc_compact_scratch(n);
  cudaStream_t st = as_stream(stream);
  launch_pdl(k_compact_count, dim3(nb), dim3(kCompactThreads), 0, st, flags, n, scratch);
  launch_pdl(k_compact_write, dim3(nb), dim3(kCompactThreads), 0, st, flags, n, scratch, idx, count);
  EVC_LAUNCH_CHECK("compact");
  return EVC_OK;
}

int evc_count_flags(const evc_tensor* t, int32_t S, int32_t* counts, void* stream) {
  EVC_CHECK_ARG(t && t->flags && counts && S > 0, "count_flags: null argument");
  TView v = view_of(*t);
  const int64_t n = (int64_t)v.C * v.GH * v.GW;
  const int blocks = (int)std::min<int64_t>(cdiv64(n, 256 * 4), 64);
  launch_pdl(k_count_flags, dim3(dim3(blocks > 0 ? blocks : 1, S)), dim3(256), 0, as_stream(stream), v, counts);
  EVC_LAUNCH_CHECK("count_flags");
  return EVC_OK;
}

int evc_copy_dense(const float* src, int64_t src_stride, float* dst, int64_t dst_stride, int64_t n, int32_t S,
                   void* stream) {
  EVC_CHECK_ARG(src && dst && S > 0 && n >= 0, "copy_dense: null argument");
  if (n == 0) return EVC_OK;
  const int blocks = (int)std::min<int64_t>(cdiv64(n, 256 * 4), 1024);
  launch_pdl(k_copy_dense, dim3(dim3(blocks, S)), dim3(256), 0, as_stream(stream), src, src_stride, dst, dst_stride, n);
  EVC_LAUNCH_CHECK("copy_dense");
  return EVC_OK;
}

int evc_max_abs_diff(const float* a, int64_t as, const float* b, int64_t bs, int64_t n, int32_t S, float* out,
                     void* stream) {
  EVC_CHECK_ARG(a && b && out && S > 0, "max_abs_diff: null argument");
  if (n == 0) return EVC_OK;
  const int blocks = (int)std::min<int64_t>(cdiv64(n, 256 * 4), 512);
  launch_pdl(k_max_abs_diff, dim3(dim3(blocks, S)), dim3(256), 0, as_stream(stream), a, as, b, bs, n, out);
  EVC_LAUNCH_CHECK("max_abs_diff");
  return EVC_OK;
}

}  // extern "C"

namespace evc {
int init_masks() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, k_diff_mask) != cudaSuccess) return EVC_ECUDA;
  return EVC_OK;
}
}  // namespace evc

extern "C" int evc_set_pdl(int32_t on) {
  evc::g_pdl = on != 0;
  return EVC_OK;
}

extern "C" int evc_init(void) {
  int rc = evc::init_masks();
  if (!rc) rc = evc::init_conv();
  if (!rc) rc = evc::init_elementwise();
  if (!rc) rc = evc::init_linear_events();
  if (rc) evc::set_error(std::string("evc: init failed: ") + cudaGetErrorString(cudaGetLastError()));
  return rc;
}
