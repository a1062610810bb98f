// Channels-innermost ("HWC") hi/lo shadow of a channel-planar tensor: the
// A-operand layout of the TMA-fed conv GEMM (conv_fused.cu, see hwc_store in
// common.cuh): per pixel the TF32 heads of the cp (= C rounded up to 32)
// channels, then their tails.  Rows are `pitch` pixels apart: the consumer conv
// keeps a zero border of its padding around the interior (y points at pixel (0, 0)).

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace evc {

// CHW -> channels-innermost shadow (channel stride cp), 32x32 tiles through SMEM
// so both the planar reads and the channel-contiguous writes are coalesced.
__global__ void __launch_bounds__(256) k_to_hwc(TView x, float* __restrict__ y, int64_t ys, int cp, int pitch) {
  __shared__ float t[32][33];
  pdl_wait();
  pdl_trigger();
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
    if (p < HW && c < x.C) {
      const int py = p / x.W, px = p - py * x.W;
      hwc_store(dst + ((int64_t)py * pitch + px) * hwc_px(cp), cp, c, t[tx][ty + 8 * k]);
    }
  }
}

// Small fp32 shadows (the CUDA-core path's cp = -C, C <= 8): one thread per pixel, coalesced planar
// reads, one contiguous run of C floats per pixel (the 32x32 transpose tile would idle 7/8 of its
// threads for C = 4).
__global__ void __launch_bounds__(256) k_to_hwc_small(TView x, float* __restrict__ y, int64_t ys, int cp, int pitch) {
  pdl_wait();
  pdl_trigger();
  const int HW = x.H * x.W, s = blockIdx.y, C = x.C, px_stride = -cp;
  const float* src = x.v + (int64_t)s * x.vs;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += gridDim.x * blockDim.x) {
    float v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = c < C ? src[(int64_t)c * HW + p] : 0.0f;
    const int py = p / x.W, px = p - py * x.W;
    float* d = y + (int64_t)s * ys + ((int64_t)py * pitch + px) * px_stride;
    if (px_stride == 4) {
      *reinterpret_cast<float4*>(d) = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c < C) d[c] = v[c];
    }
  }
}

}  // namespace evc

using namespace evc;

extern "C" {

int32_t evc_hwc_channels(int32_t c) { return (c + 31) / 32 * 32; }

int evc_to_hwc(const evc_tensor* x, float* y, int64_t y_stride, int32_t cp, int32_t pitch, int32_t S,
               void* stream) {
  EVC_CHECK_ARG(x && x->vals && y && S > 0 && std::abs(cp) >= x->C && cp % 4 == 0 && pitch >= x->W, "to_hwc: bad argument");
  TView v = view_of(*x);
  if (cp < 0 && v.C <= 8 && -cp <= 8) {
    const cudaError_t e = launch_pdl(k_to_hwc_small, dim3(std::min(cdiv(v.H * v.W, 256), 1184), S), dim3(256), 0,
                                     as_stream(stream), v, y, y_stride, cp, pitch);
    if (e != cudaSuccess) {
      set_error(std::string("evc: to_hwc: ") + cudaGetErrorString(e));
      return EVC_ECUDA;
    }
    return EVC_OK;
  }
  dim3 grid(cdiv(v.H * v.W, 32), cdiv(v.C, 32), S);
  const cudaError_t e = launch_pdl(k_to_hwc, grid, dim3(256), 0, as_stream(stream), v, y, y_stride, cp, pitch);
  if (e != cudaSuccess) {
    set_error(std::string("evc: to_hwc: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  return EVC_OK;
}

int evc_copy_bytes(const void* src, int64_t src_stride, void* dst, int64_t dst_stride, int64_t nbytes, int32_t S,
                   void* stream) {
  EVC_CHECK_ARG(src && dst && nbytes >= 0 && S > 0 && src_stride >= nbytes && dst_stride >= nbytes,
                "copy_bytes: bad argument");
  if (nbytes == 0) return EVC_OK;
  const cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dst_stride, src, (size_t)src_stride, (size_t)nbytes, (size_t)S,
                                          cudaMemcpyDeviceToDevice, as_stream(stream));
  if (e != cudaSuccess) {
    set_error(std::string("evc: copy_bytes: ") + cudaGetErrorString(e));
    return EVC_ECUDA;
  }
  return EVC_OK;
}

}  // extern "C"
