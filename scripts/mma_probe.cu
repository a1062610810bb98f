// Micro-probe: cycles per tcgen05.mma.kind::tf32 (M=128, K=8, SMEM A/B, SW128 K-major)
// as a function of N and of the accumulator pattern.  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mma_probe.bin scripts/mma_probe.cu && ./scripts/mma_probe.bin
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t desc_k(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
template <int KIND>  // 0 = tf32, 1 = f16 (bf16)
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (KIND == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                 "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int N, int KIND>
__global__ void probe(int iters, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~(uintptr_t)1023);
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(base)[i] = 0.001f * (i % 7);
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  constexpr uint32_t IDESC_TF32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // kind::f16 with bf16 inputs: a_format=1 (bf16), b_format=1, d f32
  constexpr uint32_t IDESC_BF16 = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint32_t idesc = KIND == 0 ? IDESC_TF32 : IDESC_BF16;
  const uint32_t a0 = su32(base), b0 = su32(base + 32768);
  if (threadIdx.x == 0) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ko = (i & 3) * 32;
      uint32_t d = tmem;
      if (mode == 1) d = tmem + (uint32_t)((i % 3) * N);  // rotate 3 accumulators
      mma<KIND>(d, desc_k(a0 + ko), desc_k(b0 + ko), idesc, i > 2 ? 1u : 0u);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred p;\nW1:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W1;\n\t}" ::"r"(su32(&bar)) : "memory");
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(512));
  }
}

template <int N, int KIND>
void run(int mode) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(probe<N, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 4096;
  probe<N, KIND><<<1, 128, 100 * 1024>>>(iters, mode, d);
  probe<N, KIND><<<1, 128, 100 * 1024>>>(iters, mode, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * N * (KIND == 0 ? 8 : 16);
  printf("%s N=%3d mode=%d: %6.1f cycles/MMA  %7.1f FLOP/cycle  (%s)\n", KIND == 0 ? "tf32" : "bf16", N, mode,
         (double)h / iters, flop * iters / (double)h, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<16, 0>(0);
  run<32, 0>(0);
  run<64, 0>(0);
  run<128, 0>(0);
  run<256, 0>(0);
  run<64, 0>(1);
  run<64, 1>(0);
  run<256, 1>(0);
  return 0;
}
