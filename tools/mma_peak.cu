// Micro-benchmark: tcgen05.mma issue rate from resident shared-memory operands (no loads),
// cta_group::1 (M=128) vs cta_group::2 (M=256 across a CTA pair), N = 128 / 256.
// Answers whether the single-CTA decode GEMMs are bounded by operand delivery or by the
// MMA rate itself.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak tools/mma_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t ctarank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }

template <int CG, int N>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  uint8_t* A = base;                    // 128 x 64 bf16
  uint8_t* B = base + 16384;            // (N / CG) x 64 bf16
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(N));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tbase)), "r"(N));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) { asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tbase;
  const bool leader = CG == 1 || ctarank() == 0;
  constexpr int M = 128 * CG;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0 && leader) {
    if (threadIdx.x == 0) {
      t0 = clock64();
      const uint32_t a0 = su32(A), b0 = su32(B);
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t da = desc(a0 + k * 32), db = desc(b0 + k * 32);
          const uint32_t acc = (it | k) ? 1u : 0u;
          if (CG == 1)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm), "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      }
      if (CG == 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
      else
        asm volatile("{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\ttcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(su32(&bar)) : "memory");
    }
  }
  if (threadIdx.x == 0) {
    asm volatile("{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(su32(&bar)) : "memory");
    t1 = clock64();
    if (leader) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) { asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(N));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(N));
  }
}

template <int CG, int N>
void run(int iters) {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaMemset(d, 0, 148 * 8);
  const int smem = 1024 + 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(k_mma<CG, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, k_mma<CG, N>, iters, d);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, k_mma<CG, N>, iters, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double macs_per_cta_group = (double)iters * 4 * (128.0 * CG) * N * 16;
  const double flops_total = 2.0 * macs_per_cta_group * (148 / CG);
  printf("cta_group::%d M=%d N=%d: %s  cycles %llu  MAC/clk/SM %.0f  TFLOP/s %.0f\n", CG, 128 * CG, N,
         cudaGetErrorString(err), mx, macs_per_cta_group / CG / (double)mx, flops_total / (ms * 1e-3) / 1e12);
  cudaFree(d);
}

int main() {
  const int it = 20000;
  run<1, 128>(it);
  run<1, 256>(it);
  run<2, 128>(it);
  run<2, 256>(it);
  return 0;
}
