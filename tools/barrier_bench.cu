// Grid-barrier latency microbenchmark (B200): the persistent GMRES kernel's
// "last arriver releases" barrier versus a monotonic counting barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin_barrier tools/barrier_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.add.release.gpu.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: ours (last arriver resets count and bumps gen; others poll gen with ld.acquire)
// mode 1: same, polling with ld.relaxed + one fence after the change
// mode 2: monotonic counter: every block adds 1, spins until count >= G*(it+1)
__global__ void k_bar(unsigned* count, unsigned* gen, int iters, int mode, int nsleep) {
  __shared__ unsigned s_last;
  for (int it = 0; it < iters; ++it) {
    if (mode == 2) {
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned target = gridDim.x * (unsigned)(it + 1);
        atom_add_acq_rel(count, 1u);
        while (ld_relaxed(count) < target) { if (nsleep) __nanosleep(nsleep); }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads();
      continue;
    }
    __syncthreads();
    unsigned g = 0;
    if (threadIdx.x == 0) {
      g = ld_relaxed(gen);
      const unsigned t = atom_add_acq_rel(count, 1u);
      s_last = (t == gridDim.x - 1) ? 1u : 0u;
    }
    __syncthreads();
    if (s_last) {
      if (threadIdx.x == 0) {
        *reinterpret_cast<volatile unsigned*>(count) = 0u;
        red_add_release(gen, 1u);
      }
    } else if (threadIdx.x == 0) {
      if (mode == 0) {
        while (ld_acquire(gen) == g) { if (nsleep) __nanosleep(nsleep); }
      } else {
        while (ld_relaxed(gen) == g) { if (nsleep) __nanosleep(nsleep); }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
}

int main() {
  unsigned *count, *gen;
  cudaMalloc(&count, 256);
  cudaMalloc(&gen, 256);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  int grids[] = {44, 104, 148, 208, 296};
  for (int mode = 0; mode < 3; ++mode)
    for (int ns : {0, 32})
      for (int G : grids) {
        if (G > 2 * nsm) continue;
        cudaMemset(count, 0, 256);
        cudaMemset(gen, 0, 256);
        void* args[] = {&count, &gen, (void*)&iters, &mode, &ns};
        int it2 = 100;
        void* wargs[] = {&count, &gen, (void*)&it2, &mode, &ns};
        cudaLaunchCooperativeKernel((void*)k_bar, G, 256, wargs, 0, 0);
        cudaDeviceSynchronize();
        cudaMemset(count, 0, 256);
        cudaMemset(gen, 0, 256);
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_bar, G, 256, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("mode=%d nanosleep=%d grid=%d: %.3f us per barrier (%s)\n", mode, ns, G,
               ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
