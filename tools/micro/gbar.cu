// Grid-barrier micro-benchmark: 148 co-resident CTAs run N barriers.
// (1) atomicAdd + generation flag (reset by the last arriver)
// (2) monotonic counter: red.release.gpu.add, poll ld.acquire until >= k*G
// (3) monotonic counter, relaxed polls + fence after
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void red_release(unsigned* p, unsigned v) { asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
__global__ void k(unsigned* bar, int mode, int iters, int sleep_ns, unsigned long long* out) {
  const int G = gridDim.x;
  unsigned long long t0 = clock64();
  for (int it = 1; it <= iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      if (mode == 1) {
        unsigned* cnt = bar; unsigned* gen = bar + 1;
        const unsigned g0 = ld_relaxed(gen);
        __threadfence();
        if (atomicAdd(cnt, 1u) == (unsigned)G - 1u) { atomicExch(cnt, 0u); __threadfence(); asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1) : "memory"); }
        else while (ld_relaxed(gen) == g0) { if (sleep_ns) __nanosleep(sleep_ns); }
        __threadfence();
      } else if (mode == 2) {
        red_release(bar + 2, 1u);
        const unsigned target = (unsigned)it * G;
        while (ld_acquire(bar + 2) < target) { if (sleep_ns) __nanosleep(sleep_ns); }
      } else {
        __threadfence();
        atomicAdd(bar + 3, 1u);
        const unsigned target = (unsigned)it * G;
        while (ld_relaxed(bar + 3) < target) { if (sleep_ns) __nanosleep(sleep_ns); }
        __threadfence();
      }
    }
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}
int main() {
  unsigned* bar; unsigned long long* out; cudaMalloc(&bar, 64); cudaMalloc(&out, 8);
  for (int mode = 1; mode <= 3; ++mode)
    for (int sl : {0, 32, 100}) {
      cudaMemset(bar, 0, 64);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      void* args[] = {&bar, &mode, nullptr, &sl, &out};
      int iters = 1000; args[2] = &iters;
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)k, 148, 128, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("mode %d sleep %3d: %.3f us per barrier (%s)\n", mode, sl, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
}
