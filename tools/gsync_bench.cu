// grid-wide barrier cost on the B200: cooperative_groups grid.sync() vs a
// release/acquire counter barrier, 143 CTAs x 512 threads (the config-3 grid)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 tools/gsync_bench.cu -o tools/gsync_bench.bin
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, long long* out) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = (t1 - t0) / iters;
}

__device__ __forceinline__ void bar_arrive_wait(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

__global__ void k_ra(int iters, unsigned* ctr, long long* out) {
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) bar_arrive_wait(ctr, (i + 1) * gridDim.x);
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) out[1] = (t1 - t0) / iters;
}

int main() {
  long long* out;
  unsigned* ctr;
  cudaMallocManaged(&out, 64);
  cudaMalloc(&ctr, 4);
  int iters = 2000;
  for (int grid : {143, 148}) {
    void* a1[] = {&iters, &out};
    cudaLaunchCooperativeKernel((void*)k_cg, grid, 512, a1, 0, 0);
    cudaDeviceSynchronize();
    cudaMemset(ctr, 0, 4);
    void* a2[] = {&iters, &ctr, &out};
    cudaLaunchCooperativeKernel((void*)k_ra, grid, 512, a2, 0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("grid %d: cg grid.sync %lld cycles, release/acquire barrier %lld cycles (%s)\n", grid, out[0],
           out[1], cudaGetErrorString(e));
  }
  return 0;
}
