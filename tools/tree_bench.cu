// Cycles per general tree solve on one warp: mcg_solve_tree_warp (lane per
// chain) vs mcg_solve_tree_fast (one thread), on a busyring-like tree (soma
// chain of 7, two level-1 and four level-2 branches of 8 compartments).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++20 \
//        -I paper_2411_16445_b200/csrc tools/tree_bench.cu paper_2411_16445_b200/csrc/mcg_build.cpp -o tree_bench.bin
#include <cstdio>
#include <vector>
#include "mcg_batch.cuh"
#include "mcg_build.h"

__global__ void bench(int n, const int32_t* G, const int32_t* par, int reps, int mode, long long* cyc) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  double *cap = sm, *gs = sm + n, *coup = sm + 2 * n, *rhs = sm + 3 * n, *v = sm + 4 * n, *diag = sm + 5 * n,
         *r2 = sm + 6 * n;
  int32_t* sp = reinterpret_cast<int32_t*>(sm + 7 * n);
  for (int i = lane; i < n; i += 32) {
    cap[i] = 1.0 + 0.01 * i; coup[i] = i ? 0.3 + 0.001 * i : 0.0; rhs[i] = 0.5; v[i] = -65.0 + 0.1 * i; sp[i] = par[i];
  }
  __syncwarp();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (int i = lane; i < n; i += 32) gs[i] = 0.2 + 0.001 * i;
    __syncwarp();
    if (mode == 0) mcg_solve_tree_warp(G, sp, cap, gs, coup, rhs, v, diag, r2, lane);
    else if (lane == 0) mcg_solve_tree_fast(n, sp, cap, gs, coup, rhs, v, diag, r2);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[mode] = (t1 - t0) / reps;
}

int main() {
  std::vector<int32_t> par;
  auto seg = [&](int parent, int len) { int first = par.size(); for (int k = 0; k < len; ++k) par.push_back(k == 0 ? parent : int(par.size()) - 1); return int(par.size()) - 1; (void)first; };
  par.push_back(-1);
  for (int k = 1; k < 7; ++k) par.push_back(k - 1);
  const int soma_end = 6;
  int l1a = seg(soma_end, 8), l1b = seg(soma_end, 8);
  seg(l1a, 8); seg(l1a, 8); seg(l1b, 8); seg(l1b, 8);
  const int n = par.size();
  std::vector<int32_t> sched;
  const int nch = mcg::tree_chains(n, par.data(), sched);
  printf("n %d chains %d maxlev %d\n", n, nch, sched[1]);
  int32_t *dG, *dp; long long* cyc;
  cudaMalloc(&dG, sched.size() * 4); cudaMalloc(&dp, n * 4); cudaMallocManaged(&cyc, 16);
  cudaMemcpy(dG, sched.data(), sched.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, par.data(), n * 4, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 2; ++mode) {
    bench<<<1, 32, 8 * n * 8>>>(n, dG, dp, 2000, mode, cyc);
    cudaDeviceSynchronize();
    printf("%s: %lld cycles per solve (%.0f per node)\n", mode ? "one thread" : "warp, lane per chain", cyc[mode],
           double(cyc[mode]) / n);
  }
  return 0;
}
