// Microbenchmark of the constant-diagonal Hines sweep on the consolidation
// cell's 31-compartment tree: cycles per sweep for the
// engine's loop (mcg_sweep_const_sm) and candidate schedules.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++20 tools/sweep_bench.cu -o tools/sweep_bench.bin
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cmath>
#include "../paper_2411_16445_b200/csrc/mcg_batch.cuh"
#include "../paper_2411_16445_b200/csrc/mcg_sweep.cuh"

__constant__ int PPc[31] = {-1, 0, 1, 2, 3, 4, 5, 0, 7, 8, 9, 10, 11, 6, 13, 14, 15, 16, 17, 18, 19, 20,
                            21, 22, 23, 24, 12, 26, 27, 28, 29};
__host__ __device__ constexpr int ppk(int i) {
  return i == 0 ? -1 : (i == 7 ? 0 : (i == 13 ? 6 : (i == 26 ? 12 : i - 1)));
}

// floor: fully unrolled, compile-time tree, operands in registers
__device__ __forceinline__ void sweep_unrolled(int par, int coup, int f, int d, int y, int x, int r2) {
  double* S = mcg_smem;
  double R[31];
#pragma unroll
  for (int i = 0; i < 31; ++i) R[i] = S[r2 + i];
#pragma unroll
  for (int i = 30; i >= 1; --i) R[ppk(i)] = R[ppk(i)] + S[f + i] * R[i];
  double X[31];
  X[0] = mcg_div(R[0], S[d], S[y]);
#pragma unroll
  for (int i = 1; i < 31; ++i) X[i] = mcg_div(R[i] + S[coup + i] * X[ppk(i)], S[d + i], S[y + i]);
#pragma unroll
  for (int i = 0; i < 31; ++i) S[x + i] = X[i];
}
__device__ __forceinline__ double div_fast(double x, double d, double y) {
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, d, x);
  return __fma_rn(r, y, q);
}
__device__ __forceinline__ void sweep_unrolled_nocheck(int par, int coup, int f, int d, int y, int x, int r2) {
  double* S = mcg_smem;
  double R[31];
#pragma unroll
  for (int i = 0; i < 31; ++i) R[i] = S[r2 + i];
#pragma unroll
  for (int i = 30; i >= 1; --i) R[ppk(i)] = R[ppk(i)] + S[f + i] * R[i];
  double X[31];
  X[0] = div_fast(R[0], S[d], S[y]);
#pragma unroll
  for (int i = 1; i < 31; ++i) X[i] = div_fast(R[i] + S[coup + i] * X[ppk(i)], S[d + i], S[y + i]);
#pragma unroll
  for (int i = 0; i < 31; ++i) S[x + i] = X[i];
}

__global__ void bench(int n, int variant, int reps, long long* cyc, double* out, const double* g_init) {
  double* S = mcg_smem;
  // layout: par(int, n+2 padded) | f | d | y | coup | cap | x | r2   (each n+2, one spare each side)
  const int W = n + 4;
  const int par = 0;                       // int offsets in units of int32
  const int f = W, d = 2 * W + 1, y = 3 * W + 2, coup = 4 * W + 3, cap = 5 * W + 4;
  const int x0 = 6 * W + 8, r20 = 8 * W + 8;
  const int sys = threadIdx.x;             // one system per thread
  const int x = x0 + sys * 0, r2 = r20;    // all threads share (bench of latency only, thread 0 timed)
  if (threadIdx.x == 0) {
    int32_t* PI = reinterpret_cast<int32_t*>(S);
    for (int i = 0; i < 4 * W; ++i) PI[i] = 0;
    const int pp[31] = {-1, 0, 1, 2, 3, 4, 5, 0, 7, 8, 9, 10, 11, 6, 13, 14, 15, 16, 17, 18, 19, 20,
                        21, 22, 23, 24, 12, 26, 27, 28, 29};
    for (int i = 0; i < n; ++i) PI[par + i] = pp[i];
    for (int i = 0; i < n; ++i) {
      S[f + i] = g_init[i];
      S[d + i] = g_init[n + i];
      S[y + i] = 1.0 / g_init[n + i];
      S[coup + i] = g_init[2 * n + i];
      S[cap + i] = g_init[3 * n + i];
      S[x + i] = -65.0 + i;
    }
    // chain lists: A = 25..13, 6..1 (leaf->top), B = 30..26, 12..7
    const int ch = 2 * (9 * W + 8 + 2 * W) ;  // int32 units
    int k = 0;
    for (int i = 25; i >= 13; --i) PI[ch + k++] = i;
    for (int i = 6; i >= 1; --i) PI[ch + k++] = i;
    for (int i = 30; i >= 26; --i) PI[ch + k++] = i;
    for (int i = 12; i >= 7; --i) PI[ch + k++] = i;
  }
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < n; ++i) S[r2 + i] = S[cap + i] * S[x + i] + 0.25;
      if (variant == 0) mcg_sweep_const_sm(n, par, coup, f, d, y, x, r2);
      else if (variant == 1) sweep_unrolled(par, coup, f, d, y, x, r2);
      else if (variant == 2) sweep_unrolled_nocheck(par, coup, f, d, y, x, r2);
      else if (variant == 3) { /* rhs only */ }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) {
    cyc[variant] = (t1 - t0) / reps;
    out[0] = S[x];
  }
}


// chain-lane sweep (mcg_sweep.cuh) on lanes 0/1: the 31-node tree, LP = 20
__global__ void bench_chain(int reps, long long* cyc, const double* g_init) {
  double* S = mcg_smem;
  int32_t* PI = reinterpret_cast<int32_t*>(S);
  const int n = 31, lp = 20, P = 2 * lp + 1;
  const int idx = 0;                  // int32 units, P ints
  const int fc = 64;                  // doubles: f|c|d|y|cap|glr each P
  const int r2c = fc + 6 * P + 8, x = r2c + P + 8, cap = x + n + 8;
  if (threadIdx.x == 0) {
    for (int p = 0; p < P; ++p) PI[idx + p] = -1;
    int k = 0;
    for (int i = 1; i <= 6; ++i) PI[idx + lp - 1 - k++] = i;
    for (int i = 13; i <= 25; ++i) PI[idx + lp - 1 - k++] = i;
    k = 0;
    for (int i = 7; i <= 12; ++i) PI[idx + 2 * lp - 1 - k++] = i;
    for (int i = 26; i <= 30; ++i) PI[idx + 2 * lp - 1 - k++] = i;
    PI[idx + 2 * lp] = 0;
    for (int p = 0; p < P; ++p) {
      const int i = PI[idx + p];
      S[fc + p] = i < 0 ? -0.0 : g_init[i];
      S[fc + P + p] = i < 0 ? 0.0 : g_init[2 * n + i];
      S[fc + 2 * P + p] = i < 0 ? 1.0 : g_init[n + i];
      S[fc + 3 * P + p] = i < 0 ? 1.0 : 1.0 / g_init[n + i];
      S[fc + 4 * P + p] = i < 0 ? 0.0 : g_init[3 * n + i];
      S[fc + 5 * P + p] = i < 0 ? 0.0 : 0.25;
      S[r2c + p] = i < 0 ? 0.0 : 1.5;
    }
    for (int i = 0; i < n; ++i) S[x + i] = -65.0 + i;
  }
  __syncthreads();
  McgChainLane L{threadIdx.x < 2, int(threadIdx.x & 1), lp, r2c, fc, idx, x, 0, 1, -1, -1, 0.0};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    mcg_chain_lane(L);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[10] = (t1 - t0) / reps;
}


// the kernel's lane layout: 5 cells x 3 systems x 2 sides on lanes 0..29
// (chain constants shared per system, r2c and x per cell at the kernel strides)
__global__ void bench_chain30(int reps, long long* cyc, const double* g_init, int cell_stride,
                              int ch_stride) {
  double* S = mcg_smem;
  int32_t* PI = reinterpret_cast<int32_t*>(S);
  const int n = 31, lp = 20, P = 2 * lp + 1;
  const int idx = 0;                   // int32 units
  const int fc0 = 64;                  // 3 systems x 6 P
  const int r2c0 = fc0 + 3 * 6 * P + 8;
  const int x0 = r2c0 + 5 * ch_stride + 8;
  if (threadIdx.x == 0) {
    for (int p = 0; p < P; ++p) PI[idx + p] = -1;
    int k = 0;
    for (int i = 1; i <= 6; ++i) PI[idx + lp - 1 - k++] = i;
    for (int i = 13; i <= 25; ++i) PI[idx + lp - 1 - k++] = i;
    k = 0;
    for (int i = 7; i <= 12; ++i) PI[idx + 2 * lp - 1 - k++] = i;
    for (int i = 26; i <= 30; ++i) PI[idx + 2 * lp - 1 - k++] = i;
    PI[idx + 2 * lp] = 0;
    for (int sy = 0; sy < 3; ++sy)
      for (int p = 0; p < P; ++p) {
        const int i = PI[idx + p];
        double* q = S + fc0 + sy * 6 * P;
        q[p] = i < 0 ? -0.0 : g_init[i];
        q[P + p] = i < 0 ? 0.0 : g_init[2 * n + i];
        q[2 * P + p] = i < 0 ? 1.0 : g_init[n + i];
        q[3 * P + p] = i < 0 ? 1.0 : 1.0 / g_init[n + i];
        q[4 * P + p] = i < 0 ? 0.0 : g_init[3 * n + i];
        q[5 * P + p] = i < 0 ? 0.0 : 0.25;
      }
    for (int c = 0; c < 5; ++c)
      for (int i = 0; i < 3 * n; ++i) S[x0 + c * cell_stride + i] = -65.0 + i;
  }
  __syncthreads();
  const int t = threadIdx.x, c = t / 6, sy = (t % 6) / 2, side = t & 1;
  McgChainLane L{t < 30, side, lp, r2c0 + c * ch_stride + sy * P, fc0 + sy * 6 * P, idx,
                 x0 + c * cell_stride + (sy == 0 ? 0 : n + (sy - 1) * n), 0, sy == 0, -1, -1, 0.0};
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    mcg_chain_lane(L);
    __syncwarp();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[11] = (t1 - t0) / reps;
}

int main() {
  const int n = 31;
  std::vector<double> h(4 * n);
  for (int i = 0; i < n; ++i) {
    h[i] = 0.1 + 0.01 * i;        // f
    h[n + i] = 3.0 + 0.1 * i;     // d
    h[2 * n + i] = 0.5;           // coup
    h[3 * n + i] = 2.0;           // cap
  }
  double *g, *out;
  long long* cyc;
  cudaMalloc(&g, h.size() * 8);
  cudaMalloc(&out, 64);
  cudaMallocManaged(&cyc, 64 * 8);
  cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int v = 0; v < 4; ++v) {
    bench<<<1, 32, 16 * 1024>>>(n, v, 100, cyc, out, g);
    bench<<<1, 32, 16 * 1024>>>(n, v, 1000, cyc, out, g);
    cudaError_t e = cudaDeviceSynchronize();
    printf("variant %d: %lld cycles per rhs+sweep (%s)\n", v, cyc[v], cudaGetErrorString(e));
  }
  cudaFuncSetAttribute(bench_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  bench_chain<<<1, 32, 16 * 1024>>>(100, cyc, g);
  bench_chain<<<1, 32, 16 * 1024>>>(1000, cyc, g);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("chain lanes: %lld cycles per sweep (%s)\n", cyc[10], cudaGetErrorString(e2));
  cudaFuncSetAttribute(bench_chain30, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int cs : {124, 128, 132, 125}) {
    for (int chs : {123, 128, 129}) {
      bench_chain30<<<1, 32, 64 * 1024>>>(100, cyc, g, cs, chs);
      bench_chain30<<<1, 32, 64 * 1024>>>(1000, cyc, g, cs, chs);
      cudaError_t e3 = cudaDeviceSynchronize();
      printf("chain 30 lanes cell_stride %d ch_stride %d: %lld cycles (%s)\n", cs, chs, cyc[11], cudaGetErrorString(e3));
    }
  }
  return 0;
}
