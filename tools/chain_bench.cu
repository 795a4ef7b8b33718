// Cycles per mcg_chain_lane call (mcg_sweep.cuh): one warp = 5 cells x 3
// systems x 2 chain sides (30 lanes), the consolidation cell's spider tree
// (31 or 48 compartments), warps per SM as given.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++20 tools/chain_bench.cu -o tools/chain_bench.bin
#include <cstdio>
#include <vector>
#include "../paper_2411_16445_b200/csrc/mcg_batch.cuh"

__global__ void bench(int lp, int n, int reps, int wregion, long long* cyc, int active) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int P = 2 * lp + 1;
  // kind block: idx (int32, P) then 3 systems x 6 x P doubles, shared by all warps
  const int cho = 0;
  int32_t* PI = reinterpret_cast<int32_t*>(mcg_smem);
  const int kd = (P + 1) / 2 + 18 * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    // chain A positions [0, lp): nodes top..leaf reversed; B [lp, 2lp)
    int node = -1;
    if (i < lp) { const int k = lp - 1 - i; node = k < (n - 1) / 2 + 6 ? 1 + k : -1; }
    else if (i < 2 * lp) { const int k = 2 * lp - 1 - i; node = k < (n - 1) - ((n - 1) / 2 + 6) ? 1 + (n - 1) / 2 + 6 + k : -1; }
    else node = 0;
    if (node >= n) node = -1;
    PI[i] = node;
  }
  for (int i = threadIdx.x; i < 18 * P; i += blockDim.x) {
    const int q = i % (6 * P), a = q / P;
    double v = 0.0;
    if (a == 0) v = 0.1; else if (a == 1) v = 0.05; else if (a == 2) v = 2.0; else if (a == 3) v = 0.5;
    else if (a == 4) v = 1.0; else v = 0.2;
    mcg_smem[(P + 1) / 2 + i] = v;
  }
  __syncthreads();
  const int base = kd + w * wregion;
  const int k = lane / 6, rem = lane % 6, sys = rem >> 1, side = rem & 1;
  McgChainLane L{};
  const int cell = base + k * 4 * 48;  // V | SP | SP | RC per cell (m = 48)
  if (k < 5 && lane < active) {
    L.on = 1; L.side = side; L.lp = lp;
    L.r2c = base + 5 * 4 * 48 + (k * 3 + sys) * P;
    L.idx = 2 * cho; L.fc = cho + (P + 1) / 2 + sys * 6 * P;
    L.x = cell + (sys == 0 ? 0 : 48 + (sys - 1) * n); L.a_first = 1; L.v = sys == 0;
    L.rc = sys == 0 ? cell + 3 * 48 : -1; L.pc = sys == 2 ? 0 : -1; L.prod = 0.1;
  }
  for (int i = lane; i < 5 * 4 * 48; i += 32) mcg_smem[base + i] = -65.0 + 0.01 * i;
  __syncwarp();
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    mcg_chain_lane(L);
    __syncwarp();
  }
  long long t1 = clock64();
  if (lane == 0) cyc[blockIdx.x * 32 + w] = (t1 - t0) / reps;
}

int main1();
int main2();
int main() { main2(); return main1(); }
int main1() {
  long long* cyc;
  cudaMallocManaged(&cyc, 148 * 32 * 8);
  for (int n : {31, 48}) {
    const int lp = n == 31 ? 20 : 40;
    const int P = 2 * lp + 1;
    const int wregion = 5 * 4 * 48 + 15 * P + 64;
    for (int active : {1, 2, 6, 30}) {
      const int warps = 1;
      const int smem = ((P + 1) / 2 + 18 * P + warps * wregion) * 8;
      cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      bench<<<148, 32 * warps, smem>>>(lp, n, 200, wregion, cyc, active);
      cudaDeviceSynchronize();
      printf("n %d lp %d 1 warp, %d active lanes: %lld cycles per sweep\n", n, lp, active, cyc[0]);
    }
    for (int warps : {1, 2, 3, 4, 8}) {
      const int smem = ((P + 1) / 2 + 18 * P + warps * wregion) * 8;
      cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      bench<<<148, 32 * warps, smem>>>(lp, n, 200, wregion, cyc, 32);
      cudaError_t e = cudaDeviceSynchronize();
      printf("n %d lp %d warps/SM %d: %lld cycles per sweep (%s)\n", n, lp, warps, cyc[0], cudaGetErrorString(e));
    }
  }
  return 0;
}
// FP64 issue cost: DFMA chains, 1 warp, `act` active lanes, 4 independent chains per lane
__global__ void fma_tp(int act, int iters, long long* cyc, double* out) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane, b = 0.5, c = 0.25, d = 0.125;
  long long t0 = clock64();
  if (lane < act)
    for (int i = 0; i < iters; ++i) {
      a = __fma_rn(a, 0.999, 1e-3);
      b = __fma_rn(b, 0.999, 1e-3);
      c = __fma_rn(c, 0.999, 1e-3);
      d = __fma_rn(d, 0.999, 1e-3);
    }
  __syncwarp();
  long long t1 = clock64();
  if (lane == 0) cyc[0] = (t1 - t0) / iters;
  out[threadIdx.x] = a + b + c + d;
}
int main2() {
  long long* cyc; double* out;
  cudaMallocManaged(&cyc, 64); cudaMallocManaged(&out, 4096);
  for (int act : {1, 2, 4, 8, 16, 32}) {
    fma_tp<<<1, 32>>>(act, 10000, cyc, out);
    cudaDeviceSynchronize();
    printf("DFMA x4 independent, %d active lanes: %lld cycles per iteration\n", act, cyc[0]);
  }
  return 0;
}
