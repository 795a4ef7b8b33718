// Microbenchmark: dependent-chain latency of FP64 ops and shared-memory
// round trips on the B200 (cycles per link), plus an exhaustive-ish check
// that the reciprocal + FMA-correction quotient equals IEEE division.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/fp64_lat.cu -o /tmp/fp64_lat
#include <cstdio>
#include <cstdint>
#include <cstring>

__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sm[64];
  double x = a, y = b;
  sm[threadIdx.x] = a;
  __syncthreads();
  long long t0, t1;
  // DADD chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dadd_rn(x, y);
  t1 = clock64();
  cyc[0] = t1 - t0;
  // DMUL chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __dmul_rn(x, y);
  t1 = clock64();
  cyc[1] = t1 - t0;
  // DFMA chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __fma_rn(x, y, a);
  t1 = clock64();
  cyc[2] = t1 - t0;
  // DDIV chain
  t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __ddiv_rn(x, y);
  t1 = clock64();
  cyc[3] = t1 - t0;
  // reciprocal-multiply + correction chain (y precomputed)
  const double r = 1.0 / y;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const double q = __dmul_rn(x, r);
    const double e = __fma_rn(-q, y, x);
    x = __fma_rn(e, r, q);
  }
  t1 = clock64();
  cyc[4] = t1 - t0;
  // shared store -> load round trip chain
  volatile double* vs = sm;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    vs[threadIdx.x] = x;
    x = vs[threadIdx.x];
  }
  t1 = clock64();
  cyc[5] = t1 - t0;
  // shared load -> dependent address chain (int)
  int* si = reinterpret_cast<int*>(sm);
  volatile int* vsi = si;
  if (threadIdx.x == 0) for (int i = 0; i < 64; ++i) vsi[i] = (i + 1) & 63;
  __syncthreads();
  int p = 0;
  t0 = clock64();
  for (int i = 0; i < iters; ++i) p = vsi[p];
  t1 = clock64();
  cyc[6] = t1 - t0;
  out[threadIdx.x] = x + p;
}

__global__ void mk_check(const double* divs, int nd, unsigned long long n, unsigned long long* bad,
                         unsigned long long seed) {
  const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  const unsigned long long nth = (unsigned long long)gridDim.x * blockDim.x;
  unsigned long long s = seed ^ (tid * 0x9E3779B97F4A7C15ull);
  unsigned long long cnt = 0;
  for (unsigned long long i = tid; i < n; i += nth) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const double d = divs[i % nd];
    // numerators across a wide exponent range and both signs
    const unsigned long long e = 1023 - 60 + ((s >> 52) % 120);
    const unsigned long long bits = (e << 52) | (s & 0xFFFFFFFFFFFFFull) | ((s >> 63) << 63);
    double x;
    memcpy(&x, &bits, 8);
    const double y = __ddiv_rn(1.0, d);
    const double q = __dmul_rn(x, y);
    const double r = __fma_rn(-q, d, x);
    const double q2 = __fma_rn(r, y, q);
    const double t = __ddiv_rn(x, d);
    if (__double_as_longlong(q2) != __double_as_longlong(t)) ++cnt;
  }
  if (cnt) atomicAdd(bad, cnt);
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64 * 8);
  cudaMallocManaged(&cyc, 16 * 8);
  const int it = 4096;
  lat<<<1, 1>>>(out, cyc, 1.0000001, 0.9999999, it);
  cudaDeviceSynchronize();
  lat<<<1, 1>>>(out, cyc, 1.0000001, 0.9999999, it);
  cudaDeviceSynchronize();
  const char* nm[] = {"dadd", "dmul", "dfma", "ddiv", "rcp+corr", "smem st->ld", "smem ld->addr"};
  for (int i = 0; i < 7; ++i) printf("%-14s %.1f cycles/link\n", nm[i], double(cyc[i]) / it);
  // random divisors (broad) + typical Hines diagonals
  const int nd = 1 << 16;
  double* hd = new double[nd];
  unsigned long long s = 12345;
  for (int i = 0; i < nd; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    const unsigned long long e = 1023 - 40 + ((s >> 52) % 80);
    const unsigned long long bits = (e << 52) | (s & 0xFFFFFFFFFFFFFull);
    memcpy(&hd[i], &bits, 8);
  }
  double* dd; unsigned long long* bad;
  cudaMalloc(&dd, nd * 8);
  cudaMallocManaged(&bad, 8);
  cudaMemcpy(dd, hd, nd * 8, cudaMemcpyHostToDevice);
  *bad = 0;
  const unsigned long long n = 1ull << 36;
  mk_check<<<148 * 8, 256>>>(dd, nd, n, bad, 777);
  cudaError_t e = cudaDeviceSynchronize();
  printf("markstein check: %llu mismatches of %llu (%s)\n", *bad, n, cudaGetErrorString(e));
  return 0;
}
