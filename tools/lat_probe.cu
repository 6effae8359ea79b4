// Latency probe: cycles per dependent FP64 div / sqrt / rsqrt / DFMA, per
// __syncthreads (256 threads), per dependent shared-memory load round trip.
#include <cstdio>
__global__ void k(double* out, long long* cyc, double x0, int n) {
  __shared__ double sm[256];
  __shared__ int si[256];
  double x = x0 + threadIdx.x * 1e-9;
  sm[threadIdx.x] = x;
  si[threadIdx.x] = (threadIdx.x + 1) & 255;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 2.0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 3.0);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 0.999, 1e-3);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t5 = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < n; ++i) p = si[p];
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) { x = x * sm[p & 255] + 1.0; sm[threadIdx.x] = x; __syncthreads(); }
  long long t7 = clock64();
  float xf = (float)x;
  for (int i = 0; i < n; ++i) xf = 1.0f / (xf + 1.0f);
  long long t8 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
    cyc[5] = t6 - t5; cyc[6] = t7 - t6; cyc[7] = t8 - t7;
  }
  out[threadIdx.x] = x + p + xf;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 256); cudaMalloc(&c, 8 * 8);
  const int n = 1000;
  k<<<1, 256>>>(o, c, 0.5, n);
  k<<<1, 256>>>(o, c, 0.5, n);
  long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
  const char* nm[8] = {"fp64 div", "fp64 sqrt", "fp64 rsqrt", "dfma", "syncthreads(256)", "lds chase",
                       "lds+st+sync", "fp32 div"};
  for (int i = 0; i < 8; ++i) printf("%-18s %7.1f cycles\n", nm[i], h[i] / (double)n);
  return 0;
}
