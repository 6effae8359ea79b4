// Probe: time + sweep count of the shared-memory Jacobi (jacobi.cuh) on
// random Hermitian matrices, for n in {3, 8, 16, 32, 64} and block sizes.
#include <cstdio>
#include <cstdlib>
#include "../paper_1604_03622_b200/csrc/jacobi.cuh"
int set_err(kst_ctx*, int code, const char*, ...) { return code; }
using namespace kstj;
__global__ void probe(const cplx* M, int n, int* sweeps, double* vals) {
  extern __shared__ __align__(16) char sm[];
  JacSmem j = jac_carve(sm, n);
  jac_solve(j, M, n, n, 1.0);
  if (threadIdx.x == 0) { *sweeps = j.flag[1]; for (int k = 0; k < n; ++k) vals[k] = j.val[j.order[k]]; }
}
int main() {
  cplx* dM; int* ds; double* dv;
  cudaMalloc(&dM, sizeof(cplx) * 64 * 64); cudaMalloc(&ds, 4); cudaMalloc(&dv, 8 * 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)jac_smem_bytes(64));
  int sizes[] = {3, 8, 16, 32, 64};
  for (int n : sizes) {
    cplx h[64 * 64];
    srand(n);
    for (int a = 0; a < n; ++a) for (int b = 0; b <= a; ++b) {
      double x = rand() / (double)RAND_MAX - 0.5, y = a == b ? 0 : rand() / (double)RAND_MAX - 0.5;
      double sc = (a < 3 && b < 3) ? 1000.0 : 1.0;  // spread spectrum
      h[a * n + b] = make_double2(x * sc, y * sc); h[b * n + a] = make_double2(x * sc, -y * sc);
    }
    cudaMemcpy(dM, h, sizeof(cplx) * n * n, cudaMemcpyHostToDevice);
    for (int nt : {32, 256}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      probe<<<1, nt, jac_smem_bytes(n)>>>(dM, n, ds, dv);
      cudaEventRecord(e0);
      probe<<<1, nt, jac_smem_bytes(n)>>>(dM, n, ds, dv);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int sw; cudaMemcpy(&sw, ds, 4, cudaMemcpyDeviceToHost);
      printf("n=%2d threads=%3d sweeps=%2d time=%8.1f us  err=%s\n", n, nt, sw, ms * 1e3,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
