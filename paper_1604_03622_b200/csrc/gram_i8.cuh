// Shared pieces of the int8 tensor-core Gram engines (gram_ozaki.cu: 7-bit
// slices; gram_crt.cu: modular residues): column exponents and the dlopen'd
// cuBLAS int8 GEMM entry points.
#pragma once
#include <cublas_v2.h>  // types only: every cuBLAS entry point is bound with dlsym

#include <climits>

#include "common.cuh"

namespace kst {
namespace i8 {

constexpr int kNaNExpo = INT_MIN;  // exponent sentinel of a non-finite column

// expo[a] = smallest E with max_k max(|re|, |im|) of column a < 2^E
// (kNaNExpo for non-finite columns, 0 for all-zero ones); grid cdiv(d, 32), block (32, 8)
__global__ void colmax_kernel(const cplx* __restrict__ X, int64_t n, int64_t d,
                              int* __restrict__ expo);

struct Blas {
  bool tried = false, ok = false;
  cublasStatus_t (*create)(cublasHandle_t*) = nullptr;
  cublasStatus_t (*set_stream)(cublasHandle_t, cudaStream_t) = nullptr;
  cublasStatus_t (*gemm_ex)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int,
                            const void*, const void*, cudaDataType, int, const void*, cudaDataType,
                            int, const void*, void*, cudaDataType, int, cublasComputeType_t,
                            cublasGemmAlgo_t) = nullptr;
  cublasStatus_t (*gemm_batched_ex)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int,
                                    int, const void*, const void* const[], cudaDataType, int,
                                    const void* const[], cudaDataType, int, const void*,
                                    void* const[], cudaDataType, int, int, cublasComputeType_t,
                                    cublasGemmAlgo_t) = nullptr;
};
extern Blas g_blas;
bool load_blas();
// the context's cuBLAS handle bound to `st` (created on first use); nullptr on failure
cublasHandle_t blas_handle(kst_ctx* ctx, cudaStream_t st);

}  // namespace i8
}  // namespace kst
