// capi_util.cu -- C-ABI error state + primitive entry points (GEMM) of libcoserve_cuda.so.
#include <cstdlib>
#include <string>

#include "coserve_cuda.h"
#include "kernels.h"

namespace cs {
std::atomic<long> g_launches{0};
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("CS_PDL");
    return !(v && std::atoi(v) == 0);
  }();
  return on;
}
thread_local std::string g_last_error;
int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
}  // namespace cs

extern "C" {

const char* cs_last_error(void) { return cs::g_last_error.c_str(); }



int cs_version(void) { return CS_ABI_VERSION; }

int cs_gemm_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                 int64_t M, int64_t N, int64_t K, int epi, const float* bias, int bn, int splits,
                 void* stream) {
  cs::GemmDesc d;
  d.A = A;
  d.lda = lda;
  d.B = B;
  d.ldb = ldb;
  d.C = C;
  d.ldc = ldc;
  d.M = M;
  d.N = N;
  d.K = K;
  d.epi = epi;
  d.bias = bias;
  d.bn = bn;
  d.splits = splits;
  if (!A || !B || !C) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_gemm_bf16: null pointer");
  if (bn != 0 && bn != 16 && bn != 32 && bn != 64 && bn != 128 && bn != 256)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_gemm_bf16: bn must be 0,16,32,64,128,256");
  cudaError_t e = cs::gemm_tn(d, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return cs::set_error(e == cudaErrorInvalidValue ? CS_ERR_INVALID_ARGUMENT : CS_ERR_CUDA,
                         std::string("cs_gemm_bf16: ") + cudaGetErrorString(e));
  return CS_OK;
}

int cs_gemm_bf16_mn(const void* A, int64_t lda, const void* B, int64_t ldb, void* C, int64_t ldc,
                    int64_t M, int64_t N, int64_t K, int epi, int bn, int splits, void* stream) {
  cs::GemmDesc d;
  d.A = A;
  d.lda = lda;
  d.B = B;
  d.ldb = ldb;
  d.C = C;
  d.ldc = ldc;
  d.M = M;
  d.N = N;
  d.K = K;
  d.epi = epi;
  d.bn = bn;
  d.splits = splits;
  d.b_mn = 1;
  if (!A || !B || !C) return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_gemm_bf16_mn: null pointer");
  if (bn != 0 && bn != 64 && bn != 128 && bn != 256)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_gemm_bf16_mn: bn must be 0,64,128,256");
  if (ldb < N || (N % 8) != 0)
    return cs::set_error(CS_ERR_INVALID_ARGUMENT, "cs_gemm_bf16_mn: need ldb >= N and N % 8 == 0");
  cudaError_t e = cs::gemm_tn(d, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess)
    return cs::set_error(e == cudaErrorInvalidValue ? CS_ERR_INVALID_ARGUMENT : CS_ERR_CUDA,
                         std::string("cs_gemm_bf16_mn: ") + cudaGetErrorString(e));
  return CS_OK;
}

}  // extern "C"
