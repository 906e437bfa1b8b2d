// abft_common.cuh — shared host/device definitions of the B200 ABFT library.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/abft_b200.h"

namespace abft {

// thread-local last-error message behind abft_last_error()
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_check(cudaError_t e, const char* what);

int num_sms();
int max_smem_optin();

// tolerance ratio r of checksum.py:143-148 (plus the bf16 extension, r = 2^-7)
__host__ __device__ inline double tol_ratio(int numeric) {
  switch (numeric) {
    case ABFT_NUM_BINARY16: return 0.0009765625;             // 2^-10
    case ABFT_NUM_BINARY32: return 1.1920928955078125e-07;   // 2^-23
    case ABFT_NUM_BF16: return 0.0078125;                    // 2^-7
    default: return 0.0;                                     // exact-int
  }
}

// tau = r * K * max(|lhs|, |rhs|, 1)  (checksum.py:143-148)
__host__ __device__ inline double tolerance(double r, int k, double lhs, double rhs) {
  if (r == 0.0) return 0.0;
  double m = fabs(lhs) > fabs(rhs) ? fabs(lhs) : fabs(rhs);
  if (m < 1.0) m = 1.0;
  return r * (double)k * m;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// explicit im2col (abft_aux.cu) for the few-channel conv mode
int launch_im2col(const void* x, int n, int h, int w, int c, int cr, int r, int s, int sh, int sw, int ph, int pw,
                  int P, int Q, int K, int ld, void* out, cudaStream_t st);

}  // namespace abft
