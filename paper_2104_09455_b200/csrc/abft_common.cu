// abft_common.cu — error plumbing and device introspection of the C-ABI.
#include <mutex>
#include <string>

#include "abft_common.cuh"

namespace abft {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ABFT_OK;
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return ABFT_E_CUDA;
}

static int device_attr(cudaDeviceAttr attr) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess) return 0;
  return v;
}

// cached per device ordinal (one process drives one GPU in this design)
int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) cached[dev] = device_attr(cudaDevAttrMultiProcessorCount);
  return cached[dev] > 0 ? cached[dev] : 148;
}

int max_smem_optin() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 232448;
  if (cached[dev] == 0) cached[dev] = device_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin);
  return cached[dev] > 0 ? cached[dev] : 232448;
}

}  // namespace abft

extern "C" __attribute__((visibility("default"))) const char* abft_last_error(void) { return abft::g_last_error.c_str(); }
extern "C" __attribute__((visibility("default"))) int abft_version(void) { return 100; }  // 0.1.0
extern "C" __attribute__((visibility("default"))) int abft_struct_size(int which) {
  switch (which) {
    case 0: return (int)sizeof(abft_gemm_args_t);
    case 1: return (int)sizeof(abft_conv_args_t);
    case 2: return (int)sizeof(abft_global_task_t);
    case 3: return (int)sizeof(abft_verdict_t);
    case 4: return (int)sizeof(abft_thread_verdict_t);
    case 5: return (int)sizeof(abft_fault_t);
    default: return -1;
  }
}
extern "C" __attribute__((visibility("default"))) int abft_device_sms(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return 0;
  return abft::num_sms();
}
