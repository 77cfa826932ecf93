// Error reporting and device queries shared by every libpp200 entry point.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace pp200 {

namespace {
thread_local char g_err[1024] = "";
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch: %s", what, cudaGetErrorString(e));
    return PC_ERR_CUDA;
  }
  return PC_OK;
}

int num_sms() {
  static thread_local int dev = -1, sms = 0;
  int d = 0;
  cudaGetDevice(&d);
  if (d != dev) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d);
    if (sms <= 0) sms = 148;
    dev = d;
  }
  return sms;
}

}  // namespace pp200

extern "C" const char* pc_last_error(void) { return pp200::g_err; }
extern "C" int pc_version(void) { return 1; }
extern "C" int pc_device_sm_count(void) { return pp200::num_sms(); }
