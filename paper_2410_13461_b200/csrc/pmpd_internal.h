// Internal host-side helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/pmpd_b200.h"

namespace pmpd {

// Thread-local message of the last failing call (pmpd_last_error).
std::string& last_error_slot();

inline int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  last_error_slot() = buf;
  return code;
}

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(PMPD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return PMPD_OK;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline bool is_tiled(int layout) { return layout == PMPD_LAYOUT_KN || layout == PMPD_LAYOUT_NK; }

int num_sms();

}  // namespace pmpd
