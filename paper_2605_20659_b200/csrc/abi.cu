// Miscellaneous C-ABI entry points and the per-device attribute cache.
#include <cuda_runtime.h>

#include <stdlib.h>

#include <mutex>

#include "common.cuh"

namespace ropeslr {

int num_sms() {
  static std::mutex mu;
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  std::lock_guard<std::mutex> lock(mu);
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

static bool env_off(const char* name) {
  const char* e = getenv(name);
  return e != nullptr && e[0] == '0';
}

const Tuning& tuning() {
  static const Tuning t = [] {
    Tuning r{};
    const char* k2 = getenv("ROPESLR_K2");
    r.k2_online = k2 != nullptr && k2[0] == 'o';
    r.pair64 = !env_off("ROPESLR_PAIR64");
    r.schedule = !env_off("ROPESLR_SCHEDULE");
    r.kv_evict_last = !env_off("ROPESLR_KV_EVICT_LAST");
    const char* sc = getenv("ROPESLR_SCORES");
    r.scores = sc != nullptr ? sc[0] : 0;
    r.rope_tma = !env_off("ROPESLR_ROPE_TMA");
    const char* lin = getenv("ROPESLR_LINEAR");
    r.linear_simt = lin != nullptr && lin[0] == 's';
    return r;
  }();
  return t;
}

}  // namespace ropeslr

extern "C" int ropeslr_abi_version(void) { return ROPESLR_ABI_VERSION; }

extern "C" const char* ropeslr_status_string(int status) {
  switch (status) {
    case ROPESLR_OK: return "ok";
    case ROPESLR_ERR_SHAPE: return "inconsistent or unsupported shape";
    case ROPESLR_ERR_DTYPE: return "unsupported dtype";
    case ROPESLR_ERR_ALIGN: return "pointer is misaligned (16 bytes; 32 for out / y_lr on the tensor-core path)";
    case ROPESLR_ERR_DIVIS: return "block dims do not divide the grid";
    case ROPESLR_ERR_LAUNCH: return "CUDA launch or runtime error";
    case ROPESLR_ERR_VALUE: return "scalar argument out of range";
    case ROPESLR_ERR_WORKSPACE: return "workspace missing or too small";
    case ROPESLR_ERR_ARCH: return "device is not an sm_100 (B200) GPU";
    case ROPESLR_ERR_NULL: return "required pointer is NULL";
    default: return "unknown status";
  }
}

extern "C" int ropeslr_device_check(int device) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) return ROPESLR_ERR_ARCH;
  int major = 0, minor = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess) return ROPESLR_ERR_ARCH;
  if (cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device) != cudaSuccess) return ROPESLR_ERR_ARCH;
  return (major == 10 && minor == 0) ? ROPESLR_OK : ROPESLR_ERR_ARCH;
}

extern "C" int64_t ropeslr_num_blocks(int64_t L, int32_t block) {
  if (L < 1 || block < 1) return 0;
  return ropeslr::ceil_div(L, block);
}
