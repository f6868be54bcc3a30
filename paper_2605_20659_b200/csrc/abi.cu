// Miscellaneous C-ABI entry points and the per-device attribute cache.
#include <cuda_runtime.h>

#include <stdlib.h>

#include <mutex>
#include <string.h>

#include "common.cuh"

namespace ropeslr {

static thread_local cudaError_t t_last_error = cudaSuccess;
void note_cuda_error(cudaError_t e) { t_last_error = e; }

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

static Tuning& tuning_mut() {
  static Tuning t = [] {
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
    r.screen = !env_off("ROPESLR_SCREEN");
    const char* ks = getenv("ROPESLR_KEEP_SORT");
    r.keep_bitonic = ks != nullptr && ks[0] == 'b';
    r.pairs64 = !env_off("ROPESLR_PAIRS64");
    return r;
  }();
  return t;
}

const Tuning& tuning() { return tuning_mut(); }

template <typename T>
__global__ void nonfinite_scan_kernel(const T* __restrict__ a, int64_t n, uint32_t* flag, uint32_t bit) {
  bool bad = false;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !isfinite(a[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, bit);
}

int scan_nonfinite(const void* a, bool f64, int64_t n, uint32_t* flag, uint32_t bit, cudaStream_t st) {
  if (flag == nullptr || n <= 0) return ROPESLR_OK;
  const int64_t blocks = ceil_div(n, 256 * 8);
  const unsigned grid = static_cast<unsigned>(blocks < 8 * num_sms() ? blocks : 8 * num_sms());
  if (f64)
    nonfinite_scan_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(a), n, flag, bit);
  else
    nonfinite_scan_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(a), n, flag, bit);
  return launch_status();
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

extern "C" int ropeslr_set_option(const char* name, int value) {
  if (name == nullptr) return ROPESLR_ERR_NULL;
  ropeslr::Tuning& t = ropeslr::tuning_mut();
  if (!strcmp(name, "k2_online")) t.k2_online = value != 0;
  else if (!strcmp(name, "pair64")) t.pair64 = value != 0;
  else if (!strcmp(name, "schedule")) t.schedule = value != 0;
  else if (!strcmp(name, "kv_evict_last")) t.kv_evict_last = value != 0;
  else if (!strcmp(name, "scores")) t.scores = static_cast<char>(value);
  else if (!strcmp(name, "rope_tma")) t.rope_tma = value != 0;
  else if (!strcmp(name, "linear_simt")) t.linear_simt = value != 0;
  else if (!strcmp(name, "screen")) t.screen = value != 0;
  else if (!strcmp(name, "keep_bitonic")) t.keep_bitonic = value != 0;
  else if (!strcmp(name, "pairs64")) t.pairs64 = value != 0;
  else return ROPESLR_ERR_VALUE;
  return ROPESLR_OK;
}

extern "C" int ropeslr_get_option(const char* name) {
  if (name == nullptr) return ROPESLR_ERR_NULL;
  const ropeslr::Tuning& t = ropeslr::tuning();
  if (!strcmp(name, "k2_online")) return t.k2_online;
  if (!strcmp(name, "pair64")) return t.pair64;
  if (!strcmp(name, "schedule")) return t.schedule;
  if (!strcmp(name, "kv_evict_last")) return t.kv_evict_last;
  if (!strcmp(name, "scores")) return t.scores;
  if (!strcmp(name, "rope_tma")) return t.rope_tma;
  if (!strcmp(name, "linear_simt")) return t.linear_simt;
  if (!strcmp(name, "screen")) return t.screen;
  if (!strcmp(name, "keep_bitonic")) return t.keep_bitonic;
  if (!strcmp(name, "pairs64")) return t.pairs64;
  return ROPESLR_ERR_VALUE;
}

extern "C" const char* ropeslr_last_cuda_error(void) {
  return cudaGetErrorString(ropeslr::t_last_error);
}
