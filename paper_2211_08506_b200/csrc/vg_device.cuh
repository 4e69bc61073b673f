// vg_device.cuh — per-call device selection and once-per-device kernel
// configuration, shared by the library's translation units.
//
// Every C-ABI entry point that launches work makes the device that owns its
// output (or workspace) pointer current for the duration of the call and
// restores the caller's device afterwards, so that a caller whose current
// device differs (e.g. GridPipeline(device="cuda:1") from a thread whose
// current device is 0) launches on the right GPU instead of failing with an
// invalid resource handle.
#pragma once

#include <cuda_runtime.h>

#include <mutex>

namespace vgdev {

class DeviceGuard {
 public:
  explicit DeviceGuard(const void* dev_ptr) {
    if (dev_ptr == nullptr || cudaGetDevice(&prev_) != cudaSuccess) return;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, dev_ptr) != cudaSuccess) {
      cudaGetLastError();   // not a CUDA pointer: leave the current device alone
      return;
    }
    if (a.type == cudaMemoryTypeDevice && a.device >= 0 && a.device != prev_) {
      if (cudaSetDevice(a.device) == cudaSuccess) switched_ = true;
    }
  }
  ~DeviceGuard() {
    if (switched_) cudaSetDevice(prev_);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;

 private:
  int prev_ = 0;
  bool switched_ = false;
};

// Kernel attributes (dynamic shared memory limit, carveout) must be set on
// each device before the first launch that needs them. `configure` runs at
// most once per device for a given `Once` object, under a mutex, and the
// device is marked configured only after it returned cudaSuccess: a second
// thread never launches before the attributes are in place, and a failed
// set is retried by the next call.
struct Once {
  std::mutex mu;
  unsigned long long done = 0;   // bit d: device d configured
};

template <typename F>
cudaError_t configure_once(Once& once, F&& configure) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(once.mu);
  if (once.done & bit) return cudaSuccess;
  e = configure();
  if (e == cudaSuccess) once.done |= bit;
  return e;
}

}  // namespace vgdev
