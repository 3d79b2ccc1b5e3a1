// Device properties and kernel attributes, cached per (device, kernel) under a mutex, so a
// process that drives several GPUs (or several host threads) sets every attribute on every
// device it launches on.
#include <map>
#include <mutex>
#include <tuple>

#include "internal.cuh"

namespace igacd {

static std::mutex g_mu;

static int current_device() {
  int dev = 0;
  IGACD_CUDA(cudaGetDevice(&dev));
  return dev;
}

int num_sms() {
  static std::map<int, int> cache;
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int n = 0;
  IGACD_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
  if (n <= 0) n = 148;
  cache[dev] = n;
  return n;
}

void ensure_smem_attr(const void* func, size_t bytes) {
  if (bytes <= 48 * 1024) return;
  static std::map<std::pair<int, const void*>, size_t> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_mu);
  size_t& v = done[{dev, func}];
  if (v >= bytes) return;
  IGACD_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  v = bytes;
}

int max_active_blocks(const void* func, int threads, size_t smem) {
  static std::map<std::tuple<int, const void*, int, size_t>, int> cache;
  const int dev = current_device();
  std::lock_guard<std::mutex> g(g_mu);
  auto key = std::make_tuple(dev, func, threads, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int occ = 0;
  IGACD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, func, threads, smem));
  occ = occ < 1 ? 1 : occ;
  cache[key] = occ;
  return occ;
}

}  // namespace igacd
