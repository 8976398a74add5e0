// Host <-> device copies of the host-buffer C-ABI entry points (the
// LinearMap plug-in path of INTEGRATION.md: Eigen vectors in pageable host
// memory). A plain cudaMemcpy from pageable memory is staged by the driver
// through a small bounce buffer on one CPU thread. Here the copy is a
// pipeline over K pinned chunks: CPU threads (OpenMP) copy chunk i between
// the caller's buffer and a pinned chunk while the DMA engine moves chunk
// i - 1 over PCIe. Host pointers that are already page-locked (registered or
// cudaHostAlloc'd) go straight to one cudaMemcpyAsync.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cstring>
#include <mutex>

#include "stmg.hpp"

namespace stmgb {

namespace {

constexpr int kChunks = 4;
constexpr size_t kChunkBytes = size_t(32) << 20;

struct Staging {
  double* pin[kChunks] = {};
  cudaEvent_t ev[kChunks] = {};
  cudaStream_t stream = nullptr;
  int device = -1;
};

std::mutex g_mu;
Staging g_st;

Staging& staging() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (g_st.device != dev) {
    // first use on this device (one staging set per process)
    for (int i = 0; i < kChunks; ++i) {
      if (g_st.pin[i]) cudaFreeHost(g_st.pin[i]);
      if (g_st.ev[i]) cudaEventDestroy(g_st.ev[i]);
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&g_st.pin[i]), kChunkBytes, cudaHostAllocDefault),
                 "cudaHostAlloc staging");
      cuda_check(cudaEventCreateWithFlags(&g_st.ev[i], cudaEventDisableTiming), "staging event");
    }
    if (g_st.stream) cudaStreamDestroy(g_st.stream);
    cuda_check(cudaStreamCreateWithFlags(&g_st.stream, cudaStreamNonBlocking), "staging stream");
    g_st.device = dev;
  }
  return g_st;
}

bool page_locked(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void par_memcpy(void* dst, const void* src, size_t n) {
  const int T = std::max(1, std::min(omp_get_max_threads(), static_cast<int>(n >> 20)));
  if (T == 1) {
    std::memcpy(dst, src, n);
    return;
  }
#pragma omp parallel for num_threads(T) schedule(static)
  for (int t = 0; t < T; ++t) {
    const size_t a = (n * t / T) & ~size_t(63), b = t + 1 == T ? n : ((n * (t + 1) / T) & ~size_t(63));
    std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
  }
}

}  // namespace

void copy_to_device(double* d_dst, const double* h_src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (page_locked(h_src)) {
    cuda_check(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, s), "H2D");
    cuda_check(cudaStreamSynchronize(s), "H2D sync");
    return;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  Staging& S = staging();
  cuda_check(cudaStreamSynchronize(s), "H2D order");
  const char* src = reinterpret_cast<const char*>(h_src);
  char* dst = reinterpret_cast<char*>(d_dst);
  for (size_t off = 0, i = 0; off < bytes; off += kChunkBytes, ++i) {
    const int b = static_cast<int>(i % kChunks);
    const size_t n = std::min(kChunkBytes, bytes - off);
    cuda_check(cudaEventSynchronize(S.ev[b]), "staging reuse");
    par_memcpy(S.pin[b], src + off, n);
    cuda_check(cudaMemcpyAsync(dst + off, S.pin[b], n, cudaMemcpyHostToDevice, S.stream), "H2D chunk");
    cuda_check(cudaEventRecord(S.ev[b], S.stream), "staging record");
  }
  cuda_check(cudaStreamSynchronize(S.stream), "H2D drain");
}

void copy_to_host(double* h_dst, const double* d_src, size_t bytes, cudaStream_t s) {
  if (bytes == 0) return;
  if (page_locked(h_dst)) {
    cuda_check(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "D2H sync");
    return;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  Staging& S = staging();
  cuda_check(cudaStreamSynchronize(s), "D2H order");
  const char* src = reinterpret_cast<const char*>(d_src);
  char* dst = reinterpret_cast<char*>(h_dst);
  const size_t n_chunks = (bytes + kChunkBytes - 1) / kChunkBytes;
  auto issue = [&](size_t i) {
    const int b = static_cast<int>(i % kChunks);
    const size_t off = i * kChunkBytes, n = std::min(kChunkBytes, bytes - off);
    cuda_check(cudaMemcpyAsync(S.pin[b], src + off, n, cudaMemcpyDeviceToHost, S.stream), "D2H chunk");
    cuda_check(cudaEventRecord(S.ev[b], S.stream), "staging record");
  };
  for (size_t i = 0; i < std::min<size_t>(kChunks, n_chunks); ++i) issue(i);
  for (size_t i = 0; i < n_chunks; ++i) {
    const int b = static_cast<int>(i % kChunks);
    const size_t off = i * kChunkBytes, n = std::min(kChunkBytes, bytes - off);
    cuda_check(cudaEventSynchronize(S.ev[b]), "D2H wait");
    par_memcpy(dst + off, S.pin[b], n);
    if (i + kChunks < n_chunks) issue(i + kChunks);
  }
}

}  // namespace stmgb
