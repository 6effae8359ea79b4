// Pageable host <-> device copies through a ring of pinned staging chunks.
//
// The reference API takes numpy arrays, i.e. pageable host memory, and a
// pageable cudaMemcpy moves it at ~11 GB/s on the B200 box (the driver stages
// it through a small pinned buffer with one CPU thread) against ~55 GB/s for
// pinned memory. kst_copy_staged splits the copy into CH-byte chunks: worker
// threads memcpy pageable <-> pinned chunks while the copy engine moves the
// previous ones, so the host memcpy (one thread ~14 GB/s) runs on several
// cores and overlaps the DMA. A chunk's pinned slot is reused only after the
// event recorded behind its previous DMA has completed.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <memory>
#include <thread>
#include <vector>

#include "common.cuh"

namespace {

constexpr size_t kStageChunk = 4u << 20;  // 4 MB chunks
constexpr int kMaxSlots = 32;

int stage_ring(kst_ctx* ctx, int nslots) {
  const size_t want = kStageChunk * nslots;
  if (ctx->stage_bytes < want) {
    if (ctx->stage) {
      cudaDeviceSynchronize();
      cudaFreeHost(ctx->stage);
      ctx->stage = nullptr;
      ctx->stage_bytes = 0;
    }
    if (cudaMallocHost(&ctx->stage, want) != cudaSuccess) {
      cudaGetLastError();
      ctx->stage = nullptr;
      return set_err(ctx, KST_ERR_CUDA, "copy_staged: pinned staging (%zu bytes)", want);
    }
    ctx->stage_bytes = want;
  }
  for (int s = 0; s < nslots; ++s)
    if (!ctx->stage_ev[s]) KST_CUDA(ctx, cudaEventCreateWithFlags(&ctx->stage_ev[s], cudaEventDisableTiming));
  return KST_OK;
}

inline void spin_until(const std::atomic<int>& a, int v) {
  while (a.load(std::memory_order_acquire) < v) std::this_thread::yield();
}

}  // namespace

extern "C" int kst_copy_staged(kst_ctx* ctx, void* dst, const void* src, size_t bytes, int dir,
                               int threads, void* stream) {
  CTX_GUARD(ctx);
  if (dir != 0 && dir != 1) return set_err(ctx, KST_ERR_DIMENSION, "copy_staged: dir must be 0 or 1");
  if (bytes == 0) return KST_OK;
  if (!dst || !src) return set_err(ctx, KST_ERR_DIMENSION, "copy_staged: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int nth = std::max(1, std::min(threads, 16));
  const int nslots = std::min(kMaxSlots, std::max(4, 2 * nth));
  const int64_t nch = (int64_t)((bytes + kStageChunk - 1) / kStageChunk);
  if (nch <= 1) {  // one chunk: nothing to overlap
    KST_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, dir == 0 ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost, st));
    if (dir == 1) KST_CUDA(ctx, cudaStreamSynchronize(st));
    return KST_OK;
  }
  KST_TRY(stage_ring(ctx, nslots));
  char* ring = (char*)ctx->stage;
  const int device = ctx->device;
  std::unique_ptr<std::atomic<int>[]> flag(new std::atomic<int>[nch]);
  for (int64_t i = 0; i < nch; ++i) flag[i].store(0, std::memory_order_relaxed);
  std::atomic<int64_t> next{0};
  std::atomic<int> issued{0};  // chunks whose DMA (and slot event) the main thread has enqueued
  std::atomic<int> failed{0};
  auto len_of = [&](int64_t i) { return std::min(kStageChunk, bytes - (size_t)i * kStageChunk); };
  auto worker = [&]() {
    cudaSetDevice(device);
    for (;;) {
      const int64_t i = next.fetch_add(1);
      if (i >= nch) break;
      const int slot = (int)(i % nslots);
      char* sp = ring + (size_t)slot * kStageChunk;
      if (dir == 0) {
        // the slot's previous chunk (i - nslots) must have left it
        if (i >= nslots) {
          spin_until(issued, (int)(i - nslots + 1));
          if (cudaEventSynchronize(ctx->stage_ev[slot]) != cudaSuccess) failed.store(1);
        }
        std::memcpy(sp, (const char*)src + (size_t)i * kStageChunk, len_of(i));
      } else {
        spin_until(issued, (int)(i + 1));  // this chunk's DMA is enqueued
        if (cudaEventSynchronize(ctx->stage_ev[slot]) != cudaSuccess) failed.store(1);
        std::memcpy((char*)dst + (size_t)i * kStageChunk, sp, len_of(i));
      }
      flag[i].store(1, std::memory_order_release);
    }
  };
  std::vector<std::thread> pool;
  pool.reserve(nth);
  for (int t = 0; t < nth; ++t) pool.emplace_back(worker);
  int rc = KST_OK;
  for (int64_t i = 0; i < nch && rc == KST_OK; ++i) {
    const int slot = (int)(i % nslots);
    char* sp = ring + (size_t)slot * kStageChunk;
    cudaError_t e;
    if (dir == 0) {
      spin_until(flag[i], 1);  // staged
      e = cudaMemcpyAsync((char*)dst + (size_t)i * kStageChunk, sp, len_of(i), cudaMemcpyHostToDevice, st);
    } else {
      if (i >= nslots) spin_until(flag[i - nslots], 1);  // the slot was drained
      e = cudaMemcpyAsync(sp, (const char*)src + (size_t)i * kStageChunk, len_of(i), cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaEventRecord(ctx->stage_ev[slot], st);
    if (e != cudaSuccess) rc = set_err(ctx, KST_ERR_CUDA, "copy_staged: %s", cudaGetErrorString(e));
    issued.store((int)(i + 1), std::memory_order_release);
  }
  if (rc != KST_OK) {  // release waiting workers: nothing further is enqueued
    issued.store((int)nch + nslots, std::memory_order_release);
    next.store(nch);
  }
  for (auto& t : pool) t.join();
  if (rc == KST_OK && failed.load()) rc = set_err(ctx, KST_ERR_CUDA, "copy_staged: event wait failed");
  return rc;
}
