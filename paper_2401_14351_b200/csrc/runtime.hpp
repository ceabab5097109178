// Host runtime internals: per-GPU contexts, NCCL shim, load objects.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <mutex>
#include <thread>

#include "common.hpp"
#include "kernels.cuh"

namespace sllm {

[[noreturn]] void cuda_fail(cudaError_t e, const char* what);
#define SLLM_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) ::sllm::cuda_fail(_e, #call);  \
  } while (0)

constexpr int kMaxStreams = 8;
constexpr uint32_t kTile = 64u << 10;  // bytes per kernel work tile
constexpr uint64_t kWindowBytes = 64ull << 20;   // min bytes per copy submission / kernel launch
constexpr uint64_t kVerifyBytes = 512ull << 20;  // CE mode: min bytes per verification launch

// Library-owned, per-GPU resources reused across loads (no allocation in the hot path).
struct DeviceCtx {
  int dev = -1;
  std::mutex mu;
  cudaStream_t streams[kMaxStreams] = {};
  cudaStream_t comm_stream = nullptr;
  cudaStream_t kern_stream = nullptr;
  void ensure(int n_streams);                          // caller holds mu, device set
};
DeviceCtx& device_ctx(int dev);

// ---- stream gates (gate.cpp) -------------------------------------------------------
struct Gate {
  int slot = -1;
  uint32_t value = 0;
  uint32_t* host = nullptr;
  uint64_t dev = 0;
};
Gate gate_acquire();
void gate_release(const Gate& g);
void gate_wait(cudaStream_t s, const Gate& g);        // enqueue "wait until flag >= value"
void gate_open_device(cudaStream_t s, const Gate& g); // enqueue "flag = value"
void gate_open_host(const Gate& g);                    // flag = value, now

// ---- NCCL (loaded with dlopen; only the calls the fan-out needs) -------------------
struct Nccl;
const Nccl& nccl();  // throws SLLM_E_NCCL if libnccl.so.2 cannot be loaded
void nccl_bcast_group(sllm_comm* comm, const std::vector<std::pair<uint64_t, uint64_t>>& ranges_by_root,
                      uint8_t* buf, cudaStream_t s);
int comm_nranks(const sllm_comm* c);
int comm_rank(const sllm_comm* c);
int comm_device(const sllm_comm* c);

}  // namespace sllm
