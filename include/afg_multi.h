// afg_multi.h - C++ multi-GPU host API: one host thread per device.
//
// The reference is single-threaded per interpreter instance and safe across
// instances; it has no device concept. The B200 build runs
// the BASELINE's sharded configs as one host thread per GPU: each worker
// thread binds its device once (cudaSetDevice), owns a non-blocking stream,
// and -- for groups of more than one device -- one NCCL communicator from a
// single ncclCommInitAll, so a job can call any afg_* entry point (all are
// stream-ordered and reentrant per device) and the collective ones
// (afg_gemm_splitk) on its rank. The C ABI mirror is afg_group_* (afg.h).
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "afg.h"

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

namespace afg {

class DeviceGroup {
 public:
  // with_comms: create one NCCL communicator per device (ncclCommInitAll) for
  // groups of more than one distinct device
  explicit DeviceGroup(const std::vector<int>& devices, bool with_comms = true);
  ~DeviceGroup();
  DeviceGroup(const DeviceGroup&) = delete;
  DeviceGroup& operator=(const DeviceGroup&) = delete;

  int size() const { return static_cast<int>(devices_.size()); }
  int device(int rank) const { return devices_.at(rank); }
  void* stream(int rank) const { return streams_.at(rank); }   // cudaStream_t
  void* comm(int rank) const { return comms_.at(rank); }       // ncclComm_t (nullptr for 1 device)

  // Runs fn(rank, device, stream, comm) on every device's thread concurrently
  // and returns when all have returned (the enqueued GPU work may still run).
  void run(const std::function<void(int rank, int device, void* stream, void* comm)>& fn);
  // Waits for every device's stream.
  afg_status synchronize();

 private:
  struct Worker;
  std::vector<int> devices_;
  std::vector<std::unique_ptr<Worker>> workers_;
  std::vector<void*> streams_;
  std::vector<void*> comms_;
};

}  // namespace afg

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
