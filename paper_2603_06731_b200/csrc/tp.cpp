// tp.cpp - multi-GPU plumbing of the C ABI: NCCL communicators, the split-K /
// tensor-parallel GEMM, and the thread-per-device group (include/afg_multi.h).
//
// The reference has no multi-device path (its only concurrency contract is
// independent interpreter instances); BASELINE's multi-GPU
// configs shard rows / heads / batch with no collective, and the split-K
// (row-parallel) GEMM is the one config with a real exchange step (SURVEY.md
// §8e): every rank multiplies its K slice, the fp32 partial sums are reduced
// over NVLink by NCCL (reduce-scatter to row blocks, or all-reduce), and the
// bias / activation epilogue runs on the reduced sum.
//
// libnccl is resolved at first use with dlopen("libnccl.so.2"): a process that
// already loaded NCCL (PyTorch's torch.distributed) shares that copy, and
// libafg.so itself carries no link-time NCCL dependency (the CPU test suite
// loads it without one).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/afg.h"
#include "../../include/afg_multi.h"
#include "afg_internal.h"

namespace afg {
namespace {

struct Nccl {
  bool ok = false;
  std::string why;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommInitAll) commInitAll = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclCommCount) commCount = nullptr;
  decltype(&ncclCommUserRank) commUserRank = nullptr;
  decltype(&ncclReduceScatter) reduceScatter = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
  decltype(&ncclGroupStart) groupStart = nullptr;
  decltype(&ncclGroupEnd) groupEnd = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
#define AFG_SYM(field, name)                                            \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, #name));       \
  if (!n.field) {                                                       \
    n.why = "libnccl lacks " #name;                                     \
    return;                                                             \
  }
    AFG_SYM(getUniqueId, ncclGetUniqueId)
    AFG_SYM(commInitRank, ncclCommInitRank)
    AFG_SYM(commInitAll, ncclCommInitAll)
    AFG_SYM(commDestroy, ncclCommDestroy)
    AFG_SYM(commCount, ncclCommCount)
    AFG_SYM(commUserRank, ncclCommUserRank)
    AFG_SYM(reduceScatter, ncclReduceScatter)
    AFG_SYM(allReduce, ncclAllReduce)
    AFG_SYM(errorString, ncclGetErrorString)
    AFG_SYM(groupStart, ncclGroupStart)
    AFG_SYM(groupEnd, ncclGroupEnd)
#undef AFG_SYM
    n.ok = true;
  });
  return n;
}

afg_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return AFG_OK;
  return set_error(AFG_ERR_NCCL, "%s: %s", what, nccl().errorString(r));
}

afg_status need_nccl() {
  if (!nccl().ok) return set_error(AFG_ERR_NCCL, "%s", nccl().why.c_str());
  return AFG_OK;
}

}  // namespace

// --------------------------------------------------------- DeviceGroup ---

struct DeviceGroup::Worker {
  int device = 0;
  std::thread th;
  std::mutex mu;
  std::condition_variable cv;
  std::function<void()> job;
  bool stop = false, busy = false;
};

DeviceGroup::DeviceGroup(const std::vector<int>& devices, bool with_comms) : devices_(devices) {
  if (devices_.empty()) throw std::invalid_argument("afg DeviceGroup: no devices");
  for (int d : devices_) {
    auto w = std::make_unique<Worker>();
    w->device = d;
    Worker* wp = w.get();
    w->th = std::thread([wp] {
      cudaSetDevice(wp->device);  // the thread's device for its whole life
      std::unique_lock<std::mutex> lk(wp->mu);
      while (true) {
        wp->cv.wait(lk, [wp] { return wp->stop || wp->busy; });
        if (wp->stop) return;
        lk.unlock();
        wp->job();
        lk.lock();
        wp->busy = false;
        wp->cv.notify_all();
      }
    });
    workers_.push_back(std::move(w));
  }
  streams_.resize(devices_.size());
  std::vector<afg_status> st(devices_.size(), AFG_OK);
  run([&](int rank, int, void*, void*) {
    cudaStream_t s = nullptr;
    st[rank] = cuda_status(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    streams_[rank] = s;
  });
  comms_.assign(devices_.size(), nullptr);
  const bool distinct =
      std::set<int>(devices_.begin(), devices_.end()).size() == devices_.size();
  if (with_comms && distinct && devices_.size() > 1 && need_nccl() == AFG_OK) {
    std::vector<ncclComm_t> c(devices_.size());
    if (nccl().commInitAll(c.data(), static_cast<int>(devices_.size()), devices_.data()) ==
        ncclSuccess)
      for (size_t i = 0; i < c.size(); ++i) comms_[i] = c[i];
  }
}

DeviceGroup::~DeviceGroup() {
  run([&](int rank, int, void* s, void* comm) {
    if (comm) nccl().commDestroy(static_cast<ncclComm_t>(comm));
    if (s) cudaStreamDestroy(static_cast<cudaStream_t>(s));
    (void)rank;
  });
  for (auto& w : workers_) {
    {
      std::lock_guard<std::mutex> lk(w->mu);
      w->stop = true;
    }
    w->cv.notify_all();
    w->th.join();
  }
}

void DeviceGroup::run(const std::function<void(int, int, void*, void*)>& fn) {
  for (size_t r = 0; r < workers_.size(); ++r) {
    Worker* w = workers_[r].get();
    std::lock_guard<std::mutex> lk(w->mu);
    w->job = [this, &fn, r] {
      fn(static_cast<int>(r), devices_[r], r < streams_.size() ? streams_[r] : nullptr,
         r < comms_.size() ? comms_[r] : nullptr);
    };
    w->busy = true;
    w->cv.notify_all();
  }
  for (auto& w : workers_) {
    std::unique_lock<std::mutex> lk(w->mu);
    w->cv.wait(lk, [&] { return !w->busy; });
  }
}

afg_status DeviceGroup::synchronize() {
  std::vector<afg_status> st(workers_.size(), AFG_OK);
  run([&](int rank, int, void* s, void*) {
    st[rank] = cuda_status(cudaStreamSynchronize(static_cast<cudaStream_t>(s)), "sync");
  });
  for (afg_status x : st)
    if (x != AFG_OK) return x;
  return AFG_OK;
}

}  // namespace afg

using namespace afg;

extern "C" {

afg_status afg_comm_unique_id(void* id_out) {
  if (!id_out) return set_error(AFG_ERR_INVALID_ARG, "afg_comm_unique_id: null output");
  afg_status st = need_nccl();
  if (st != AFG_OK) return st;
  ncclUniqueId id;
  st = nccl_status(nccl().getUniqueId(&id), "ncclGetUniqueId");
  if (st == AFG_OK) std::memcpy(id_out, &id, sizeof(id));
  return st;
}

afg_status afg_comm_init_rank(void** comm, int world, const void* id, int rank) {
  if (!comm || !id || world < 1 || rank < 0 || rank >= world)
    return set_error(AFG_ERR_INVALID_ARG, "afg_comm_init_rank: bad arguments");
  afg_status st = need_nccl();
  if (st != AFG_OK) return st;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t c = nullptr;
  st = nccl_status(nccl().commInitRank(&c, world, u, rank), "ncclCommInitRank");
  *comm = st == AFG_OK ? c : nullptr;
  return st;
}

afg_status afg_comm_init_all(void** comms, int ndev, const int* devices) {
  if (!comms || ndev < 1) return set_error(AFG_ERR_INVALID_ARG, "afg_comm_init_all: bad arguments");
  afg_status st = need_nccl();
  if (st != AFG_OK) return st;
  std::vector<ncclComm_t> c(ndev);
  st = nccl_status(nccl().commInitAll(c.data(), ndev, devices), "ncclCommInitAll");
  for (int i = 0; i < ndev; ++i) comms[i] = st == AFG_OK ? c[i] : nullptr;
  return st;
}

afg_status afg_comm_destroy(void* comm) {
  if (!comm) return AFG_OK;
  afg_status st = need_nccl();
  if (st != AFG_OK) return st;
  return nccl_status(nccl().commDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
}

size_t afg_gemm_splitk_workspace(int64_t M, int64_t N, int world, int mode) {
  if (M <= 0 || N <= 0 || world < 1) return 0;
  const size_t part = static_cast<size_t>(M * N) * 4;
  const size_t recv = mode == AFG_SPLITK_REDUCE_SCATTER ? part / world : 0;
  return ((part + 255) & ~size_t(255)) + recv + 256;
}

afg_status afg_gemm_splitk(const void* A, int64_t lda, const void* B, int64_t ldb,
                           const float* bias, void* C, int64_t ldc, int64_t M, int64_t N,
                           int64_t K_local, afg_dtype ab_dtype, afg_dtype c_dtype,
                           afg_layout b_layout, afg_epilogue epi, void* comm, int mode,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (!comm) return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_splitk: null communicator");
  if (mode != AFG_SPLITK_REDUCE_SCATTER && mode != AFG_SPLITK_ALL_REDUCE)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_splitk: bad mode %d", mode);
  afg_status st = need_nccl();
  if (st != AFG_OK) return st;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int world = 1, rank = 0;
  if ((st = nccl_status(nccl().commCount(c, &world), "ncclCommCount")) != AFG_OK) return st;
  if ((st = nccl_status(nccl().commUserRank(c, &rank), "ncclCommUserRank")) != AFG_OK) return st;
  if (mode == AFG_SPLITK_REDUCE_SCATTER && M % world != 0)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_splitk: M=%lld not divisible by %d ranks",
                     (long long)M, world);
  if (workspace_bytes < afg_gemm_splitk_workspace(M, N, world, mode) || !workspace)
    return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_splitk: workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // one rank: its partial is the whole sum -- the fused-epilogue GEMM, no
  // fp32 round trip and no collective (NCCL would only copy the buffer)
  if (world == 1)
    return afg_gemm(A, lda, B, ldb, bias, nullptr, C, ldc, M, N, K_local, ab_dtype, c_dtype,
                    b_layout, epi, stream);
  // 1) this rank's fp32 partial product over its K slice (K1 on tcgen05)
  float* part = static_cast<float*>(workspace);
  st = afg_gemm(A, lda, B, ldb, nullptr, nullptr, part, N, M, N, K_local, ab_dtype, AFG_F32,
                b_layout, AFG_EPI_NONE, stream);
  if (st != AFG_OK) return st;
  // 2) the exchange step over NVLink: sum the partials across ranks
  const size_t part_bytes = (static_cast<size_t>(M * N) * 4 + 255) & ~size_t(255);
  const float* sum = part;
  int64_t rows = M;
  if (mode == AFG_SPLITK_REDUCE_SCATTER) {
    float* recv = reinterpret_cast<float*>(static_cast<char*>(workspace) + part_bytes);
    rows = M / world;
    st = nccl_status(nccl().reduceScatter(part, recv, static_cast<size_t>(rows * N), ncclFloat32,
                                          ncclSum, c, s),
                     "ncclReduceScatter");
    sum = recv;
  } else {
    st = nccl_status(nccl().allReduce(part, part, static_cast<size_t>(M * N), ncclFloat32, ncclSum,
                                      c, s),
                     "ncclAllReduce");
  }
  if (st != AFG_OK) return st;
  // 3) the epilogue on the reduced sum (this rank's row block, or all rows)
  if (ldc < N) return set_error(AFG_ERR_INVALID_ARG, "afg_gemm_splitk: ldc < N");
  if (ldc == N)
    return afg_epilogue_apply(sum, bias, nullptr, C, rows, N, N, epi, AFG_F32, c_dtype, stream);
  for (int64_t r = 0; r < rows; ++r) {  // strided C: one row at a time
    st = afg_epilogue_apply(sum + r * N, bias, nullptr,
                            static_cast<char*>(C) + r * ldc * dtype_bytes(c_dtype), 1, N, N, epi,
                            AFG_F32, c_dtype, stream);
    if (st != AFG_OK) return st;
  }
  return AFG_OK;
}

afg_status afg_group_create(int ndev, const int* devices, afg_group** out) {
  if (!out || ndev < 1 || !devices) return set_error(AFG_ERR_INVALID_ARG, "afg_group_create: bad arguments");
  try {
    *out = reinterpret_cast<afg_group*>(
        new DeviceGroup(std::vector<int>(devices, devices + ndev)));
    return AFG_OK;
  } catch (const std::exception& e) {
    return set_error(AFG_ERR_INTERNAL, "afg_group_create: %s", e.what());
  }
}

void afg_group_destroy(afg_group* g) { delete reinterpret_cast<DeviceGroup*>(g); }

int afg_group_size(const afg_group* g) {
  return g ? reinterpret_cast<const DeviceGroup*>(g)->size() : 0;
}

afg_status afg_group_run(afg_group* g, afg_group_fn fn, void* user) {
  if (!g || !fn) return set_error(AFG_ERR_INVALID_ARG, "afg_group_run: bad arguments");
  auto* dg = reinterpret_cast<DeviceGroup*>(g);
  std::vector<afg_status> st(dg->size(), AFG_OK);
  dg->run([&](int rank, int device, void* stream, void* comm) {
    st[rank] = fn(user, rank, device, stream, comm);
  });
  for (afg_status x : st)
    if (x != AFG_OK) return x;
  return dg->synchronize();
}

}  // extern "C"
