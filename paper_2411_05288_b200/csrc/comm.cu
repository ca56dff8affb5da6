// Collective backends (comm.h): NCCL, and the loopback backend that runs
// several ranks on one GPU through device mailboxes.
#include <cuda_bf16.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "comm.h"
#include "common.h"

namespace vp {

// ============================================================================
// NCCL
// ============================================================================
namespace {

ncclDataType_t nccl_type(DType d) { return d == DType::F32 ? ncclFloat32 : ncclBfloat16; }

class NcclComm final : public Comm {
 public:
  NcclComm(ncclComm_t c, int n, int r) : comm_(c) {
    nranks = n;
    rank = r;
  }
  ~NcclComm() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  const char* backend() const override { return "nccl"; }
  void all_gather(const void* send, void* recv, size_t count, DType dt, cudaStream_t st) override {
    VP_NCCL(ncclAllGather(send, recv, count, nccl_type(dt), comm_, st));
  }
  void all_reduce(const void* send, void* recv, size_t count, DType dt, RedOp op, cudaStream_t st) override {
    VP_NCCL(ncclAllReduce(send, recv, count, nccl_type(dt), op == RedOp::Sum ? ncclSum : ncclMax, comm_, st));
  }
  void broadcast(const void* send, void* recv, size_t count, DType dt, int root, cudaStream_t st) override {
    VP_NCCL(ncclBroadcast(send, recv, count, nccl_type(dt), root, comm_, st));
  }
  void group_start() override { VP_NCCL(ncclGroupStart()); }
  void group_end() override { VP_NCCL(ncclGroupEnd()); }

 private:
  ncclComm_t comm_ = nullptr;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* id128, int max_ctas) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.maxCTAs = max_ctas;  // NCCL runs beside the persistent GEMMs on the SMs they leave free
  ncclComm_t c = nullptr;
  VP_NCCL(ncclCommInitRankConfig(&c, nranks, id, rank, &cfg));
  return std::make_unique<NcclComm>(c, nranks, rank);
}

std::unique_ptr<Comm> wrap_nccl_comm(ncclComm_t comm, int nranks, int rank) {
  return std::make_unique<NcclComm>(comm, nranks, rank);
}

// ============================================================================
// Loopback
// ============================================================================
namespace {

constexpr char kMagic[8] = {'V', 'P', 'L', 'O', 'O', 'P', 'B', 'K'};
constexpr int kLbMaxRanks = 16;
constexpr size_t kMailboxBytes = size_t(32) << 20;  // per rank; larger collectives run in chunks

struct LbSlot {
  std::atomic<int> ready;
  int pid;
  int device;
  int nranks;
  uint64_t raw_mail;            // device pointer (same process)
  uint64_t raw_ev[2];           // cudaEvent_t [ready, done] (same process)
  int ipc_ok;                   // the IPC handles below are valid
  cudaIpcMemHandle_t mem;       // other processes
  cudaIpcEventHandle_t ev[2];
  unsigned char uuid[16];       // physical GPU (ranks sharing one partition its SMs)
};

struct LbShared {
  std::atomic<int> count;
  std::atomic<int> gen;
  std::atomic<int> aborted;
  LbSlot slots[kLbMaxRanks];
};

struct LbPtrs {
  const void* p[kLbMaxRanks];
};

template <typename T>
__device__ __forceinline__ float lb_load(const void* p, size_t i) {
  if constexpr (sizeof(T) == 4) return static_cast<const float*>(p)[i];
  else return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
}

// out[i] = op over ranks k = 0..n-1 (rank order: identical bits on every rank)
template <typename T>
__global__ void k_lb_reduce(LbPtrs in, int n, size_t count, int op_max, T* __restrict__ out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count; i += size_t(gridDim.x) * blockDim.x) {
    float acc = lb_load<T>(in.p[0], i);
    for (int k = 1; k < n; ++k) {
      const float x = lb_load<T>(in.p[k], i);
      acc = op_max ? fmaxf(acc, x) : acc + x;
    }
    if constexpr (sizeof(T) == 4) out[i] = acc;
    else out[i] = __float2bfloat16(acc);
  }
}

class LoopbackComm final : public Comm {
 public:
  LoopbackComm(int n, int r, const void* id128, int device) : device_(device) {
    nranks = n;
    rank = r;
    require(n >= 1 && n <= kLbMaxRanks, "loopback comm: nranks must be in 1..16");
    require(r >= 0 && r < n, "loopback comm: bad rank");
    char name[65] = {};
    std::memcpy(name, static_cast<const char*>(id128) + 8, 64);
    name_ = name;
    const int fd = shm_open(name, O_CREAT | O_RDWR, 0600);
    if (fd < 0) throw NcclError("loopback comm: shm_open(" + name_ + ") failed");
    if (ftruncate(fd, sizeof(LbShared)) != 0) {
      close(fd);
      throw NcclError("loopback comm: ftruncate failed");
    }
    void* m = mmap(nullptr, sizeof(LbShared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) throw NcclError("loopback comm: mmap failed");
    sh_ = static_cast<LbShared*>(m);
    try {
      join();
    } catch (...) {
      release();
      throw;
    }
  }
  ~LoopbackComm() override {
    // Peers may still be reading this rank's mailbox (their reads precede
    // their latest `done` event).  No rendezvous here — ranks are often
    // destroyed one after another from a single thread.  Ranks of this
    // process share the device's primary context, so a device synchronize
    // covers their streams; ranks of other processes are waited for through
    // their IPC `done` events.
    std::vector<int> devs{device_};
    for (int k = 0; sh_ && k < nranks; ++k)
      if (sh_->slots[k].pid == int(getpid())) devs.push_back(sh_->slots[k].device);
    std::sort(devs.begin(), devs.end());
    devs.erase(std::unique(devs.begin(), devs.end()), devs.end());
    for (int d : devs)
      if (cudaSetDevice(d) == cudaSuccess) cudaDeviceSynchronize();
    for (size_t i = 1; i < opened_ev_.size(); i += 2) cudaEventSynchronize(opened_ev_[i]);
    cudaSetDevice(device_);
    (void)cudaGetLastError();
    release();
  }
  const char* backend() const override { return "loopback"; }
  bool capturable() const override { return false; }
  int colocated() const override { return colocated_; }

  void all_reduce(const void* send, void* recv, size_t count, DType dt, RedOp op, cudaStream_t st) override {
    const size_t esz = dt == DType::F32 ? 4 : 2, per = kMailboxBytes / esz;
    for (size_t off = 0; off < count; off += per) {
      const size_t n = std::min(per, count - off);
      stage_in(static_cast<const char*>(send) + off * esz, n * esz, st);
      LbPtrs in{};
      for (int k = 0; k < nranks; ++k) in.p[k] = mail_[size_t(k)];
      const unsigned grid = unsigned(std::min<size_t>((n + 255) / 256, 148 * 8));
      if (dt == DType::F32)
        k_lb_reduce<float><<<grid, 256, 0, st>>>(in, nranks, n, op == RedOp::Max,
                                                  static_cast<float*>(recv) + off);
      else
        k_lb_reduce<__nv_bfloat16><<<grid, 256, 0, st>>>(in, nranks, n, op == RedOp::Max,
                                                          static_cast<__nv_bfloat16*>(recv) + off);
      VP_KCHECK();
      finish(st);
    }
  }
  void all_gather(const void* send, void* recv, size_t count, DType dt, cudaStream_t st) override {
    const size_t esz = dt == DType::F32 ? 4 : 2, per = kMailboxBytes / esz;
    for (size_t off = 0; off < count; off += per) {
      const size_t n = std::min(per, count - off);
      stage_in(static_cast<const char*>(send) + off * esz, n * esz, st);
      for (int k = 0; k < nranks; ++k)
        VP_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + (size_t(k) * count + off) * esz, mail_[size_t(k)], n * esz,
                                cudaMemcpyDefault, st));
      finish(st);
    }
  }
  void broadcast(const void* send, void* recv, size_t count, DType dt, int root, cudaStream_t st) override {
    require(root >= 0 && root < nranks, "loopback comm: bad broadcast root");
    const size_t esz = dt == DType::F32 ? 4 : 2, per = kMailboxBytes / esz;
    for (size_t off = 0; off < count; off += per) {
      const size_t n = std::min(per, count - off);
      wait_all(st, 1);  // peers are done with my mailbox
      if (rank == root)
        VP_CUDA(cudaMemcpyAsync(mail_[size_t(rank)], static_cast<const char*>(send) + off * esz, n * esz,
                                cudaMemcpyDefault, st));
      VP_CUDA(cudaEventRecord(ev_[size_t(rank)][0], st));
      barrier(timeout_);
      VP_CUDA(cudaStreamWaitEvent(st, ev_[size_t(root)][0], 0));
      if (rank != root)
        VP_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + off * esz, mail_[size_t(root)], n * esz, cudaMemcpyDefault,
                                st));
      else if (recv != send)
        VP_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + off * esz, static_cast<const char*>(send) + off * esz,
                                n * esz, cudaMemcpyDefault, st));
      VP_CUDA(cudaEventRecord(ev_[size_t(rank)][1], st));
      barrier(timeout_);
    }
  }

 private:
  // my input -> my mailbox (after every peer finished reading the previous
  // content), announce it, meet the peers, and order my stream after theirs
  void stage_in(const void* src, size_t bytes, cudaStream_t st) {
    wait_all(st, 1);
    VP_CUDA(cudaMemcpyAsync(mail_[size_t(rank)], src, bytes, cudaMemcpyDefault, st));
    VP_CUDA(cudaEventRecord(ev_[size_t(rank)][0], st));
    barrier(timeout_);
    wait_all(st, 0);
  }
  // my reads of the peers' mailboxes are issued: announce, and meet again so
  // no peer refills its mailbox before it has waited for them
  void finish(cudaStream_t st) {
    VP_CUDA(cudaEventRecord(ev_[size_t(rank)][1], st));
    barrier(timeout_);
  }
  void wait_all(cudaStream_t st, int which) {
    for (int k = 0; k < nranks; ++k)
      if (k != rank || which == 1) VP_CUDA(cudaStreamWaitEvent(st, ev_[size_t(k)][size_t(which)], 0));
  }

  // sense-reversing barrier over the shared segment (threads or processes)
  void barrier(double timeout_s) {
    const int g = sh_->gen.load(std::memory_order_acquire);
    if (sh_->count.fetch_add(1, std::memory_order_acq_rel) + 1 == nranks) {
      sh_->count.store(0, std::memory_order_relaxed);
      sh_->gen.store(g + 1, std::memory_order_release);
      return;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0; sh_->gen.load(std::memory_order_acquire) == g; ++spin) {
      if (sh_->aborted.load(std::memory_order_relaxed)) throw NcclError("loopback comm: a peer rank aborted");
      if (spin < 1000) {
        std::this_thread::yield();
        continue;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(50));
      if ((spin & 255) == 0 &&
          std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
        sh_->aborted.store(1, std::memory_order_relaxed);
        throw NcclError("loopback comm: rendezvous timed out (a peer rank is missing or issued a different "
                        "collective sequence)");
      }
    }
  }

  void join() {
    VP_CUDA(cudaSetDevice(device_));
    VP_CUDA(cudaMalloc(&own_mail_, kMailboxBytes));
    for (auto& e : own_ev_) VP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventInterprocess));
    LbSlot& s = sh_->slots[rank];
    require(s.ready.load() == 0, "loopback comm: rank joined twice");
    s.pid = int(getpid());
    s.device = device_;
    s.nranks = nranks;
    s.raw_mail = reinterpret_cast<uint64_t>(own_mail_);
    cudaDeviceProp prop;
    VP_CUDA(cudaGetDeviceProperties(&prop, device_));
    std::memcpy(s.uuid, &prop.uuid, 16);
    // IPC handles only matter for ranks in other processes (best effort here)
    bool ipc = cudaIpcGetMemHandle(&s.mem, own_mail_) == cudaSuccess;
    for (int i = 0; i < 2; ++i) {
      s.raw_ev[i] = reinterpret_cast<uint64_t>(own_ev_[i]);
      ipc = ipc && cudaIpcGetEventHandle(&s.ev[i], own_ev_[i]) == cudaSuccess;
    }
    (void)cudaGetLastError();
    s.ipc_ok = ipc ? 1 : 0;
    s.ready.store(1, std::memory_order_release);
    barrier(timeout_);  // every slot is filled
    if (rank == 0) shm_unlink(name_.c_str());  // every rank has it mapped
    mail_.assign(size_t(nranks), nullptr);
    ev_.assign(size_t(nranks), {nullptr, nullptr});
    for (int k = 0; k < nranks; ++k) {
      const LbSlot& o = sh_->slots[k];
      require(o.ready.load(std::memory_order_acquire) == 1 && o.nranks == nranks,
              "loopback comm: ranks disagree on the group size");
      if (k == rank) {
        mail_[size_t(k)] = own_mail_;
        ev_[size_t(k)] = {own_ev_[0], own_ev_[1]};
      } else if (o.pid == int(getpid())) {
        if (o.device != device_) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(o.device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) VP_CUDA(e);
          (void)cudaGetLastError();
        }
        mail_[size_t(k)] = reinterpret_cast<void*>(o.raw_mail);
        ev_[size_t(k)] = {reinterpret_cast<cudaEvent_t>(o.raw_ev[0]), reinterpret_cast<cudaEvent_t>(o.raw_ev[1])};
      } else {
        require(o.ipc_ok == 1, "loopback comm: a peer process could not export CUDA IPC handles");
        void* p = nullptr;
        VP_CUDA(cudaIpcOpenMemHandle(&p, o.mem, cudaIpcMemLazyEnablePeerAccess));
        opened_mem_.push_back(p);
        mail_[size_t(k)] = p;
        cudaEvent_t e0, e1;
        VP_CUDA(cudaIpcOpenEventHandle(&e0, o.ev[0]));
        VP_CUDA(cudaIpcOpenEventHandle(&e1, o.ev[1]));
        opened_ev_.push_back(e0);
        opened_ev_.push_back(e1);
        ev_[size_t(k)] = {e0, e1};
      }
    }
    barrier(timeout_);  // every rank opened its peers
    colocated_ = 0;
    for (int k = 0; k < nranks; ++k)
      if (std::memcmp(sh_->slots[k].uuid, sh_->slots[rank].uuid, 16) == 0) ++colocated_;
  }

  void release() {
    for (void* p : opened_mem_) cudaIpcCloseMemHandle(p);
    for (cudaEvent_t e : opened_ev_) cudaEventDestroy(e);
    opened_mem_.clear();
    opened_ev_.clear();
    for (auto& e : own_ev_)
      if (e) cudaEventDestroy(e), e = nullptr;
    if (own_mail_) cudaFree(own_mail_), own_mail_ = nullptr;
    if (sh_) munmap(sh_, sizeof(LbShared)), sh_ = nullptr;
  }

  int device_;
  int colocated_ = 1;
  std::string name_;
  LbShared* sh_ = nullptr;
  double timeout_ = loopback_timeout_s();
  void* own_mail_ = nullptr;
  cudaEvent_t own_ev_[2] = {nullptr, nullptr};
  std::vector<void*> mail_;
  std::vector<std::array<cudaEvent_t, 2>> ev_;
  std::vector<void*> opened_mem_;
  std::vector<cudaEvent_t> opened_ev_;
};

}  // namespace

// ============================================================================
// Peer memory (both backends): one all-gather of a 128-byte record per rank.
// ============================================================================
namespace {
struct PeerRecord {
  int32_t pid;
  int32_t device;
  uint64_t ptr;
  uint64_t host;  // hash of the host name: IPC only maps buffers of this node
  int32_t ipc_ok;
  int32_t pad;
  cudaIpcMemHandle_t h;  // 64 bytes
  char fill[128 - 32 - sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(PeerRecord) == 128, "peer record is 128 bytes");

uint64_t host_hash() {
  char name[256] = {};
  gethostname(name, sizeof(name) - 1);
  uint64_t x = 1469598103934665603ull;
  for (const char* c = name; *c; ++c) x = (x ^ uint64_t(uint8_t(*c))) * 1099511628211ull;
  return x;
}
}  // namespace

std::vector<void*> Comm::open_peers(void* local, cudaStream_t st) {
  int dev = 0;
  VP_CUDA(cudaGetDevice(&dev));
  PeerRecord mine{};
  mine.pid = int32_t(getpid());
  mine.device = dev;
  mine.ptr = reinterpret_cast<uint64_t>(local);
  mine.host = host_hash();
  mine.ipc_ok = cudaIpcGetMemHandle(&mine.h, local) == cudaSuccess ? 1 : 0;
  (void)cudaGetLastError();
  // a persistent staging buffer: no cudaFree here — it synchronises the whole
  // device, and ranks that already left this exchange may have queued
  // stream-side waits on flags this rank has not written yet
  if (xbuf_ == nullptr) VP_CUDA(cudaMalloc(&xbuf_, sizeof(PeerRecord) * size_t(nranks + 1) + 16));
  void* d = xbuf_;
  std::vector<PeerRecord> all(static_cast<size_t>(nranks));
  std::vector<void*> out(static_cast<size_t>(nranks), nullptr);
  std::vector<void*> opened;
  float fail = 0.f;
  try {
    VP_CUDA(cudaMemcpyAsync(d, &mine, sizeof(mine), cudaMemcpyHostToDevice, st));
    char* recv = static_cast<char*>(d) + sizeof(PeerRecord);
    all_gather(d, recv, sizeof(PeerRecord) / 2, DType::BF16, st);
    VP_CUDA(cudaMemcpyAsync(all.data(), recv, sizeof(PeerRecord) * size_t(nranks), cudaMemcpyDeviceToHost, st));
    VP_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k < nranks && fail == 0.f; ++k) {
      const PeerRecord& o = all[size_t(k)];
      if (k == rank) {
        out[size_t(k)] = local;
      } else if (o.host != mine.host) {
        fail = 1.f;
      } else if (o.pid == mine.pid) {
        if (o.device != dev) {
          int can = 0;
          if (cudaDeviceCanAccessPeer(&can, dev, o.device) != cudaSuccess || !can) {
            fail = 1.f;
            break;
          }
          const cudaError_t e = cudaDeviceEnablePeerAccess(o.device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) fail = 1.f;
        }
        out[size_t(k)] = reinterpret_cast<void*>(o.ptr);
      } else if (!o.ipc_ok) {
        fail = 1.f;
      } else {
        void* p = nullptr;
        if (cudaIpcOpenMemHandle(&p, o.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
          fail = 1.f;
        } else {
          opened.push_back(p);
          out[size_t(k)] = p;
        }
      }
    }
    (void)cudaGetLastError();
    // every rank learns whether all of them mapped all of their peers
    VP_CUDA(cudaMemcpyAsync(d, &fail, sizeof(float), cudaMemcpyHostToDevice, st));
    all_reduce(d, d, 1, DType::F32, RedOp::Max, st);
    VP_CUDA(cudaMemcpyAsync(&fail, d, sizeof(float), cudaMemcpyDeviceToHost, st));
    VP_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    throw;
  }
  if (fail != 0.f) {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    (void)cudaGetLastError();
    return {};
  }
  ipc_opened_.insert(ipc_opened_.end(), opened.begin(), opened.end());
  return out;
}

void Comm::close_peers(const std::vector<void*>& peers) {
  for (void* p : peers) {
    auto it = std::find(ipc_opened_.begin(), ipc_opened_.end(), p);
    if (it == ipc_opened_.end()) continue;
    cudaIpcCloseMemHandle(p);
    ipc_opened_.erase(it);
  }
  (void)cudaGetLastError();
}

double loopback_timeout_s() {
  const char* e = std::getenv("VPIPE_LOOPBACK_TIMEOUT");
  const double v = e ? std::atof(e) : 0.0;
  return v > 0.0 ? v : 300.0;
}

void make_loopback_id(void* id128) {
  char* b = static_cast<char*>(id128);
  std::memset(b, 0, 128);
  std::memcpy(b, kMagic, 8);
  std::random_device rd;
  const unsigned long long r = (static_cast<unsigned long long>(rd()) << 32) ^ rd();
  std::snprintf(b + 8, 64, "/vpipe_lb_%d_%llx", int(getpid()), r);
}

bool is_loopback_id(const void* id128) { return std::memcmp(id128, kMagic, 8) == 0; }

std::unique_ptr<Comm> make_loopback_comm(int nranks, int rank, const void* id128, int device) {
  return std::make_unique<LoopbackComm>(nranks, rank, id128, device);
}

}  // namespace vp
