// Collective backends of a vp_ctx: the exchanges of the vocabulary passes
// (stats all-gather, dX / loss / input all-reduce, naive max / sum
// all-reduce, the executor's C0 broadcast) go through this interface.
//
//   NCCL      production: one rank per GPU, NVLink / NVSwitch.  Created from
//             an ncclUniqueId (one process per GPU) or by ncclCommInitAll
//             (one process driving several GPUs, one host thread per rank).
//   loopback  several ranks that may share ONE GPU (threads of one process,
//             or processes of one node).  Every rank owns a device "mailbox"
//             buffer and two events; a collective copies the rank's input
//             into its mailbox, meets the other ranks at a host barrier, and
//             reduces / gathers straight out of the peers' mailboxes on its
//             own stream (stream-ordered through the peers' events).  It lets
//             the library's nranks > 1 code paths run — and be checked
//             against the oracle — on one B200; NCCL refuses two ranks on one
//             device.  Sums run in rank order, so every rank gets the same
//             bits.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstddef>
#include <cstdint>
#include <memory>
#include <vector>

namespace vp {

enum class DType { F32 = 0, BF16 = 1 };
enum class RedOp { Sum = 0, Max = 1 };

class Comm {
 public:
  virtual ~Comm() { release_peer_staging(); }
  virtual const char* backend() const = 0;
  // recv[k * count + i] = send_k[i]  (rank order)
  virtual void all_gather(const void* send, void* recv, size_t count, DType dt, cudaStream_t st) = 0;
  // recv = op_k send_k (in place allowed)
  virtual void all_reduce(const void* send, void* recv, size_t count, DType dt, RedOp op, cudaStream_t st) = 0;
  // recv = send of `root` (in place allowed)
  virtual void broadcast(const void* send, void* recv, size_t count, DType dt, int root, cudaStream_t st) = 0;
  virtual void group_start() {}
  virtual void group_end() {}
  // NCCL calls can be captured into a CUDA graph; the loopback's host
  // rendezvous cannot.
  virtual bool capturable() const { return true; }
  // ranks of this group on this rank's physical GPU (itself included): they
  // share its SMs, so the persistent GEMMs of each get a 1/colocated share
  virtual int colocated() const { return 1; }

  // Peer memory for the fused exchanges (the dX GEMM that stores its tiles
  // straight into the owning rank's buffer over NVLink).  Collective and
  // host-blocking: every rank passes one device buffer it allocated with
  // cudaMalloc (base pointer); returns every rank's buffer as addressable
  // from this rank (own pointer, a peer-enabled pointer of a GPU this process
  // drives, or a CUDA IPC mapping of another process's buffer).  Returns an
  // empty vector on every rank when any rank cannot map some peer (other
  // node, no P2P path): the caller then keeps the collective path.
  std::vector<void*> open_peers(void* local, cudaStream_t st);
  // Unmaps what open_peers mapped (IPC mappings; no-op for the rest).
  void close_peers(const std::vector<void*>& peers);
  int nranks = 1, rank = 0;

 protected:
  void release_peer_staging() {
    if (xbuf_) cudaFree(xbuf_), xbuf_ = nullptr;
  }

 private:
  std::vector<void*> ipc_opened_;
  void* xbuf_ = nullptr;  // open_peers' staging buffer (kept: see open_peers)
};

// NCCL from a 128-byte ncclUniqueId; max_ctas bounds NCCL's SM use.
std::unique_ptr<Comm> make_nccl_comm(int nranks, int rank, const void* id128, int max_ctas);
// Wraps a communicator made elsewhere (ncclCommInitAll); takes ownership.
std::unique_ptr<Comm> wrap_nccl_comm(ncclComm_t comm, int nranks, int rank);

// Loopback ids carry a magic prefix so vp_ctx_comm_init can dispatch on them.
void make_loopback_id(void* id128);
bool is_loopback_id(const void* id128);
// Joins the loopback group named by id128 (blocks until all nranks joined).
// `device` is the caller's current CUDA device.
std::unique_ptr<Comm> make_loopback_comm(int nranks, int rank, const void* id128, int device);

// Seconds a loopback rank waits at a rendezvous before failing (a peer died
// or issued a different collective sequence).  Default 300; env
// VPIPE_LOOPBACK_TIMEOUT overrides.
double loopback_timeout_s();

}  // namespace vp
