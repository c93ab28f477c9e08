// comm.h -- tensor-parallel exchange for the co-serving step.
//
// Megatron-style TP ("dependent parallelization", north_star): QKV and gate||up are
// column-parallel (heads / ffn columns), O and down are row-parallel; the residual stream
// is replicated and the row-parallel partial sums are all-reduced in place:
//   forward : 2 all-reduces [T, h] per layer (after O, after down [+ the LoRA up, folded])
//   backward: 2 all-reduces [s, h] per window and layer (dX of gate||up and of QKV)
//   Adam    : 1 all-reduce of dB [layers, r, h] per mini-batch (the folded LoRA layout)
// Three backends behind one interface:
//   * NCCL (one process per GPU, ncclCommInitRank from a unique id shared by the host),
//   * local group (ranks are engines of one process, each driven by its own host thread):
//     a one-shot peer all-reduce kernel -- every rank reduces its 1/tp slice of all ranks'
//     buffers in a fixed order and writes the sum back into every buffer -- ordered by
//     CUDA events exchanged at two host barriers.  Over NVSwitch the peer pointers are
//     NVLink loads/stores (peer access enabled); on one device the same code runs with
//     plain device pointers, which is how the TP math is tested on a single B200;
//   * IPC group (one process per GPU, no NCCL): every rank maps the other ranks' engine arenas
//     with CUDA IPC handles the host exchanges (cs_engine_ipc_handle / cs_engine_ipc_attach);
//     cross-rank ordering is a device-side flag barrier (system-scope release stores into each
//     peer's flag slots, acquire spins on the local ones), so the fused row-parallel GEMM +
//     all-reduce and the one-shot peer all-reduce run across processes over NVLink exactly as
//     in a single-process group.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include <string>

namespace cs {

struct Comm {
  virtual ~Comm() {}
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // in-place sum over the ranks of buf[0, n), stream-ordered on st; 0 on success
  virtual int allreduce_f32(float* buf, size_t n, cudaStream_t st, std::string* err) = 0;
  // Peer-memory groups (every rank's device buffers are addressable from every rank: the
  // ranks of one process over NVLink / NVSwitch peer access) run the fused row-parallel GEMM
  // + all-reduce (engine.cu tp_rowpar): false for NCCL.
  virtual bool peer_capable() const { return false; }
  // every rank passes its local device pointer; out[r] = rank r's (host barrier); 0 on success
  virtual int exchange_ptr(void* local, void** out, std::string* err) {
    if (err) *err = "exchange_ptr: not a peer-memory group";
    return -1;
  }
  // cross-rank stream ordering point: work enqueued on every rank's stream before the call
  // completes before work any rank enqueues after it; 0 on success
  virtual int stream_barrier(cudaStream_t st, std::string* err) {
    if (err) *err = "stream_barrier: not a peer-memory group";
    return -1;
  }
  // the engine's device arena (IPC groups map the peers' arenas; flags: 8 zeroed uint32 in it)
  virtual void bind_arena(void* base, size_t bytes, unsigned* flags) {}
  // IPC groups: export this rank's arena handle / map the other ranks' (handles[tp][64])
  virtual int ipc_handle(void* out64, std::string* err) {
    if (err) *err = "ipc_handle: not an IPC group";
    return -1;
  }
  virtual int ipc_attach(const void* handles, const int64_t* arena_bytes, std::string* err) {
    if (err) *err = "ipc_attach: not an IPC group";
    return -1;
  }
};

// Second half of the fused row-parallel GEMM + all-reduce: rank `rank` owns rows
// [rank * rpo, min(M, (rank + 1) * rpo)); it sums the ranks' partial slots of its local
// staging buffer [nranks][rpo][ld] in rank order (+ the replicated old value of the
// destination when add_old), zeroes the slots (the GEMM's split-K atomics rely on zeroed
// slots), and stores the sum into every rank's destination (peer stores): bit-identical on
// every rank.
cudaError_t tp_reduce_bcast(float* stage, long ld, int nranks, int rank, int rpo, int M, int h,
                            float* const* dst, long ldd, int add_old, cudaStream_t st);

// NCCL communicator from a 128-byte ncclUniqueId (all ranks call concurrently)
Comm* make_nccl_comm(const void* unique_id, int rank, int size, std::string* err);
int nccl_unique_id(void* out128, std::string* err);

struct LocalGroup;
LocalGroup* local_group_create(int size, std::string* err);
void local_group_destroy(LocalGroup* g);
int local_group_size(const LocalGroup* g);
Comm* make_local_comm(LocalGroup* g, int rank, int device, std::string* err);
Comm* make_ipc_comm(int rank, int size, int device, std::string* err);

}  // namespace cs
