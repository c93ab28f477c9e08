// comm.cu -- TP all-reduce backends (see comm.h): NCCL, and the local-group one-shot peer
// all-reduce (reduce-scatter + all-gather in one kernel over peer pointers).
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "comm.h"
#include "common.cuh"
#include "kernels.h"

namespace cs {

// ================================================================================ NCCL
namespace {
struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  int r = 0, n = 1;
  ~NcclComm() override {
    if (comm) ncclCommDestroy(comm);
  }
  int rank() const override { return r; }
  int size() const override { return n; }
  int allreduce_f32(float* buf, size_t count, cudaStream_t st, std::string* err) override {
    ncclResult_t res = ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, comm, st);
    if (res != ncclSuccess) {
      if (err) *err = std::string("ncclAllReduce: ") + ncclGetErrorString(res);
      return -1;
    }
    return 0;
  }
};
}  // namespace

int nccl_unique_id(void* out128, std::string* err) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  ncclResult_t res = ncclGetUniqueId(&id);
  if (res != ncclSuccess) {
    if (err) *err = std::string("ncclGetUniqueId: ") + ncclGetErrorString(res);
    return -1;
  }
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

Comm* make_nccl_comm(const void* unique_id, int rank, int size, std::string* err) {
  auto* c = new NcclComm();
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclResult_t res = ncclCommInitRank(&c->comm, size, id, rank);
  if (res != ncclSuccess) {
    if (err) *err = std::string("ncclCommInitRank: ") + ncclGetErrorString(res);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  c->r = rank;
  c->n = size;
  return c;
}

// ========================================================================= local group
constexpr int kMaxRanks = 8;

struct PeerPtrs {
  float* p[kMaxRanks];
};

// rank `me` owns float4 slots [lo, hi) of n4: sum over ranks in rank order (bit-identical on
// every rank), store the sum into every rank's buffer.  Rank 0 also handles the n % 4 tail.
__global__ void __launch_bounds__(256) peer_allreduce_kernel(PeerPtrs ptrs, int nranks, int me,
                                                             size_t n) {
  const size_t n4 = n / 4;
  const size_t per = (n4 + nranks - 1) / nranks;
  const size_t lo = (size_t)me * per, hi = lo + per < n4 ? lo + per : n4;
  for (size_t i = lo + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hi;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 s = reinterpret_cast<const float4*>(ptrs.p[0])[i];
    for (int j = 1; j < nranks; ++j) {
      const float4 v = reinterpret_cast<const float4*>(ptrs.p[j])[i];
      s.x += v.x;
      s.y += v.y;
      s.z += v.z;
      s.w += v.w;
    }
    for (int j = 0; j < nranks; ++j) reinterpret_cast<float4*>(ptrs.p[j])[i] = s;
  }
  if (me == 0 && blockIdx.x == 0 && threadIdx.x < (int)(n % 4)) {
    const size_t i = n4 * 4 + threadIdx.x;
    float s = ptrs.p[0][i];
    for (int j = 1; j < nranks; ++j) s += ptrs.p[j][i];
    for (int j = 0; j < nranks; ++j) ptrs.p[j][i] = s;
  }
}

struct LocalGroup {
  int n = 0;
  // sense-reversing spin barrier (the ranks are host threads of this process)
  std::atomic<int> arrived{0};
  std::atomic<int> gen{0};
  std::atomic<int> attached{0};
  std::atomic<bool> broken{false};
  float* ptrs[kMaxRanks] = {};
  void* xptrs[kMaxRanks] = {};                // exchange_ptr
  cudaEvent_t ev_sb[2][kMaxRanks] = {};       // stream_barrier (alternating sets)
  cudaEvent_t ev_ready[kMaxRanks] = {};
  cudaEvent_t ev_done[kMaxRanks] = {};
  int device[kMaxRanks] = {};

  // false on timeout (a rank died or took a different path): the group is then broken
  bool barrier() {
    if (broken.load(std::memory_order_acquire)) return false;
    const int g = gen.load(std::memory_order_acquire);
    if (arrived.fetch_add(1, std::memory_order_acq_rel) == n - 1) {
      arrived.store(0, std::memory_order_relaxed);
      gen.fetch_add(1, std::memory_order_acq_rel);
      return true;
    }
    const auto t0 = std::chrono::steady_clock::now();
    long spins = 0;
    while (gen.load(std::memory_order_acquire) == g) {
      if (++spins > 64) std::this_thread::yield();
      if ((spins & 1023) == 0 &&
          std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
        broken.store(true, std::memory_order_release);
        return false;
      }
      if (broken.load(std::memory_order_acquire)) return false;
    }
    return true;
  }
};

namespace {
struct LocalComm final : Comm {
  LocalGroup* g = nullptr;
  int r = 0;
  int sb_parity = 0;
  bool peer_capable() const override { return true; }
  int exchange_ptr(void* local, void** out, std::string* err) override {
    g->xptrs[r] = local;
    if (!g->barrier()) {
      if (err) *err = "tp barrier timeout (ranks diverged)";
      return -1;
    }
    for (int j = 0; j < g->n; ++j) out[j] = g->xptrs[j];
    if (!g->barrier()) {  // nobody overwrites xptrs before every rank has read them
      if (err) *err = "tp barrier timeout (ranks diverged)";
      return -1;
    }
    return 0;
  }
  // one host barrier per call; the event set alternates, so a rank re-records set p only
  // after the barrier of set 1-p, which every rank reaches after its waits on set p
  int stream_barrier(cudaStream_t st, std::string* err) override {
    const int p = sb_parity;
    sb_parity ^= 1;
    cudaEventRecord(g->ev_sb[p][r], st);
    if (!g->barrier()) {
      if (err) *err = "tp barrier timeout (ranks diverged)";
      return -1;
    }
    for (int j = 0; j < g->n; ++j)
      if (j != r) cudaStreamWaitEvent(st, g->ev_sb[p][j], 0);
    return 0;
  }
  int rank() const override { return r; }
  int size() const override { return g->n; }
  int allreduce_f32(float* buf, size_t count, cudaStream_t st, std::string* err) override {
    const int n = g->n;
    if (count == 0) return 0;
    if ((reinterpret_cast<uintptr_t>(buf) & 15) != 0) {
      if (err) *err = "local all-reduce: buffer not 16-byte aligned";
      return -1;
    }
    g->ptrs[r] = buf;
    cudaEventRecord(g->ev_ready[r], st);
    if (!g->barrier()) {
      if (err) *err = "tp barrier timeout (ranks diverged)";
      return -1;
    }
    for (int j = 0; j < n; ++j)
      if (j != r) cudaStreamWaitEvent(st, g->ev_ready[j], 0);
    PeerPtrs pp{};
    for (int j = 0; j < n; ++j) pp.p[j] = g->ptrs[j];
    const size_t per4 = (count / 4 + n - 1) / n;
    const int blocks = (int)std::max<size_t>(1, std::min<size_t>((per4 + 255) / 256, 148 * 4));
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    peer_allreduce_kernel<<<blocks, 256, 0, st>>>(pp, n, r, count);
    cudaError_t e = cudaGetLastError();
    cudaEventRecord(g->ev_done[r], st);
    // all slices written before anyone reads its buffer again; ptrs[] may be reused after
    if (!g->barrier()) {
      if (err) *err = "tp barrier timeout (ranks diverged)";
      return -1;
    }
    for (int j = 0; j < n; ++j)
      if (j != r) cudaStreamWaitEvent(st, g->ev_done[j], 0);
    if (e != cudaSuccess) {
      if (err) *err = std::string("peer_allreduce_kernel: ") + cudaGetErrorString(e);
      return -1;
    }
    return 0;
  }
};
}  // namespace

__global__ void __launch_bounds__(256) tp_reduce_bcast_kernel(float* __restrict__ stage, long ld,
                                                              int nranks, int rank, int rpo, int M,
                                                              int h, PeerPtrs dst, long ldd,
                                                              int add_old) {
  const int row0 = rank * rpo;
  const int nrows = min(rpo, M - row0);
  const int h4 = h / 4;
  const long total = (long)max(nrows, 0) * h4;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
    const int lr = (int)(i / h4), c = (int)(i % h4) * 4;
    const long drow = (long)(row0 + lr) * ldd + c;
    float4 v = add_old ? *reinterpret_cast<const float4*>(dst.p[rank] + drow) : make_float4(0.f, 0.f, 0.f, 0.f);
    for (int s = 0; s < nranks; ++s) {
      float4* sp = reinterpret_cast<float4*>(stage + ((long)s * rpo + lr) * ld + c);
      const float4 t = *sp;
      v.x += t.x;
      v.y += t.y;
      v.z += t.z;
      v.w += t.w;
      *sp = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int j = 0; j < nranks; ++j) *reinterpret_cast<float4*>(dst.p[j] + drow) = v;
  }
}

cudaError_t tp_reduce_bcast(float* stage, long ld, int nranks, int rank, int rpo, int M, int h,
                            float* const* dst, long ldd, int add_old, cudaStream_t st) {
  if (nranks < 1 || nranks > kMaxRanks || (h % 4) != 0 || rpo < 1) return cudaErrorInvalidValue;
  PeerPtrs pp{};
  for (int j = 0; j < nranks; ++j) pp.p[j] = dst[j];
  const long work = (long)std::max(0, std::min(rpo, M - rank * rpo)) * (h / 4);
  if (work <= 0) return cudaSuccess;
  const int blocks = (int)std::max<long>(1, std::min<long>((work + 255) / 256, 148 * 8));
  cs::g_launches.fetch_add(1, std::memory_order_relaxed);
  tp_reduce_bcast_kernel<<<blocks, 256, 0, st>>>(stage, ld, nranks, rank, rpo, M, h, pp, ldd, add_old);
  return cudaGetLastError();
}

// ============================================================================ IPC group
// Device-side barrier across processes: thread j stores `epoch` into slot `rank` of rank j's
// flag array (system-scope release: every earlier write of this rank -- the previous kernels on
// this stream included -- is visible to rank j before the flag), then spins (acquire) until
// rank j's store of the same epoch reached slot j of the local array.  20 s bound -> trap.
struct IpcFlags {
  unsigned* peer[kMaxRanks];  // peer[j] = rank j's flag array (mapped)
  unsigned* local;
};
__global__ void ipc_barrier_kernel(IpcFlags f, int rank, int nranks, unsigned epoch) {
  const int j = threadIdx.x;
  if (j >= nranks) return;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.peer[j] + rank), "r"(epoch) : "memory");
  const unsigned long long t0 = globaltimer_ns();
  while (true) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f.local + j) : "memory");
    if ((int)(v - epoch) >= 0) break;
    if (globaltimer_ns() - t0 > 20000000000ull) __trap();
  }
}

namespace {
struct IpcComm final : Comm {
  int r = 0, n = 1, device = 0;
  char* base = nullptr;
  size_t bytes = 0;
  unsigned* flags = nullptr;
  char* peer_base[kMaxRanks] = {};
  bool opened[kMaxRanks] = {};
  bool attached = false;
  unsigned epoch = 0;
  ~IpcComm() override {
    for (int j = 0; j < n; ++j)
      if (opened[j]) cudaIpcCloseMemHandle(peer_base[j]);
  }
  int rank() const override { return r; }
  int size() const override { return n; }
  bool peer_capable() const override { return attached; }
  void bind_arena(void* b, size_t nbytes, unsigned* f) override {
    base = static_cast<char*>(b);
    bytes = nbytes;
    flags = f;
  }
  int ipc_handle(void* out64, std::string* err) override {
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, base);
    if (e != cudaSuccess) {
      if (err) *err = std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
      return -1;
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(out64, &h, 64);
    return 0;
  }
  int ipc_attach(const void* handles, const int64_t* arena_bytes, std::string* err) override {
    if (attached) return 0;
    for (int j = 0; j < n; ++j) {
      if (arena_bytes[j] != (int64_t)bytes) {
        if (err) *err = "ipc_attach: ranks' engine arenas differ (different configs?)";
        return -1;
      }
      if (j == r) {
        peer_base[j] = base;
        continue;
      }
      cudaIpcMemHandle_t h;
      std::memcpy(&h, static_cast<const char*>(handles) + 64 * j, 64);
      void* p = nullptr;
      const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        if (err) *err = "cudaIpcOpenMemHandle(rank " + std::to_string(j) + "): " + cudaGetErrorString(e);
        return -1;
      }
      peer_base[j] = static_cast<char*>(p);
      opened[j] = true;
    }
    attached = true;
    return 0;
  }
  int exchange_ptr(void* local, void** out, std::string* err) override {
    // every rank's arena has the same layout: a buffer's peer address is the peer's arena
    // base plus the local offset
    const char* p = static_cast<const char*>(local);
    if (!attached || p < base || p >= base + bytes) {
      if (err) *err = attached ? "ipc exchange_ptr: pointer outside the engine arena" : "ipc group not attached";
      return -1;
    }
    for (int j = 0; j < n; ++j) out[j] = peer_base[j] + (p - base);
    return 0;
  }
  int stream_barrier(cudaStream_t st, std::string* err) override {
    if (!attached) {
      if (err) *err = "ipc group not attached (cs_engine_ipc_attach)";
      return -1;
    }
    IpcFlags f{};
    const size_t off = reinterpret_cast<char*>(flags) - base;
    for (int j = 0; j < n; ++j) f.peer[j] = reinterpret_cast<unsigned*>(peer_base[j] + off);
    f.local = flags;
    ++epoch;
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    ipc_barrier_kernel<<<1, 32, 0, st>>>(f, r, n, epoch);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (err) *err = std::string("ipc_barrier_kernel: ") + cudaGetErrorString(e);
      return -1;
    }
    return 0;
  }
  int allreduce_f32(float* buf, size_t count, cudaStream_t st, std::string* err) override {
    if (count == 0) return 0;
    void* out[kMaxRanks] = {};
    if (exchange_ptr(buf, out, err) != 0) return -1;
    if ((reinterpret_cast<uintptr_t>(buf) & 15) != 0) {
      if (err) *err = "ipc all-reduce: buffer not 16-byte aligned";
      return -1;
    }
    if (stream_barrier(st, err) != 0) return -1;  // every rank's buffer is final
    PeerPtrs pp{};
    for (int j = 0; j < n; ++j) pp.p[j] = static_cast<float*>(out[j]);
    const size_t per4 = (count / 4 + n - 1) / n;
    const int blocks = (int)std::max<size_t>(1, std::min<size_t>((per4 + 255) / 256, 148 * 4));
    cs::g_launches.fetch_add(1, std::memory_order_relaxed);
    peer_allreduce_kernel<<<blocks, 256, 0, st>>>(pp, n, r, count);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      if (err) *err = std::string("peer_allreduce_kernel: ") + cudaGetErrorString(e);
      return -1;
    }
    return stream_barrier(st, err);  // every slice written before anyone reads its buffer
  }
};
}  // namespace

Comm* make_ipc_comm(int rank, int size, int device, std::string* err) {
  if (size < 1 || size > kMaxRanks || rank < 0 || rank >= size) {
    if (err) *err = "ipc tp comm: need 0 <= rank < size <= 8";
    return nullptr;
  }
  auto* c = new IpcComm();
  c->r = rank;
  c->n = size;
  c->device = device;
  return c;
}

LocalGroup* local_group_create(int size, std::string* err) {
  if (size < 1 || size > kMaxRanks) {
    if (err) *err = "tp group size must be in [1, 8]";
    return nullptr;
  }
  auto* g = new LocalGroup();
  g->n = size;
  for (int i = 0; i < size; ++i) g->device[i] = -1;
  return g;
}

int local_group_size(const LocalGroup* g) { return g ? g->n : 0; }

void local_group_destroy(LocalGroup* g) {
  if (!g) return;
  for (int i = 0; i < g->n; ++i) {
    if (g->ev_ready[i]) cudaEventDestroy(g->ev_ready[i]);
    if (g->ev_done[i]) cudaEventDestroy(g->ev_done[i]);
    for (int p = 0; p < 2; ++p)
      if (g->ev_sb[p][i]) cudaEventDestroy(g->ev_sb[p][i]);
  }
  delete g;
}

Comm* make_local_comm(LocalGroup* g, int rank, int device, std::string* err) {
  if (!g || rank < 0 || rank >= g->n) {
    if (err) *err = "local tp comm: bad group / rank";
    return nullptr;
  }
  if (g->device[rank] != -1) {
    if (err) *err = "local tp comm: rank already attached";
    return nullptr;
  }
  // events live on the rank's device; peers may sit on other devices of this process
  cudaEventCreateWithFlags(&g->ev_ready[rank], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&g->ev_done[rank], cudaEventDisableTiming);
  for (int p = 0; p < 2; ++p) cudaEventCreateWithFlags(&g->ev_sb[p][rank], cudaEventDisableTiming);
  g->device[rank] = device;
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  for (int j = 0; j < ndev; ++j) {
    if (j == device) continue;
    int ok = 0;
    cudaDeviceCanAccessPeer(&ok, device, j);
    if (ok) {
      cudaError_t e = cudaDeviceEnablePeerAccess(j, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    }
  }
  g->attached.fetch_add(1);
  auto* c = new LocalComm();
  c->g = g;
  c->r = rank;
  return c;
}

}  // namespace cs
