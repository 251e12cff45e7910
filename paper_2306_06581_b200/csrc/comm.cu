// comm.cu -- the collectives of the sharded solve, owned by the
// library so a C / C++ caller reaches the multi-GPU path through the C ABI
// (include/spk.h spk_comm_*, spk_sharded_*):
//
// * NcclComm     -- NCCL over NVLink / NVSwitch. libnccl is loaded at run
//                   time (dlopen; the copy torch already loaded when there is
//                   one, else SPK_NCCL_LIB, else libnccl.so.2), so the library
//                   has no link-time NCCL dependency. Collectives are stream-
//                   ordered on the context stream and CUDA-graph capturable.
// * EmulatedComm -- W ranks as host threads of one process sharing one GPU:
//                   every collective synchronises the caller's stream, meets
//                   the other threads at a host barrier and copies through
//                   host memory. No kernel ever waits on another rank's kernel
//                   (tests only: it cannot be graph-captured).
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"
#include "internal.h"

namespace spk {

namespace {

// ---- NCCL, loaded at run time ---------------------------------------------------
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (e.g. torch's)
    if (!h && std::getenv("SPK_NCCL_LIB")) h = dlopen(std::getenv("SPK_NCCL_LIB"), RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    bool all = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) all = false;
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommInitAll, "ncclCommInitAll");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.AllGather, "ncclAllGather");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    api.ok = all;
    if (!all) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Failure(SPK_STATUS_DEVICE, SPK_E_DEVICE,
                  std::string("NCCL error in ") + what + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

NcclApi& nccl_required() {
  NcclApi& a = nccl();
  if (!a.ok) throw Failure(SPK_STATUS_DEVICE, SPK_E_DEVICE, "NCCL unavailable: " + a.why);
  return a;
}

ncclDataType_t nccl_type(CommType t) {
  switch (t) {
    case CommType::F64: return ncclFloat64;
    case CommType::I64: return ncclInt64;
    default: return ncclUint8;
  }
}

struct NcclComm final : Comm {
  ncclComm_t comm = nullptr;
  bool owns = true;
  ~NcclComm() override {
    if (comm && owns) nccl().CommDestroy(comm);
  }
  void all_gather(void* buf, size_t chunk_bytes, cudaStream_t s) override {
    char* b = static_cast<char*>(buf);
    // in place: this rank's block is the send buffer
    nccl_check(nccl().AllGather(b + (size_t)rank * chunk_bytes, b, chunk_bytes, ncclUint8, comm, s), "all_gather");
  }
  void all_to_all_v(const void* send, const int64_t* send_bytes, void* recv, const int64_t* recv_bytes,
                    cudaStream_t s) override {
    NcclApi& a = nccl();
    nccl_check(a.GroupStart(), "group_start");
    int64_t so = 0, ro = 0;
    for (int p = 0; p < world; ++p) {
      if (send_bytes[p])
        nccl_check(a.Send(static_cast<const char*>(send) + so, (size_t)send_bytes[p], ncclUint8, p, comm, s), "send");
      if (recv_bytes[p])
        nccl_check(a.Recv(static_cast<char*>(recv) + ro, (size_t)recv_bytes[p], ncclUint8, p, comm, s), "recv");
      so += send_bytes[p];
      ro += recv_bytes[p];
    }
    nccl_check(a.GroupEnd(), "group_end");
  }
  void all_reduce_sum(void* buf, size_t count, CommType t, cudaStream_t s) override {
    nccl_check(nccl().AllReduce(buf, buf, count, nccl_type(t), ncclSum, comm, s), "all_reduce");
  }
  bool capturable() const override { return true; }
};

// ---- emulated ranks (threads of one process, one GPU) ---------------------------
struct HostGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  bool broken = false;
  std::vector<std::vector<char>> slot;   // per rank payload
  std::vector<std::vector<int64_t>> sizes;  // per rank: send sizes of an all-to-all
  explicit HostGroup(int w) : world(w), slot(w), sizes(w) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (broken) throw Failure(SPK_STATUS_DEVICE, SPK_E_DEVICE, "emulated communicator: a rank failed");
    const long long g = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return generation != g || broken; });
    if (broken) throw Failure(SPK_STATUS_DEVICE, SPK_E_DEVICE, "emulated communicator: a rank failed");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

struct EmulatedComm final : Comm {
  std::shared_ptr<HostGroup> g;
  ~EmulatedComm() override = default;
  void sync(cudaStream_t s) { SPK_CUDA(cudaStreamSynchronize(s)); }
  template <class F>
  void guarded(F&& f) {
    try {
      f();
    } catch (...) {
      g->abort();
      throw;
    }
  }
  void all_gather(void* buf, size_t chunk_bytes, cudaStream_t s) override {
    guarded([&] {
      sync(s);
      char* b = static_cast<char*>(buf);
      g->slot[rank].resize(chunk_bytes);
      SPK_CUDA(cudaMemcpy(g->slot[rank].data(), b + (size_t)rank * chunk_bytes, chunk_bytes, cudaMemcpyDeviceToHost));
      g->barrier();
      for (int r = 0; r < world; ++r)
        if (r != rank)
          SPK_CUDA(cudaMemcpy(b + (size_t)r * chunk_bytes, g->slot[r].data(), chunk_bytes, cudaMemcpyHostToDevice));
      g->barrier();
    });
  }
  void all_to_all_v(const void* send, const int64_t* send_bytes, void* recv, const int64_t* recv_bytes,
                    cudaStream_t s) override {
    guarded([&] {
      sync(s);
      int64_t tot = 0;
      for (int p = 0; p < world; ++p) tot += send_bytes[p];
      g->slot[rank].resize((size_t)tot);
      g->sizes[rank].assign(send_bytes, send_bytes + world);
      if (tot) SPK_CUDA(cudaMemcpy(g->slot[rank].data(), send, (size_t)tot, cudaMemcpyDeviceToHost));
      g->barrier();
      int64_t ro = 0;
      for (int src = 0; src < world; ++src) {
        int64_t off = 0;
        for (int p = 0; p < rank; ++p) off += g->sizes[src][p];
        const int64_t nb = g->sizes[src][rank];
        if (nb != recv_bytes[src]) throw Failure(SPK_STATUS_INPUT, SPK_E_LENGTH_MISMATCH, "all_to_all size mismatch");
        if (nb)
          SPK_CUDA(cudaMemcpy(static_cast<char*>(recv) + ro, g->slot[src].data() + off, (size_t)nb,
                              cudaMemcpyHostToDevice));
        ro += nb;
      }
      g->barrier();
    });
  }
  void all_reduce_sum(void* buf, size_t count, CommType t, cudaStream_t s) override {
    guarded([&] {
      sync(s);
      const size_t eb = 8;  // F64 / I64
      g->slot[rank].resize(count * eb);
      SPK_CUDA(cudaMemcpy(g->slot[rank].data(), buf, count * eb, cudaMemcpyDeviceToHost));
      g->barrier();
      std::vector<char> out(count * eb);
      for (size_t k = 0; k < count; ++k) {
        if (t == CommType::F64) {
          double acc = 0.0;  // rank order
          for (int r = 0; r < world; ++r) acc += reinterpret_cast<const double*>(g->slot[r].data())[k];
          reinterpret_cast<double*>(out.data())[k] = acc;
        } else {
          int64_t acc = 0;
          for (int r = 0; r < world; ++r) acc += reinterpret_cast<const int64_t*>(g->slot[r].data())[k];
          reinterpret_cast<int64_t*>(out.data())[k] = acc;
        }
      }
      g->barrier();
      SPK_CUDA(cudaMemcpy(buf, out.data(), count * eb, cudaMemcpyHostToDevice));
    });
  }
  bool capturable() const override { return false; }
};

}  // namespace

}  // namespace spk

struct spk_comm_group {
  std::shared_ptr<spk::HostGroup> g;
};

using namespace spk;

extern "C" {

int spk_comm_unique_id(unsigned char id[128]) {
  if (!id) return SPK_STATUS_INPUT;
  return guard(nullptr, [&] {
    ncclUniqueId u;
    nccl_check(nccl_required().GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == 128, "ncclUniqueId size");
    std::memcpy(id, u.internal, 128);
  });
}

int spk_comm_init(spk_ctx* ctx, const unsigned char id[128], int world, int rank, spk_comm** out) {
  if (!ctx || !id || !out || world < 1 || rank < 0 || rank >= world) return SPK_STATUS_INPUT;
  *out = nullptr;
  return guard(ctx, [&] {
    auto c = std::make_unique<NcclComm>();
    c->world = world;
    c->rank = rank;
    c->ctx = ctx;
    ncclUniqueId u;
    std::memcpy(u.internal, id, 128);
    nccl_check(nccl_required().CommInitRank(&c->comm, world, u, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

int spk_comm_init_all(const int* devices, int ndev, spk_ctx** ctxs, spk_comm** comms) {
  if (!devices || ndev < 1 || !ctxs || !comms) return SPK_STATUS_INPUT;
  for (int r = 0; r < ndev; ++r) {
    if (!ctxs[r] || ctxs[r]->device != devices[r]) return SPK_STATUS_INPUT;
    comms[r] = nullptr;
  }
  return guard(ctxs[0], [&] {
    std::vector<ncclComm_t> nc(ndev, nullptr);
    nccl_check(nccl_required().CommInitAll(nc.data(), ndev, devices), "ncclCommInitAll");
    for (int r = 0; r < ndev; ++r) {
      auto c = std::make_unique<NcclComm>();
      c->world = ndev;
      c->rank = r;
      c->ctx = ctxs[r];
      c->comm = nc[r];
      comms[r] = c.release();
    }
  });
}

int spk_comm_group_create(int world, spk_comm_group** out) {
  if (world < 1 || !out) return SPK_STATUS_INPUT;
  *out = new spk_comm_group{std::make_shared<HostGroup>(world)};
  return SPK_OK;
}

void spk_comm_group_destroy(spk_comm_group* g) { delete g; }

int spk_comm_init_emulated(spk_ctx* ctx, spk_comm_group* group, int rank, spk_comm** out) {
  if (!ctx || !group || !out || rank < 0 || rank >= group->g->world) return SPK_STATUS_INPUT;
  auto c = std::make_unique<EmulatedComm>();
  c->world = group->g->world;
  c->rank = rank;
  c->ctx = ctx;
  c->g = group->g;
  *out = c.release();
  return SPK_OK;
}

void spk_comm_destroy(spk_comm* comm) { delete comm; }

int spk_comm_info(const spk_comm* comm, int* world, int* rank, int* nccl_backed) {
  if (!comm) return SPK_STATUS_INPUT;
  if (world) *world = comm->world;
  if (rank) *rank = comm->rank;
  if (nccl_backed) *nccl_backed = comm->capturable() ? 1 : 0;
  return SPK_OK;
}

}  // extern "C"
