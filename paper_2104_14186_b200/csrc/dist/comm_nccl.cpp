// NCCL communicator for the distributed driver: one world communicator per rank
// (ncclCommInitRank from a unique id shared by the caller, e.g. over
// torch.distributed), split into the grid's row and column communicators
// (ncclCommSplit).  Every collective is enqueued on the rank's engine stream, so
// it is ordered after the kernels that produced its buffer and before the ones
// that consume it; over NVLink/NVSwitch NCCL picks its own channels (NVLS where
// available).  libnccl is loaded at run time (dlopen), so libqdwhg itself has no
// link-time NCCL dependency and the single-GPU paths never touch it.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "dist.hpp"

namespace qdwhg {
namespace dist {

namespace {

typedef void* nccl_comm;
typedef int nccl_result;
struct nccl_uid {
  char internal[128];
};
constexpr int kNcclFloat64 = 8;

struct NcclApi {
  nccl_result (*GetUniqueId)(nccl_uid*);
  nccl_result (*CommInitRank)(nccl_comm*, int, nccl_uid, int);
  nccl_result (*CommSplit)(nccl_comm, int, int, nccl_comm*, void*);
  nccl_result (*CommDestroy)(nccl_comm);
  nccl_result (*Broadcast)(const void*, void*, size_t, int, int, nccl_comm, void*);
  nccl_result (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm, void*);
  nccl_result (*Send)(const void*, size_t, int, int, nccl_comm, void*);
  nccl_result (*Recv)(void*, size_t, int, int, nccl_comm, void*);
  nccl_result (*GroupStart)();
  nccl_result (*GroupEnd)();
  const char* (*GetErrorString)(nccl_result);
};

const NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = nullptr;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      err = std::string("NCCL not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* s) {
      void* p = dlsym(h, s);
      if (!p) err = std::string("NCCL symbol missing: ") + s;
      return p;
    };
    a.GetUniqueId = (decltype(a.GetUniqueId))sym("ncclGetUniqueId");
    a.CommInitRank = (decltype(a.CommInitRank))sym("ncclCommInitRank");
    a.CommSplit = (decltype(a.CommSplit))sym("ncclCommSplit");
    a.CommDestroy = (decltype(a.CommDestroy))sym("ncclCommDestroy");
    a.Broadcast = (decltype(a.Broadcast))sym("ncclBroadcast");
    a.AllReduce = (decltype(a.AllReduce))sym("ncclAllReduce");
    a.Send = (decltype(a.Send))sym("ncclSend");
    a.Recv = (decltype(a.Recv))sym("ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))sym("ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))sym("ncclGroupEnd");
    a.GetErrorString = (decltype(a.GetErrorString))sym("ncclGetErrorString");
  });
  if (!err.empty()) throw NcclError(err);
  return a;
}

void check(nccl_result r, const char* what) {
  if (r != 0) throw NcclError(std::string(what) + ": " + api().GetErrorString(r));
}

class NcclComm : public Comm {
 public:
  NcclComm(const void* uid, int rank, int world, const Grid& g, void* stream) : rank_(rank), world_(world),
                                                                               stream_(stream) {
    P = g.P;
    Q = g.Q;
    const NcclApi& a = api();
    nccl_uid id;
    std::memcpy(&id, uid, sizeof(id));
    check(a.CommInitRank(&world_c_, world, id, rank), "ncclCommInitRank");
    const int p = rank / Q, q = rank % Q;
    check(a.CommSplit(world_c_, p, q, &row_c_, nullptr), "ncclCommSplit(row)");
    check(a.CommSplit(world_c_, q, p, &col_c_, nullptr), "ncclCommSplit(col)");
  }
  ~NcclComm() override {
    const NcclApi& a = api();
    if (row_c_) a.CommDestroy(row_c_);
    if (col_c_) a.CommDestroy(col_c_);
    if (world_c_) a.CommDestroy(world_c_);
  }
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  void group_begin() override { check(api().GroupStart(), "ncclGroupStart"); }
  void group_end() override { check(api().GroupEnd(), "ncclGroupEnd"); }
  void bcast(double* buf, size_t count, int root, Team team) override {
    if (!count) return;
    int r = root;
    nccl_comm c = world_c_;
    if (team == Team::Row) {
      c = row_c_;
      r = root % Q;
    } else if (team == Team::Col) {
      c = col_c_;
      r = root / Q;
    }
    check(api().Broadcast(buf, buf, count, kNcclFloat64, r, c, stream_), "ncclBroadcast");
  }
  void allreduce(double* buf, size_t count, RedOp op, Team team) override {
    if (!count) return;
    nccl_comm c = team == Team::Row ? row_c_ : team == Team::Col ? col_c_ : world_c_;
    const int o = op == RedOp::Sum ? 0 : op == RedOp::Max ? 2 : 3;
    check(api().AllReduce(buf, buf, count, kNcclFloat64, o, c, stream_), "ncclAllReduce");
  }
  void send(const double* buf, size_t count, int peer) override {
    check(api().Send(buf, count, kNcclFloat64, peer, world_c_, stream_), "ncclSend");
  }
  void recv(double* buf, size_t count, int peer) override {
    check(api().Recv(buf, count, kNcclFloat64, peer, world_c_, stream_), "ncclRecv");
  }

 private:
  int rank_, world_;
  void* stream_;
  nccl_comm world_c_ = nullptr, row_c_ = nullptr, col_c_ = nullptr;
};

}  // namespace

void nccl_unique_id(void* out128) {
  nccl_uid id;
  check(api().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

Comm* nccl_comm_create(const void* uid128, int rank, int world, const Grid& g, void* stream) {
  return new NcclComm(uid128, rank, world, g, stream);
}

}  // namespace dist
}  // namespace qdwhg
