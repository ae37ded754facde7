// In-process loopback communicator: every emulated rank is a host thread of one
// process (its own qdwhg handle / stream, or a host engine in the CPU tests).
// A collective is a rendezvous of the team's threads: each rank first flushes
// its queued work (sync), then buffers are copied with the engine's synchronous
// copy.  No kernel ever waits on another rank, so emulating several ranks on
// one GPU is safe (B200_PROFILING.md: no cross-rank spinning kernels).
// Point-to-point sends are buffered at the send; receives complete at
// group_end (NCCL group semantics: no ordering deadlock inside a group).
#include <condition_variable>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <tuple>

#include "dist.hpp"

namespace qdwhg {
namespace dist {

class LoopbackWorld {
 public:
  explicit LoopbackWorld(int n) : nranks(n) {}
  struct TeamState {
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    std::vector<void*> bufs;
  };
  TeamState& team(int kind, int index, int members) {
    std::lock_guard<std::mutex> lk(mu);
    auto& t = teams[{kind, index}];
    if (!t) {
      t.reset(new TeamState());
      t->bufs.assign(members, nullptr);
    }
    return *t;
  }
  void barrier(TeamState& t, int members) {
    std::unique_lock<std::mutex> lk(t.mu);
    const uint64_t g = t.gen;
    if (++t.arrived == members) {
      t.arrived = 0;
      ++t.gen;
      t.cv.notify_all();
    } else {
      t.cv.wait(lk, [&] { return t.gen != g; });
    }
  }
  // mailbox: (src, dst) -> FIFO of buffered messages
  std::mutex mbox_mu;
  std::condition_variable mbox_cv;
  std::map<std::pair<int, int>, std::vector<std::vector<char>>> mbox;
  int nranks;

 private:
  std::mutex mu;
  std::map<std::pair<int, int>, std::unique_ptr<TeamState>> teams;
};

LoopbackWorld* loopback_world_create(int nranks) { return new LoopbackWorld(nranks); }
void loopback_world_destroy(LoopbackWorld* w) { delete w; }

namespace {

class LoopbackComm : public Comm {
 public:
  LoopbackComm(LoopbackWorld* w, int rank, const Grid& g,
               std::function<void(void*, const void*, size_t)> copy_fn, std::function<void()> sync)
      : w_(w), rank_(rank), copy_(std::move(copy_fn)), sync_(std::move(sync)) {
    P = g.P;
    Q = g.Q;
    p_ = rank / Q;
    q_ = rank % Q;
  }
  int rank() const override { return rank_; }
  int size() const override { return w_->nranks; }
  void group_begin() override { ++depth_; }
  void group_end() override {
    if (--depth_ == 0) flush_recvs();
  }

  void bcast(double* buf, size_t count, int root, Team team) override {
    sync_();
    int members, idx, ridx;
    auto& t = team_of(team, root, &members, &idx, &ridx);
    {
      std::lock_guard<std::mutex> lk(t.mu);
      t.bufs[idx] = buf;
    }
    w_->barrier(t, members);
    if (idx != ridx && count) copy_(buf, t.bufs[ridx], count * sizeof(double));
    w_->barrier(t, members);
  }

  void allreduce(double* buf, size_t count, RedOp op, Team team) override {
    sync_();
    int members, idx, ridx;
    auto& t = team_of(team, rank_, &members, &idx, &ridx);
    {
      std::lock_guard<std::mutex> lk(t.mu);
      t.bufs[idx] = buf;
    }
    w_->barrier(t, members);
    // every member reduces all members' buffers in member order (identical bits)
    std::vector<double> acc(count), tmp(count);
    for (int m = 0; m < members; ++m) {
      copy_(tmp.data(), t.bufs[m], count * sizeof(double));
      for (size_t i = 0; i < count; ++i) {
        if (m == 0) acc[i] = tmp[i];
        else if (op == RedOp::Sum) acc[i] += tmp[i];
        else if (op == RedOp::Max) acc[i] = std::max(acc[i], tmp[i]);
        else acc[i] = std::min(acc[i], tmp[i]);
      }
    }
    w_->barrier(t, members);  // nobody overwrites before all have read
    if (count) copy_(buf, acc.data(), count * sizeof(double));
  }

  void send(const double* buf, size_t count, int peer) override {
    sync_();
    std::vector<char> msg(count * sizeof(double));
    if (count) copy_(msg.data(), buf, msg.size());
    {
      std::lock_guard<std::mutex> lk(w_->mbox_mu);
      w_->mbox[{rank_, peer}].push_back(std::move(msg));
    }
    w_->mbox_cv.notify_all();
  }
  void recv(double* buf, size_t count, int peer) override {
    pending_.push_back({buf, count, peer});
    if (depth_ == 0) flush_recvs();
  }

 private:
  struct Pending {
    double* buf;
    size_t count;
    int peer;
  };
  void flush_recvs() {
    if (pending_.empty()) return;
    sync_();
    for (const Pending& pr : pending_) {
      std::vector<char> msg;
      {
        std::unique_lock<std::mutex> lk(w_->mbox_mu);
        auto key = std::make_pair(pr.peer, rank_);
        w_->mbox_cv.wait(lk, [&] { return !w_->mbox[key].empty(); });
        auto& q = w_->mbox[key];
        msg = std::move(q.front());
        q.erase(q.begin());
      }
      if (msg.size() != pr.count * sizeof(double))
        throw InvalidArgument("loopback recv: message size mismatch");
      if (pr.count) copy_(pr.buf, msg.data(), msg.size());
    }
    pending_.clear();
  }
  LoopbackWorld::TeamState& team_of(Team team, int root, int* members, int* idx, int* ridx) {
    if (team == Team::World) {
      *members = w_->nranks;
      *idx = rank_;
      *ridx = root;
      return w_->team(0, 0, *members);
    }
    if (team == Team::Row) {  // ranks with my p, indexed by q
      *members = Q;
      *idx = q_;
      *ridx = root % Q;
      return w_->team(1, p_, *members);
    }
    *members = P;  // Col: ranks with my q, indexed by p
    *idx = p_;
    *ridx = root / Q;
    return w_->team(2, q_, *members);
  }

  LoopbackWorld* w_;
  int rank_, p_, q_;
  int depth_ = 0;
  std::vector<Pending> pending_;
  std::function<void(void*, const void*, size_t)> copy_;
  std::function<void()> sync_;
};

}  // namespace

Comm* loopback_comm_create(LoopbackWorld* w, int rank, const Grid& g,
                           std::function<void(void*, const void*, size_t)> copy_fn,
                           std::function<void()> sync) {
  return new LoopbackComm(w, rank, g, std::move(copy_fn), std::move(sync));
}

}  // namespace dist
}  // namespace qdwhg
