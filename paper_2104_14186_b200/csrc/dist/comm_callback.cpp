// Communicator over caller-supplied callbacks (qdwhg_comm_callbacks): lets a
// host application plug its own transport (MPI, torch.distributed, ...) under
// the distributed driver.  Buffers passed to the callbacks are the engine's
// (device memory in libqdwhg) and the rank's stream has been synchronized
// before each call, so a blocking transport sees final data.  Team ids:
// 0 world, 1 grid row, 2 grid column; roots are world ranks.
#include "dist.hpp"

namespace qdwhg {
namespace dist {

namespace {
class CallbackComm : public Comm {
 public:
  CallbackComm(const CommCallbacks& cb, int rank, int world, const Grid& g, std::function<void()> sync)
      : cb_(cb), rank_(rank), world_(world), sync_(std::move(sync)) {
    P = g.P;
    Q = g.Q;
  }
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  void group_begin() override { check(cb_.group_begin ? cb_.group_begin(cb_.ctx) : 0, "group_begin"); }
  void group_end() override { check(cb_.group_end ? cb_.group_end(cb_.ctx) : 0, "group_end"); }
  void bcast(double* buf, size_t count, int root, Team team) override {
    sync_();
    check(cb_.bcast(cb_.ctx, buf, count, root, (int)team), "bcast");
  }
  void allreduce(double* buf, size_t count, RedOp op, Team team) override {
    sync_();
    check(cb_.allreduce(cb_.ctx, buf, count, (int)op, (int)team), "allreduce");
  }
  void send(const double* buf, size_t count, int peer) override {
    sync_();
    check(cb_.send(cb_.ctx, buf, count, peer), "send");
  }
  void recv(double* buf, size_t count, int peer) override {
    sync_();
    check(cb_.recv(cb_.ctx, buf, count, peer), "recv");
  }

 private:
  static void check(int rc, const char* what) {
    if (rc != 0) throw InvalidArgument(std::string("communicator callback failed: ") + what);
  }
  CommCallbacks cb_;
  int rank_, world_;
  std::function<void()> sync_;
};
}  // namespace

Comm* callback_comm_create(const CommCallbacks& cb, int rank, int world, const Grid& g,
                           std::function<void()> sync) {
  if (!cb.bcast || !cb.allreduce || !cb.send || !cb.recv)
    throw InvalidArgument("communicator callbacks: bcast, allreduce, send and recv are required");
  return new CallbackComm(cb, rank, world, g, std::move(sync));
}

}  // namespace dist
}  // namespace qdwhg
