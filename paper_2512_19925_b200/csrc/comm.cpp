// NCCL and loopback implementations of the driver's collectives (comm.h).
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "capi_util.h"

#define COMM_CUDA(call)                                                                 \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      throw ::hwwg::CudaError(std::string(#call) + ": " + cudaGetErrorString(e_));      \
  } while (0)

// NCCL is opened at run time, only by a multi-GPU driver: a link-time
// dependency on libnccl.so.2 would put the system NCCL in the process first,
// and torch (whose bundled NCCL is newer) then fails to import next to it. With
// dlopen, "libnccl.so.2" resolves to the copy already loaded (torch's, under
// torchrun) or the system one otherwise.
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclGroupStart) GroupStart = nullptr;
  decltype(&ncclGroupEnd) GroupEnd = nullptr;
  decltype(&ncclSend) Send = nullptr;
  decltype(&ncclRecv) Recv = nullptr;
  decltype(&ncclGetErrorString) GetErrorString = nullptr;
};

static const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw hwwg::ApiError(HWWG_ECUDA, std::string("cannot load NCCL: ") + dlerror());
    auto sym = [&](auto& f, const char* name) {
      f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(h, name));
      if (!f) throw hwwg::ApiError(HWWG_ECUDA, std::string("NCCL symbol missing: ") + name);
    };
    sym(a.GetUniqueId, "ncclGetUniqueId");
    sym(a.CommInitRank, "ncclCommInitRank");
    sym(a.CommDestroy, "ncclCommDestroy");
    sym(a.AllReduce, "ncclAllReduce");
    sym(a.AllGather, "ncclAllGather");
    sym(a.GroupStart, "ncclGroupStart");
    sym(a.GroupEnd, "ncclGroupEnd");
    sym(a.Send, "ncclSend");
    sym(a.Recv, "ncclRecv");
    sym(a.GetErrorString, "ncclGetErrorString");
    return a;
  }();
  return api;
}

#define COMM_NCCL(call)                                                                   \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      throw ::hwwg::ApiError(HWWG_ECUDA,                                                   \
                             std::string(#call) + ": " + nccl().GetErrorString(r_));       \
  } while (0)

// In-process hub of the loopback ranks: one stream, staging, mailboxes, barrier.
struct hwwg_loopback {
  int world = 1;
  int device = 0;
  cudaStream_t stream = nullptr;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;  // a rank failed mid-collective: release the others
  std::vector<std::vector<unsigned char>> stage;
  std::map<std::pair<int, int>, std::deque<std::vector<unsigned char>>> mail;

  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) throw hwwg::ApiError(HWWG_ESTATE, "loopback peer failed");
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || broken; });
    if (broken && gen == g) throw hwwg::ApiError(HWWG_ESTATE, "loopback peer failed");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(m);
    broken = true;
    cv.notify_all();
  }
};

namespace hwwg {

namespace {

ncclDataType_t nccl_type(DType t) {
  return t == DType::kF64 ? ncclDouble : (t == DType::kU64 ? ncclUint64 : ncclUint32);
}

class NcclComm final : public Comm {
 public:
  NcclComm(const uint8_t id_bytes[128], int rank, int world) : rank_(rank), world_(world) {
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    COMM_NCCL(nccl().CommInitRank(&comm_, world, id, rank));
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int world() const override { return world_; }
  void all_reduce(const void* send, void* recv, size_t count, DType t, RedOp op,
                  cudaStream_t s) override {
    COMM_NCCL(nccl().AllReduce(send, recv, count, nccl_type(t), op == RedOp::kSum ? ncclSum : ncclMax,
                            comm_, s));
  }
  void all_gather(const void* send, void* recv, size_t count, DType t, cudaStream_t s) override {
    COMM_NCCL(nccl().AllGather(send, recv, count, nccl_type(t), comm_, s));
  }
  void group_start() override { COMM_NCCL(nccl().GroupStart()); }
  void send(const void* buf, size_t count, DType t, int peer, cudaStream_t s) override {
    COMM_NCCL(nccl().Send(buf, count, nccl_type(t), peer, comm_, s));
  }
  void recv(void* buf, size_t count, DType t, int peer, cudaStream_t s) override {
    COMM_NCCL(nccl().Recv(buf, count, nccl_type(t), peer, comm_, s));
  }
  void group_end(cudaStream_t) override { COMM_NCCL(nccl().GroupEnd()); }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
};

class LoopbackComm final : public Comm {
 public:
  LoopbackComm(hwwg_loopback* hub, int rank) : hub_(hub), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return hub_->world; }
  cudaStream_t shared_stream() const override { return hub_->stream; }

  void all_reduce(const void* send, void* recv, size_t count, DType t, RedOp op,
                  cudaStream_t s) override {
    guarded([&] {
      const size_t bytes = count * dtype_bytes(t);
      post(send, bytes, s);
      hub_->barrier();
      std::vector<unsigned char> out(hub_->stage[0]);  // rank order: deterministic
      for (int r = 1; r < hub_->world; ++r) {
        const unsigned char* in = hub_->stage[r].data();
        for (size_t i = 0; i < count; ++i) combine(out.data(), in, i, t, op);
      }
      hub_->barrier();  // every rank has read the staging buffers
      COMM_CUDA(cudaMemcpyAsync(recv, out.data(), bytes, cudaMemcpyHostToDevice, s));
      COMM_CUDA(cudaStreamSynchronize(s));
    });
  }
  void all_gather(const void* send, void* recv, size_t count, DType t, cudaStream_t s) override {
    guarded([&] {
      const size_t bytes = count * dtype_bytes(t);
      post(send, bytes, s);
      hub_->barrier();
      std::vector<unsigned char> out(bytes * hub_->world);
      for (int r = 0; r < hub_->world; ++r)
        if (bytes) std::memcpy(out.data() + bytes * r, hub_->stage[r].data(), bytes);
      hub_->barrier();
      COMM_CUDA(cudaMemcpyAsync(recv, out.data(), out.size(), cudaMemcpyHostToDevice, s));
      COMM_CUDA(cudaStreamSynchronize(s));
    });
  }
  void group_start() override { pending_.clear(); }
  void send(const void* buf, size_t count, DType t, int peer, cudaStream_t s) override {
    guarded([&] {
      std::vector<unsigned char> v(count * dtype_bytes(t));
      COMM_CUDA(cudaStreamSynchronize(s));
      if (!v.empty()) COMM_CUDA(cudaMemcpy(v.data(), buf, v.size(), cudaMemcpyDeviceToHost));
      std::lock_guard<std::mutex> lk(hub_->m);
      hub_->mail[{rank_, peer}].push_back(std::move(v));
    });
  }
  void recv(void* buf, size_t count, DType t, int peer, cudaStream_t) override {
    pending_.push_back(Pending{buf, count * dtype_bytes(t), peer});
  }
  void group_end(cudaStream_t s) override {
    guarded([&] {
      hub_->barrier();  // every send of the group is posted
      for (const Pending& p : pending_) {
        std::vector<unsigned char> v;
        {
          std::lock_guard<std::mutex> lk(hub_->m);
          auto& q = hub_->mail[{p.peer, rank_}];
          if (q.empty()) throw ApiError(HWWG_ESTATE, "loopback recv without a matching send");
          v = std::move(q.front());
          q.pop_front();
        }
        if (v.size() != p.bytes) throw ApiError(HWWG_ESTATE, "loopback send/recv size mismatch");
        if (!v.empty()) COMM_CUDA(cudaMemcpy(p.buf, v.data(), v.size(), cudaMemcpyHostToDevice));
      }
      pending_.clear();
      COMM_CUDA(cudaStreamSynchronize(s));
      hub_->barrier();
    });
  }

 private:
  struct Pending {
    void* buf;
    size_t bytes;
    int peer;
  };
  hwwg_loopback* hub_;
  int rank_;
  std::vector<Pending> pending_;

  // a failing rank releases its peers (they would wait at the barrier forever)
  template <class F>
  void guarded(F f) {
    try {
      f();
    } catch (...) {
      hub_->abort();
      throw;
    }
  }
  void post(const void* send, size_t bytes, cudaStream_t s) {
    COMM_CUDA(cudaStreamSynchronize(s));
    std::vector<unsigned char>& st = hub_->stage[rank_];
    st.resize(bytes);
    if (bytes) COMM_CUDA(cudaMemcpy(st.data(), send, bytes, cudaMemcpyDeviceToHost));
  }
  static void combine(unsigned char* out, const unsigned char* in, size_t i, DType t, RedOp op) {
    if (t == DType::kF64) {
      double a, b;
      std::memcpy(&a, out + 8 * i, 8);
      std::memcpy(&b, in + 8 * i, 8);
      const double r = op == RedOp::kSum ? a + b : (b > a ? b : a);
      std::memcpy(out + 8 * i, &r, 8);
    } else if (t == DType::kU64) {
      unsigned long long a, b;
      std::memcpy(&a, out + 8 * i, 8);
      std::memcpy(&b, in + 8 * i, 8);
      const unsigned long long r = op == RedOp::kSum ? a + b : (b > a ? b : a);
      std::memcpy(out + 8 * i, &r, 8);
    } else {
      unsigned a, b;
      std::memcpy(&a, out + 4 * i, 4);
      std::memcpy(&b, in + 4 * i, 4);
      const unsigned r = op == RedOp::kSum ? a + b : (b > a ? b : a);
      std::memcpy(out + 4 * i, &r, 4);
    }
  }
};

}  // namespace

Comm* make_nccl_comm(const uint8_t id[128], int rank, int world) {
  return new NcclComm(id, rank, world);
}
Comm* make_loopback_comm(hwwg_loopback* hub, int rank) { return new LoopbackComm(hub, rank); }
int loopback_world(const hwwg_loopback* hub) { return hub->world; }

}  // namespace hwwg

extern "C" {

int hwwg_loopback_create(int32_t world, int32_t device, hwwg_loopback** out) {
  HWWG_API_BEGIN
  if (!out || world < 1) return hwwg::fail(HWWG_EINVAL, "loopback: world >= 1 and out required");
  *out = nullptr;
  auto* h = new hwwg_loopback();
  h->world = world;
  h->device = device;
  h->stage.resize(world);
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    cudaGetLastError();
    delete h;
    return hwwg::fail(HWWG_ECUDA, std::string("loopback: ") + cudaGetErrorString(e));
  }
  *out = h;
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_nccl_unique_id(uint8_t* out) {
  HWWG_API_BEGIN
  if (!out) return hwwg::fail(HWWG_EINVAL, "NULL argument");
  ncclUniqueId id;
  COMM_NCCL(nccl().GetUniqueId(&id));
  std::memset(out, 0, 128);
  std::memcpy(out, &id, sizeof(id) < 128 ? sizeof(id) : 128);
  return HWWG_OK;
  HWWG_API_END
}

int hwwg_nccl_selftest(int32_t device, uint8_t* report, uint64_t report_bytes) {
  HWWG_API_BEGIN
  // The driver's NCCL collectives on a one-rank communicator: the run-time
  // NCCL load, the unique-id hand-off, CommInitRank and every call the
  // multi-GPU driver makes (sum/max all-reduce, all-gather, grouped
  // send/recv — here to itself), with their results checked.
  COMM_CUDA(cudaSetDevice(device));
  uint8_t id[128];
  {
    ncclUniqueId u;
    COMM_NCCL(nccl().GetUniqueId(&u));
    std::memset(id, 0, sizeof id);
    std::memcpy(id, &u, sizeof(u) < 128 ? sizeof(u) : 128);
  }
  cudaStream_t s;
  COMM_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::string msg;
  {
    using namespace hwwg;
    std::unique_ptr<Comm> cp(make_nccl_comm(id, 0, 1));
    Comm& c = *cp;
    const double hd[3] = {1.5, -2.0, 3.25};
    const unsigned long long hu[2] = {7ULL, 1ULL << 40};
    void* dmem = nullptr;
    COMM_CUDA(cudaMalloc(&dmem, 256));
    double* d_in = static_cast<double*>(dmem);
    double* d_out = d_in + 4;
    unsigned long long* u_in = reinterpret_cast<unsigned long long*>(d_in + 8);
    unsigned long long* u_out = u_in + 4;
    COMM_CUDA(cudaMemcpy(d_in, hd, sizeof hd, cudaMemcpyHostToDevice));
    COMM_CUDA(cudaMemcpy(u_in, hu, sizeof hu, cudaMemcpyHostToDevice));
    c.all_reduce(d_in, d_out, 3, DType::kF64, RedOp::kSum, s);
    c.all_reduce(u_in, u_out, 2, DType::kU64, RedOp::kMax, s);
    double rd[3];
    unsigned long long ru[2], rg[2], rs[2];
    COMM_CUDA(cudaStreamSynchronize(s));
    COMM_CUDA(cudaMemcpy(rd, d_out, sizeof rd, cudaMemcpyDeviceToHost));
    COMM_CUDA(cudaMemcpy(ru, u_out, sizeof ru, cudaMemcpyDeviceToHost));
    c.all_gather(u_in, u_out, 2, DType::kU64, s);
    COMM_CUDA(cudaStreamSynchronize(s));
    COMM_CUDA(cudaMemcpy(rg, u_out, sizeof rg, cudaMemcpyDeviceToHost));
    COMM_CUDA(cudaMemset(u_out, 0, 16));
    c.group_start();
    c.send(u_in, 2, DType::kU64, 0, s);
    c.recv(u_out, 2, DType::kU64, 0, s);
    c.group_end(s);
    COMM_CUDA(cudaStreamSynchronize(s));
    COMM_CUDA(cudaMemcpy(rs, u_out, sizeof rs, cudaMemcpyDeviceToHost));
    COMM_CUDA(cudaFree(dmem));
    for (int i = 0; i < 3; ++i)
      if (rd[i] != hd[i]) msg += "all_reduce sum f64 differs; ";
    for (int i = 0; i < 2; ++i) {
      if (ru[i] != hu[i]) msg += "all_reduce max u64 differs; ";
      if (rg[i] != hu[i]) msg += "all_gather u64 differs; ";
      if (rs[i] != hu[i]) msg += "send/recv u64 differs; ";
    }
  }
  COMM_CUDA(cudaStreamDestroy(s));
  if (report && report_bytes) {
    const std::string r = msg.empty() ? "ok" : msg;
    std::memset(report, 0, report_bytes);
    std::memcpy(report, r.data(), std::min<size_t>(r.size(), report_bytes - 1));
  }
  return msg.empty() ? HWWG_OK : hwwg::fail(HWWG_ECUDA, "nccl self-test: " + msg);
  HWWG_API_END
}

void hwwg_loopback_destroy(hwwg_loopback* h) {
  if (!h) return;
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

}  // extern "C"
