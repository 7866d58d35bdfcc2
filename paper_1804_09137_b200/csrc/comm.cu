// comm.cu — NCCL and loopback communicators (comm.cuh).
#include "comm.cuh"
#include <condition_variable>
#include <mutex>
#include <stdexcept>

namespace tlrb {

#define TLRB_NCCL_CHECK(call)                                                                         \
  do {                                                                                                \
    ncclResult_t r_ = (call);                                                                         \
    if (r_ != ncclSuccess) throw CudaError(cudaErrorUnknown, ncclGetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

namespace {

ncclDataType_t nccl_type(CType t) { return t == CType::I32 ? ncclInt32 : ncclFloat64; }

class NcclComm final : public Comm {
 public:
  explicit NcclComm(ncclComm_t c) : c_(c) {
    TLRB_NCCL_CHECK(ncclCommUserRank(c_, &rank_));
    TLRB_NCCL_CHECK(ncclCommCount(c_, &size_));
  }
  ~NcclComm() override {
    if (c_) ncclCommDestroy(c_);
  }
  int rank() const override { return rank_; }
  int size() const override { return size_; }
  const char* kind() const override { return "nccl"; }
  ncclComm_t raw() const { return c_; }
  void bcast(void* buf, size_t count, CType t, int root, cudaStream_t s) override {
    if (size_ < 2 || !count) return;
    TLRB_NCCL_CHECK(ncclBroadcast(buf, buf, count, nccl_type(t), root, c_, s));
  }
  void allreduce_sum(void* buf, size_t count, CType t, cudaStream_t s) override {
    if (size_ < 2 || !count) return;
    TLRB_NCCL_CHECK(ncclAllReduce(buf, buf, count, nccl_type(t), ncclSum, c_, s));
  }
  void reduce_sum(void* buf, size_t count, CType t, int root, cudaStream_t s) override {
    if (size_ < 2 || !count) return;
    TLRB_NCCL_CHECK(ncclReduce(buf, buf, count, nccl_type(t), ncclSum, root, c_, s));
  }
  void abort() override {
    if (c_) ncclCommAbort(c_);
    c_ = nullptr;
  }

 private:
  ncclComm_t c_ = nullptr;
  int rank_ = 0, size_ = 1;
};

template <class T>
__global__ void ordered_sum_kernel(T* __restrict__ out, const T* __restrict__ parts, size_t count, int n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    T a = parts[i];
    for (int m = 1; m < n; ++m) a += parts[(size_t)m * count + i];   // member order 0, 1, ..., n-1
    out[i] = a;
  }
}

}  // namespace

// --------------------------------------------------------------- loopback
struct LocalGroup {
  explicit LocalGroup(int n) : n(n), slots(n) {}
  struct Slot {
    void* buf = nullptr;      // the member's in-place buffer of the current collective
    void* stage = nullptr;    // its staged copy (reductions)
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  const int n;
  std::vector<Slot> slots;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool aborted = false;

  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw CudaError(cudaErrorUnknown, "loopback collective aborted by another rank", __FILE__, __LINE__);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    cv.wait(lk, [&] { return gen != g || aborted; });
    if (aborted) throw CudaError(cudaErrorUnknown, "loopback collective aborted by another rank", __FILE__, __LINE__);
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

std::shared_ptr<LocalGroup> make_local_group(int size) { return std::make_shared<LocalGroup>(size); }

namespace {

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank, int device) : g_(std::move(g)), rank_(rank), dev_(device) {
    TLRB_CUDA(cudaSetDevice(dev_));
    auto& sl = g_->slots[rank_];
    TLRB_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
    TLRB_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
  }
  ~LocalComm() override {
    auto& sl = g_->slots[rank_];
    if (sl.ready) cudaEventDestroy(sl.ready);
    if (sl.done) cudaEventDestroy(sl.done);
    if (stage_) cudaFree(stage_);
    if (gather_) cudaFree(gather_);
  }
  int rank() const override { return rank_; }
  int size() const override { return g_->n; }
  const char* kind() const override { return "loopback"; }

  void bcast(void* buf, size_t count, CType t, int root, cudaStream_t s) override {
    const size_t bytes = count * ctype_size(t);
    if (g_->n < 2 || !bytes) return;
    auto& sl = g_->slots;
    sl[rank_].buf = buf;
    TLRB_CUDA(cudaEventRecord(sl[rank_].ready, s));
    g_->barrier();   // 1: every member published its buffer / ready event
    if (rank_ != root) {
      TLRB_CUDA(cudaStreamWaitEvent(s, sl[root].ready, 0));
      TLRB_CUDA(cudaMemcpyAsync(buf, sl[root].buf, bytes, cudaMemcpyDefault, s));
    }
    TLRB_CUDA(cudaEventRecord(sl[rank_].done, s));
    g_->barrier();   // 2: every copy is enqueued
    if (rank_ == root)   // the root's buffer stays untouched until the copies are done
      for (int m = 0; m < g_->n; ++m)
        if (m != root) TLRB_CUDA(cudaStreamWaitEvent(s, sl[m].done, 0));
    g_->barrier();   // 3: waits enqueued before any event is recorded again
  }

  void allreduce_sum(void* buf, size_t count, CType t, cudaStream_t s) override { reduce(buf, count, t, -1, s); }
  void reduce_sum(void* buf, size_t count, CType t, int root, cudaStream_t s) override {
    reduce(buf, count, t, root, s);
  }
  void abort() override { g_->abort(); }

 private:
  // root < 0: all-reduce
  void reduce(void* buf, size_t count, CType t, int root, cudaStream_t s) {
    const size_t bytes = count * ctype_size(t);
    const int n = g_->n;
    if (n < 2 || !bytes) return;
    auto& sl = g_->slots;
    grow(stage_, stage_cap_, bytes);
    TLRB_CUDA(cudaMemcpyAsync(stage_, buf, bytes, cudaMemcpyDeviceToDevice, s));
    sl[rank_].stage = stage_;
    TLRB_CUDA(cudaEventRecord(sl[rank_].ready, s));
    g_->barrier();   // 1: every member's contribution is staged (stream ordered)
    const bool me = root < 0 || rank_ == root;
    if (me) {
      grow(gather_, gather_cap_, bytes * n);
      for (int m = 0; m < n; ++m) {
        if (m != rank_) TLRB_CUDA(cudaStreamWaitEvent(s, sl[m].ready, 0));
        TLRB_CUDA(cudaMemcpyAsync(static_cast<char*>(gather_) + (size_t)m * bytes, sl[m].stage, bytes,
                                  cudaMemcpyDefault, s));
      }
      const int blocks = (int)std::min<size_t>(1184, (count + 255) / 256);
      if (t == CType::I32)
        ordered_sum_kernel<int><<<blocks, 256, 0, s>>>(static_cast<int*>(buf), static_cast<const int*>(gather_),
                                                       count, n);
      else
        ordered_sum_kernel<double><<<blocks, 256, 0, s>>>(static_cast<double*>(buf),
                                                          static_cast<const double*>(gather_), count, n);
      post_launch();
    }
    TLRB_CUDA(cudaEventRecord(sl[rank_].done, s));
    g_->barrier();   // 2: every read of the staged buffers is enqueued
    // a member's stage is free once every reader is done with it
    for (int m = 0; m < n; ++m)
      if (m != rank_ && (root < 0 || m == root)) TLRB_CUDA(cudaStreamWaitEvent(s, sl[m].done, 0));
    g_->barrier();   // 3: waits enqueued before any event is recorded again
  }

  void grow(void*& p, size_t& cap, size_t bytes) {
    if (bytes <= cap) return;
    // only this member reads / writes its own buffers between collectives;
    // readers of the previous collective were waited for (barrier 3 + event)
    if (p) {
      TLRB_CUDA(cudaDeviceSynchronize());
      TLRB_CUDA(cudaFree(p));
    }
    cap = std::max(bytes, cap + cap / 2);
    TLRB_CUDA(cudaMalloc(&p, cap));
  }

  std::shared_ptr<LocalGroup> g_;
  int rank_, dev_;
  void* stage_ = nullptr;
  size_t stage_cap_ = 0;
  void* gather_ = nullptr;
  size_t gather_cap_ = 0;
};

}  // namespace

std::unique_ptr<Comm> make_nccl_comm(ncclComm_t c) { return std::make_unique<NcclComm>(c); }

std::unique_ptr<Comm> split_nccl_comm(Comm& parent, int color, int key) {
  auto* p = dynamic_cast<NcclComm*>(&parent);
  if (!p) throw CudaError(cudaErrorInvalidValue, "split of a non-NCCL communicator", __FILE__, __LINE__);
  ncclComm_t c = nullptr;
  TLRB_NCCL_CHECK(ncclCommSplit(p->raw(), color, key, &c, nullptr));
  return make_nccl_comm(c);
}

std::unique_ptr<Comm> make_local_comm(std::shared_ptr<LocalGroup> g, int rank, int device) {
  return std::make_unique<LocalComm>(std::move(g), rank, device);
}

}  // namespace tlrb
