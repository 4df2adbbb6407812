// Process-group collectives of the engine.
//
// NcclGroup is the product path: NCCL over NVLink / NVSwitch, issued on CUDA
// streams (graph-capturable).  HostGroup runs the same operations through
// caller-supplied host callbacks (vnt_comm_ops, include/vnt_engine.h): the
// engine synchronises the stream, stages the device buffer through pinned
// memory and calls the callback.  It exists so that several engine processes
// (or threads) sharing ONE GPU can run the multi-rank code paths — sharded
// update, resize migration — with a host-side exchange (gloo, shared memory);
// no kernel ever waits on another rank's kernel.
#pragma once

#include <nccl.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/vnt_engine.h"
#include "common.cuh"

namespace vntb {

class CommGroup {
 public:
  CommGroup(int rank, int size) : rank_(rank), size_(size) {}
  virtual ~CommGroup() = default;
  int rank() const { return rank_; }
  int size() const { return size_; }
  // May be recorded into a CUDA graph / overlapped on a side stream.
  virtual bool on_stream() const = 0;
  virtual void allreduce_sum_i64(long long* buf, size_t n, cudaStream_t s) = 0;
  virtual void allreduce_max_u64(unsigned long long* buf, size_t n, cudaStream_t s) = 0;
  // recv[recv_n] = rank r's block of sum over ranks of send[size * recv_n]
  virtual void reduce_scatter_sum_i64(const long long* send, long long* recv, size_t recv_n,
                                      cudaStream_t s) = 0;
  // recv[size * bytes] = concat over ranks of send[bytes]
  virtual void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
  virtual void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) = 0;
  virtual void send(const void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, cudaStream_t s) = 0;
  // Collective over this group: the members passing color >= 0 form a new
  // group ranked by key; the others get nullptr.
  virtual std::unique_ptr<CommGroup> split(int color, int key) = 0;

 protected:
  int rank_, size_;
};

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw EngineError(VNT_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

class NcclGroup final : public CommGroup {
 public:
  // max_ctas > 0 caps the CTAs of this communicator's kernels (they run beside GEMMs).
  NcclGroup(const ncclUniqueId& id, int rank, int size, int max_ctas) : CommGroup(rank, size), ctas_(max_ctas) {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (max_ctas > 0) cfg.maxCTAs = max_ctas;
    nccl_check(ncclCommInitRankConfig(&comm_, size, id, rank, &cfg), "ncclCommInitRankConfig");
  }
  NcclGroup(ncclComm_t c, int rank, int size, int max_ctas) : CommGroup(rank, size), comm_(c), ctas_(max_ctas) {}
  ~NcclGroup() override {
    if (comm_) ncclCommDestroy(comm_);
  }
  bool on_stream() const override { return true; }
  void allreduce_sum_i64(long long* buf, size_t n, cudaStream_t s) override {
    nccl_check(ncclAllReduce(buf, buf, n, ncclInt64, ncclSum, comm_, s), "ncclAllReduce");
  }
  void allreduce_max_u64(unsigned long long* buf, size_t n, cudaStream_t s) override {
    nccl_check(ncclAllReduce(buf, buf, n, ncclUint64, ncclMax, comm_, s), "ncclAllReduce(max)");
  }
  void reduce_scatter_sum_i64(const long long* send, long long* recv, size_t recv_n,
                              cudaStream_t s) override {
    nccl_check(ncclReduceScatter(send, recv, recv_n, ncclInt64, ncclSum, comm_, s), "ncclReduceScatter");
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    nccl_check(ncclAllGather(send, recv, bytes, ncclUint8, comm_, s), "ncclAllGather");
  }
  void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    nccl_check(ncclBroadcast(buf, buf, bytes, ncclUint8, root, comm_, s), "ncclBroadcast");
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
    nccl_check(ncclSend(buf, bytes, ncclUint8, peer, comm_, s), "ncclSend");
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
    nccl_check(ncclRecv(buf, bytes, ncclUint8, peer, comm_, s), "ncclRecv");
  }
  std::unique_ptr<CommGroup> split(int color, int key) override {
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    if (ctas_ > 0) cfg.maxCTAs = ctas_;
    ncclComm_t c = nullptr;
    nccl_check(ncclCommSplit(comm_, color >= 0 ? color : NCCL_SPLIT_NOCOLOR, key, &c, &cfg),
               "ncclCommSplit");
    if (color < 0 || !c) return nullptr;
    int r = 0, n = 0;
    nccl_check(ncclCommUserRank(c, &r), "ncclCommUserRank");
    nccl_check(ncclCommCount(c, &n), "ncclCommCount");
    return std::make_unique<NcclGroup>(c, r, n, ctas_);
  }

 private:
  ncclComm_t comm_ = nullptr;
  int ctas_ = 0;
};

class HostGroup final : public CommGroup {
 public:
  explicit HostGroup(const vnt_comm_ops& ops) : CommGroup(ops.rank, ops.size), ops_(ops) {}
  ~HostGroup() override {
    if (a_) cudaFreeHost(a_);
    if (b_) cudaFreeHost(b_);
    if (ops_.release) ops_.release(ops_.ctx);
  }
  bool on_stream() const override { return false; }
  void allreduce_sum_i64(long long* buf, size_t n, cudaStream_t s) override {
    void* h = down(buf, n * 8, s);
    call(ops_.allreduce(ops_.ctx, h, n, VNT_COMM_SUM_I64), "allreduce");
    up(buf, h, n * 8, s);
  }
  void allreduce_max_u64(unsigned long long* buf, size_t n, cudaStream_t s) override {
    void* h = down(buf, n * 8, s);
    call(ops_.allreduce(ops_.ctx, h, n, VNT_COMM_MAX_U64), "allreduce(max)");
    up(buf, h, n * 8, s);
  }
  void reduce_scatter_sum_i64(const long long* send, long long* recv, size_t recv_n,
                              cudaStream_t s) override {
    void* h = down(send, recv_n * 8 * size_, s);
    void* r = stage(b_, bcap_, recv_n * 8);
    call(ops_.reduce_scatter(ops_.ctx, h, r, recv_n), "reduce_scatter");
    up(recv, r, recv_n * 8, s);
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    void* h = down(send, bytes, s);
    void* r = stage(b_, bcap_, bytes * size_);
    call(ops_.allgather(ops_.ctx, h, r, bytes), "allgather");
    up(recv, r, bytes * size_, s);
  }
  void broadcast(void* buf, size_t bytes, int root, cudaStream_t s) override {
    void* h = down(buf, bytes, s);
    call(ops_.broadcast(ops_.ctx, h, bytes, root), "broadcast");
    up(buf, h, bytes, s);
  }
  void send(const void* buf, size_t bytes, int peer, cudaStream_t s) override {
    void* h = down(buf, bytes, s);
    call(ops_.send(ops_.ctx, h, bytes, peer), "send");
  }
  void recv(void* buf, size_t bytes, int peer, cudaStream_t s) override {
    VNT_CUDA(cudaStreamSynchronize(s));
    void* h = stage(a_, acap_, bytes);
    call(ops_.recv(ops_.ctx, h, bytes, peer), "recv");
    up(buf, h, bytes, s);
  }
  std::unique_ptr<CommGroup> split(int color, int key) override {
    vnt_comm_ops sub{};
    call(ops_.split(ops_.ctx, color, key, &sub), "split");
    if (color < 0 || !sub.ctx) return nullptr;
    return std::make_unique<HostGroup>(sub);
  }

 private:
  static void call(int rc, const char* what) {
    if (rc != 0) throw EngineError(VNT_ERR_NCCL, std::string("host collective ") + what + " failed");
  }
  static void* stage(void*& p, size_t& cap, size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      cap = std::max<size_t>(bytes, 4096);
      VNT_CUDA(cudaMallocHost(&p, cap));
    }
    return p;
  }
  // device -> pinned staging (after the stream's pending work)
  void* down(const void* dev, size_t bytes, cudaStream_t s) {
    void* h = stage(a_, acap_, bytes);
    VNT_CUDA(cudaMemcpyAsync(h, dev, bytes, cudaMemcpyDeviceToHost, s));
    VNT_CUDA(cudaStreamSynchronize(s));
    return h;
  }
  void up(void* dev, const void* h, size_t bytes, cudaStream_t s) {
    VNT_CUDA(cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice, s));
    VNT_CUDA(cudaStreamSynchronize(s));   // the staging buffer is reused by the next call
  }
  vnt_comm_ops ops_;
  void *a_ = nullptr, *b_ = nullptr;
  size_t acap_ = 0, bcap_ = 0;
};

}  // namespace vntb
