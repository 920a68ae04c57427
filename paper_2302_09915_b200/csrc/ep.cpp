#include "ep.hpp"

#include <cstring>
#include <stdexcept>
#include <string>

#include "common.hpp"

namespace tamoe {

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}
#define TAMOE_NCCL(expr) nccl_check((expr), #expr)

void ep_plan(int P, int E, const long long* recv, int* seg_start, int* seg_rows, long long* src_off) {
  long long row = 0;
  for (int e = 0; e < E; ++e) {
    seg_start[e] = static_cast<int>(row);
    for (int i = 0; i < P; ++i) {
      src_off[i * E + e] = row;
      row += (recv[i * E + e] + 15) / 16 * 16;
    }
    seg_rows[e] = static_cast<int>(row - seg_start[e]);
  }
}

EpComm::EpComm(int world, int rank, const ncclUniqueId& id) : world_(world), rank_(rank) {
  require(world >= 1 && world <= kMaxRanks && rank >= 0 && rank < world, "bad expert-parallel world / rank");
  TAMOE_NCCL(ncclCommInitRank(&comm_, world, id, rank));
}

EpComm::~EpComm() {
  close_peers();
  if (comm_) ncclCommDestroy(comm_);
}

void EpComm::close_peers() {
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  opened_.clear();
}

void EpComm::allgather_counts(const int* my_counts, int* all_counts, int N, cudaStream_t s) {
  TAMOE_NCCL(ncclAllGather(my_counts, all_counts, N, ncclInt32, comm_, s));
}

void EpComm::barrier(int* flag, cudaStream_t s) {
  TAMOE_NCCL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, comm_, s));
}

void EpComm::allreduce_sum(double* buf, size_t n, cudaStream_t s) {
  TAMOE_NCCL(ncclAllReduce(buf, buf, n, ncclFloat64, ncclSum, comm_, s));
}

void EpComm::map_peers(void* local_base, std::vector<char*>& bases) {
  cudaIpcMemHandle_t h;
  TAMOE_CUDA(cudaIpcGetMemHandle(&h, local_base));
  char* d_buf = nullptr;
  const size_t hs = sizeof(cudaIpcMemHandle_t);
  TAMOE_CUDA(cudaMalloc(&d_buf, hs * (world_ + 1)));
  TAMOE_CUDA(cudaMemcpy(d_buf + hs * world_, &h, hs, cudaMemcpyHostToDevice));
  TAMOE_NCCL(ncclAllGather(d_buf + hs * world_, d_buf, hs, ncclChar, comm_, nullptr));
  TAMOE_CUDA(cudaStreamSynchronize(nullptr));
  std::vector<cudaIpcMemHandle_t> all(world_);
  TAMOE_CUDA(cudaMemcpy(all.data(), d_buf, hs * world_, cudaMemcpyDeviceToHost));
  TAMOE_CUDA(cudaFree(d_buf));
  bases.assign(world_, nullptr);
  for (int j = 0; j < world_; ++j) {
    if (j == rank_) {
      bases[j] = static_cast<char*>(local_base);
    } else {
      void* p = nullptr;
      TAMOE_CUDA(cudaIpcOpenMemHandle(&p, all[j], cudaIpcMemLazyEnablePeerAccess));
      opened_.push_back(p);
      bases[j] = static_cast<char*>(p);
    }
  }
}

P2PProbe::P2PProbe(int world, int rank, const ncclUniqueId& id, size_t max_bytes)
    : comm_(world, rank, id), max_bytes_(max_bytes) {
  require(max_bytes >= 16, "p2p probe buffer too small");
  TAMOE_CUDA(cudaMalloc(&buf_, 2 * max_bytes_));
  TAMOE_CUDA(cudaMemset(buf_, 1, 2 * max_bytes_));
  TAMOE_CUDA(cudaMalloc(&flag_, sizeof(int)));
  TAMOE_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  comm_.map_peers(buf_, bases_);
}

P2PProbe::~P2PProbe() {
  // every rank unmaps the others' buffers before anybody frees its own
  comm_.close_peers();
  if (flag_ && stream_) {
    try {
      comm_.barrier(flag_, stream_);
    } catch (...) {
    }
    cudaStreamSynchronize(stream_);
  }
  if (stream_) cudaStreamDestroy(stream_);
  if (flag_) cudaFree(flag_);
  if (buf_) cudaFree(buf_);
}

std::vector<double> P2PProbe::sweep(const double* sizes_mb, int nsizes, int reps, int warmup) {
  const int W = comm_.world(), me = comm_.rank();
  require(nsizes >= 1 && reps >= 1 && warmup >= 0, "p2p sweep: bad sizes / reps");
  for (int s = 0; s < nsizes; ++s)
    require(sizes_mb[s] > 0.0 && sizes_mb[s] * 1e6 <= static_cast<double>(max_bytes_),
            "p2p sweep: message size outside the probe buffer");
  std::vector<double> out(static_cast<size_t>(W) * W * nsizes * reps, 0.0);
  cudaEvent_t e0, e1;
  TAMOE_CUDA(cudaEventCreate(&e0));
  TAMOE_CUDA(cudaEventCreate(&e1));
  for (int src = 0; src < W; ++src)
    for (int dst = 0; dst < W; ++dst)
      for (int si = 0; si < nsizes; ++si) {
        const size_t bytes = (static_cast<size_t>(sizes_mb[si] * 1e6) + 15) & ~static_cast<size_t>(15);
        for (int r = -warmup; r < reps; ++r) {
          comm_.barrier(flag_, stream_);  // everybody idle, previous transfer done
          if (me == src) {
            TAMOE_CUDA(cudaEventRecord(e0, stream_));
            p2p_copy(bases_[static_cast<size_t>(dst)] + max_bytes_, buf_, bytes, stream_,
                     link_emulation().factor(src, dst));
            TAMOE_CUDA(cudaEventRecord(e1, stream_));
            TAMOE_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            TAMOE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (r >= 0) out[((static_cast<size_t>(src) * W + dst) * nsizes + si) * reps + r] = ms * 1e3;
          }
        }
      }
  TAMOE_CUDA(cudaStreamSynchronize(stream_));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  // every entry was written by exactly one rank: a sum all-reduce gathers them
  double* d = nullptr;
  TAMOE_CUDA(cudaMalloc(&d, sizeof(double) * out.size()));
  TAMOE_CUDA(cudaMemcpy(d, out.data(), sizeof(double) * out.size(), cudaMemcpyHostToDevice));
  comm_.allreduce_sum(d, out.size(), stream_);
  TAMOE_CUDA(cudaStreamSynchronize(stream_));
  TAMOE_CUDA(cudaMemcpy(out.data(), d, sizeof(double) * out.size(), cudaMemcpyDeviceToHost));
  cudaFree(d);
  return out;
}

}  // namespace tamoe
