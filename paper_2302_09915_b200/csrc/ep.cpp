#include "ep.hpp"

#include <stdexcept>
#include <string>

#include "common.hpp"

namespace tamoe {

static void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw std::runtime_error(std::string(what) + ": " + ncclGetErrorString(r));
}
#define TAMOE_NCCL(expr) nccl_check((expr), #expr)

void ep_plan(int P, int E, const long long* recv, int* seg_start, int* seg_rows, long long* blk_off,
             long long* blk_rows) {
  long long row = 0;
  for (int i = 0; i < P; ++i) {
    blk_off[i] = row;
    for (int e = 0; e < E; ++e) {
      const long long r = (recv[i * E + e] + 15) / 16 * 16;
      seg_start[i * E + e] = static_cast<int>(row);
      seg_rows[i * E + e] = static_cast<int>(r);
      row += r;
    }
    blk_rows[i] = row - blk_off[i];
  }
}

EpComm::EpComm(int world, int rank, const ncclUniqueId& id) : world_(world), rank_(rank) {
  require(world >= 1 && rank >= 0 && rank < world, "bad expert-parallel world / rank");
  TAMOE_NCCL(ncclCommInitRank(&comm_, world, id, rank));
}

EpComm::~EpComm() {
  if (comm_) ncclCommDestroy(comm_);
  if (h_counts_) cudaFreeHost(h_counts_);
}

void EpComm::exchange_counts(const int* my_counts, int* recv_counts, int N, cudaStream_t s) {
  require(N % world_ == 0, "N must be divisible by the number of ranks");
  E_ = N / world_;
  if (!h_counts_) TAMOE_CUDA(cudaMallocHost(&h_counts_, sizeof(int) * (N + world_ * E_)));
  TAMOE_NCCL(ncclGroupStart());
  for (int j = 0; j < world_; ++j) {
    TAMOE_NCCL(ncclSend(my_counts + j * E_, E_, ncclInt32, j, comm_, s));
    TAMOE_NCCL(ncclRecv(recv_counts + j * E_, E_, ncclInt32, j, comm_, s));
  }
  TAMOE_NCCL(ncclGroupEnd());
  TAMOE_CUDA(cudaMemcpyAsync(h_counts_, my_counts, sizeof(int) * N, cudaMemcpyDeviceToHost, s));
  TAMOE_CUDA(cudaMemcpyAsync(h_counts_ + N, recv_counts, sizeof(int) * world_ * E_, cudaMemcpyDeviceToHost, s));
  TAMOE_CUDA(cudaStreamSynchronize(s));
  plan(N);
}

void EpComm::plan(int N) {
  send_cnt_.assign(h_counts_, h_counts_ + N);
  send_blk_off_.assign(world_, 0);
  send_blk_rows_.assign(world_, 0);
  long long row = 0;
  for (int j = 0; j < world_; ++j) {
    send_blk_off_[j] = row;
    for (int e = 0; e < E_; ++e) row += (send_cnt_[j * E_ + e] + 15) / 16 * 16;
    send_blk_rows_[j] = row - send_blk_off_[j];
  }
  recv_cnt_.assign(h_counts_ + N, h_counts_ + N + world_ * E_);
  seg_start_.assign(world_ * E_, 0);
  seg_rows_.assign(world_ * E_, 0);
  recv_blk_off_.assign(world_, 0);
  recv_blk_rows_.assign(world_, 0);
  ep_plan(world_, E_, recv_cnt_.data(), seg_start_.data(), seg_rows_.data(), recv_blk_off_.data(),
          recv_blk_rows_.data());
  recv_rows_ = static_cast<int>(recv_blk_off_[world_ - 1] + recv_blk_rows_[world_ - 1]);
}

void EpComm::dispatch(const __nv_bfloat16* send, __nv_bfloat16* recv, int w, cudaStream_t s) {
  last_bytes_ = 0;
  TAMOE_NCCL(ncclGroupStart());
  for (int j = 0; j < world_; ++j)
    if (send_blk_rows_[j] > 0) {
      TAMOE_NCCL(ncclSend(send + send_blk_off_[j] * w, static_cast<size_t>(send_blk_rows_[j]) * w, ncclBfloat16, j,
                          comm_, s));
      if (j != rank_) last_bytes_ += send_blk_rows_[j] * w * 2;
    }
  for (int i = 0; i < world_; ++i)
    if (recv_blk_rows_[i] > 0)
      TAMOE_NCCL(ncclRecv(recv + recv_blk_off_[i] * w, static_cast<size_t>(recv_blk_rows_[i]) * w, ncclBfloat16, i,
                          comm_, s));
  TAMOE_NCCL(ncclGroupEnd());
}

void EpComm::combine(const __nv_bfloat16* recv, __nv_bfloat16* send, int w, cudaStream_t s) {
  last_bytes_ = 0;
  TAMOE_NCCL(ncclGroupStart());
  for (int i = 0; i < world_; ++i)
    if (recv_blk_rows_[i] > 0) {
      TAMOE_NCCL(ncclSend(recv + recv_blk_off_[i] * w, static_cast<size_t>(recv_blk_rows_[i]) * w, ncclBfloat16, i,
                          comm_, s));
      if (i != rank_) last_bytes_ += recv_blk_rows_[i] * w * 2;
    }
  for (int j = 0; j < world_; ++j)
    if (send_blk_rows_[j] > 0)
      TAMOE_NCCL(ncclRecv(send + send_blk_off_[j] * w, static_cast<size_t>(send_blk_rows_[j]) * w, ncclBfloat16, j,
                          comm_, s));
  TAMOE_NCCL(ncclGroupEnd());
}

}  // namespace tamoe
