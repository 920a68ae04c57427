// Expert-parallel exchange over NCCL (NVLink / NVSwitch): the real all-to-all that the
// reference only models (comm_cost.cpp:24-55, exchange_cost).  Rank j owns experts
// [jE, (j+1)E) (dispatch.hpp:31); rank i sends c_ie rows to expert e (dispatch.cpp:21-26).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <vector>

namespace tamoe {

class EpComm {
 public:
  EpComm(int world, int rank, const ncclUniqueId& id);
  ~EpComm();
  int world() const { return world_; }
  int rank() const { return rank_; }

  // Counts all-to-all ("one extra all-to-all for sizes", PAPER §4.3): my kept counts per global expert
  // (device int32 [N]) -> counts received for my E local experts from every rank (device int32 [P x E]).
  // Then both are copied to the host (pinned) and the stream is synchronised; build the plan.
  void exchange_counts(const int* my_counts, int* recv_counts, int N, cudaStream_t s);

  // Receiver layout: local expert e gets, in ascending source-rank order, recv[src][e] rows padded to 16
  // (the reference bucket order: process, then token).  Host arrays, valid after exchange_counts.
  const std::vector<int>& seg_start() const { return seg_start_; }
  const std::vector<int>& seg_rows() const { return seg_rows_; }
  const std::vector<int>& seg_real() const { return seg_real_; }
  const std::vector<long long>& send_counts() const { return send_cnt_; }
  const std::vector<long long>& recv_counts() const { return recv_cnt_; }
  int recv_rows() const { return recv_rows_; }

  // send layout (packed, expert-major rows of width w) -> receiver layout (padded segments)
  void dispatch(const __nv_bfloat16* send, __nv_bfloat16* recv, int w, cudaStream_t s);
  // receiver layout -> send layout (reverse of dispatch)
  void combine(const __nv_bfloat16* recv, __nv_bfloat16* send, int w, cudaStream_t s);

  // bytes sent to other ranks by the last dispatch / combine (all-to-all bus accounting)
  long long last_offrank_bytes() const { return last_bytes_; }

 private:
  void plan(int N);
  int world_, rank_, E_ = 0;
  ncclComm_t comm_ = nullptr;
  int* h_counts_ = nullptr;  // pinned: [N] mine, then [P x E] received
  std::vector<long long> send_cnt_, send_off_, recv_cnt_, recv_off_;
  std::vector<int> seg_start_, seg_rows_, seg_real_;
  int recv_rows_ = 0;
  long long last_bytes_ = 0;
};

// Host-side plan (also used by the CPU tests): given recv[src][e] (P x E), the padded receiver
// segments and the row offset of every (src, e) block.
void ep_plan(int P, int E, const long long* recv, int* seg_start, int* seg_rows, long long* recv_off);

}  // namespace tamoe
