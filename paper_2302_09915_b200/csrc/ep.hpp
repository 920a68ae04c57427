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

  // Layouts.  Send side = the local padded expert-major layout (route_permute, 16-row segments), so
  // the rows for destination j are one contiguous block.  Receive side = one block per source rank,
  // each holding the source's 16-padded segments of this rank's E experts: segment (src, e) at index
  // src*E + e.  The grouped GEMMs consume these (source, expert) segments directly (w_mod / nsub).
  const std::vector<int>& seg_start() const { return seg_start_; }  // [P*E]
  const std::vector<int>& seg_rows() const { return seg_rows_; }    // [P*E]
  const std::vector<long long>& send_counts() const { return send_cnt_; }
  const std::vector<long long>& recv_counts() const { return recv_cnt_; }
  int recv_rows() const { return recv_rows_; }

  // send layout (padded, expert-major rows of width w) -> receive layout (one NCCL op per peer)
  void dispatch(const __nv_bfloat16* send, __nv_bfloat16* recv, int w, cudaStream_t s);
  // receive layout -> send layout (reverse of dispatch)
  void combine(const __nv_bfloat16* recv, __nv_bfloat16* send, int w, cudaStream_t s);

  // bytes sent to other ranks by the last dispatch / combine (all-to-all bus accounting)
  long long last_offrank_bytes() const { return last_bytes_; }

 private:
  void plan(int N);
  int world_, rank_, E_ = 0;
  ncclComm_t comm_ = nullptr;
  int* h_counts_ = nullptr;  // pinned: [N] mine, then [P x E] received
  std::vector<long long> send_cnt_, recv_cnt_;
  std::vector<long long> send_blk_off_, send_blk_rows_, recv_blk_off_, recv_blk_rows_;
  std::vector<int> seg_start_, seg_rows_;
  int recv_rows_ = 0;
  long long last_bytes_ = 0;
};

// Host-side receive plan (also used by the CPU tests): recv[src][e] (P x E) rows -> (source, expert)
// segments seg_start/seg_rows [P*E] (16-row padded, source-major) and block offsets/rows per source [P].
void ep_plan(int P, int E, const long long* recv, int* seg_start, int* seg_rows, long long* blk_off,
             long long* blk_rows);

}  // namespace tamoe
