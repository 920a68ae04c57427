// Expert parallelism over NVLink / NVSwitch: the real exchange the reference only models
// (comm_cost.cpp:24-55).  Rank j owns experts [jE, (j+1)E) (dispatch.hpp:31); rank i sends its
// c_ie kept rows to expert e (dispatch.cpp:21-26).
//
// Data path (no payload goes through NCCL): every rank's workspace arena is mapped into every
// other rank's address space with CUDA IPC, so
//   dispatch  = the permute kernel storing rows straight into the owner's receive layout,
//   combine   = the owner's fwd2 epilogue storing expert outputs straight into the source's local layout,
//               then the combine kernel reading them locally and storing dO into the owner,
//   dX return = the owner's dgrad1 epilogue storing the expert-path gradients into the source.
// NCCL carries only the counts all-gather (the paper's "extra all-to-all for sizes") and
// stream-ordered barriers between the phases.  Offsets are computed on the device, so a step has
// no host synchronisation.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <memory>
#include <vector>

#include "route.hpp"

namespace tamoe {

// Per-step device plan, identical on all ranks up to the `me` perspective.  Receive layout of a rank:
// expert-major; expert e_l holds one 16-row-padded segment per source rank (in rank order), so every
// local expert is one contiguous GEMM group whose rows follow the reference order (process, token).
struct EpPlanDev {
  int* all_counts = nullptr;  // [P x N] kept counts of every rank (all-gather)
  int* seg_start = nullptr;   // [E] receive segment of each local expert
  int* seg_rows = nullptr;    // [E]
  int* dst_off = nullptr;     // [N] where this rank's rows for global expert e start at the owner
  int* recv_rows = nullptr;   // [1]
  int* flag = nullptr;        // [1] NCCL barrier scratch (TAMOE_NCCL_BARRIER=1)
  int* push_row = nullptr;    // [rows] receive row -> (source rank << 27 | row in the source's local layout)
};

void ep_plan_device(const EpPlanDev& plan, int P, int E, int me, cudaStream_t s);

// Device-side barrier over the peer-mapped workspaces (no NCCL on the step path): every rank stores a
// monotonically increasing epoch into every rank's signal slot `me` (st.release.sys) and spins on its own
// slots (ld.acquire.sys) until all peers reached the same epoch.  With `my_counts` it first stores this
// rank's kept counts into row `me` of every rank's all_counts -- the counts all-gather folded into the
// barrier.  A peer that never arrives traps the kernel after 20 s instead of hanging the GPU.
struct EpSignal {
  unsigned int* sig[kMaxRanks];  // every rank's signal slots [kMaxRanks]
  unsigned int* epoch;           // this rank's barrier counter
  int* counts_dst[kMaxRanks];    // every rank's all_counts [P x N]
  const int* my_counts;          // null: plain barrier
  int P, me, N;
  // teardown barrier: give up after ~5 s instead of trapping (a peer that exits without destroying its
  // layer must not kill this rank's context)
  int soft = 0;
};
void ep_signal_barrier(const EpSignal& a, cudaStream_t s);

// Store `words` 32-bit words from src into every rank's copy at dst[r] + word offset (NVLink peer stores):
// the expert-parallel global capacity gathers every rank's picks this way.
struct PeerWords {
  unsigned int* p[kMaxRanks];
};
void peer_broadcast_words(const PeerWords& dst, long long dst_off_words, const void* src, long long words, int P,
                          cudaStream_t s);

// What one rank publishes so the others can map its workspace: the CUDA IPC handle of the allocation plus a
// fingerprint of the layout (bytes, configuration hash) that every rank must agree on -- every peer pointer
// is this rank's offset applied to the peer's base, so a mismatching peer would be written out of bounds.
struct PeerBlob {
  cudaIpcMemHandle_t handle;    // 64 bytes
  long long bytes;              // size of the mapped allocation
  unsigned long long fingerprint;
  int world, rank, pid, device;
  char pad[128 - 64 - 16 - 16];
};
static_assert(sizeof(PeerBlob) == 128, "PeerBlob is the 128-byte tamoe_ep_blob");

// Communicator of the expert-parallel ranks.  Two bootstraps:
//   * NCCL (one process per GPU): the blobs are all-gathered over NCCL;
//   * external (no NCCL, ranks may share a device): the caller exchanges the 128-byte blobs with any transport
//     (a TCP store, MPI, a gloo all-gather) and hands all of them back.
class EpComm {
 public:
  EpComm(int world, int rank, const ncclUniqueId& id);
  EpComm(int world, int rank);  // external bootstrap
  ~EpComm();
  int world() const { return world_; }
  int rank() const { return rank_; }
  bool has_nccl() const { return comm_ != nullptr; }
  PeerBlob make_blob(void* local_base, long long bytes, unsigned long long fingerprint) const;
  // validate every rank's blob against this rank's and map the peers' allocations; bases[j] = rank j's
  void open_peers(const PeerBlob* all, void* local_base, std::vector<char*>& bases);
  std::vector<PeerBlob> allgather_blobs(const PeerBlob& mine);  // NCCL bootstrap only
  // my kept counts [N] -> everybody's [P x N] (stream-ordered; doubles as the step-start barrier)
  void allgather_counts(const int* my_counts, int* all_counts, int N, cudaStream_t s);
  // all ranks' streams reach this point before any proceeds (1-int all-reduce)
  void barrier(int* flag, cudaStream_t s);
  void allreduce_sum(double* buf, size_t n, cudaStream_t s);
  void close_peers();  // unmap every peer allocation opened by open_peers

 private:
  int world_, rank_;
  ncclComm_t comm_ = nullptr;
  std::vector<void*> opened_;
};

// NVLink point-to-point sweep feeding the measured-topology pipeline: every ordered
// pair (src, dst), src == dst included, and every message size is timed `reps` times as one SM-driven peer
// copy -- the mechanism the dispatch uses -- with CUDA events on the source rank while the other ranks idle
// between stream barriers.  Result on every rank: time_us[src][dst][size][rep] (the reference's
// TransferSample rows, profile_io.hpp:8-13; alpha then absorbs the launch latency).
// Phases are separated by the device signal barrier over the mapped buffers; with NCCL the sweep's rows are
// summed over ranks at the end, with the external bootstrap each rank returns the rows it timed (src == rank).
class P2PProbe {
 public:
  P2PProbe(std::unique_ptr<EpComm> comm, size_t max_bytes);  // NCCL comm: maps the peers at once
  ~P2PProbe();
  PeerBlob blob() const;
  void connect(const PeerBlob* all);  // external bootstrap
  std::vector<double> sweep(const double* sizes_mb, int nsizes, int reps, int warmup);

 private:
  void barrier(bool soft = false);
  std::unique_ptr<EpComm> comm_;
  size_t max_bytes_;
  char* buf_ = nullptr;  // [signal slots + epoch (256 B) | src half | dst half]
  std::vector<char*> bases_;
  cudaStream_t stream_ = nullptr;
  EpSignal sig_{};
  bool connected_ = false;
};

void p2p_copy(void* dst, const void* src, size_t bytes, cudaStream_t s, int rep = 1);

// Host reference of the receive plan (CPU-testable): recv[src][e] (P x E) rows -> per local expert the
// segment seg_start/seg_rows [E] and the row where each source's rows for it start, src_off [P x E].
void ep_plan(int P, int E, const long long* recv, int* seg_start, int* seg_rows, long long* src_off);

}  // namespace tamoe
