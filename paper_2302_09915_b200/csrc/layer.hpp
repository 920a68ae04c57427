// TA-MoE layer: one object per (rank, device).  Owns the routing state and all
// activation workspaces; weights, gradients and inputs are caller-owned.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include <memory>

#include "ep.hpp"
#include "gate_bwd.hpp"
#include "route.hpp"

namespace tamoe {

// Device arena: pointers are registered first, then one cudaMalloc backs them all
// (256-byte aligned slices) and the registered pointers are patched in commit().
class Arena {
 public:
  ~Arena();
  template <class T>
  void reserve(T*& ptr, long long count) {
    const long long off = (size_ + 255) & ~255ll;
    size_ = off + (count > 0 ? count : 1) * static_cast<long long>(sizeof(T));
    slots_.push_back({reinterpret_cast<void**>(&ptr), off});
  }
  void commit();
  long long bytes() const { return size_; }
  char* base() const { return base_; }

 private:
  struct Slot {
    void** ptr;
    long long off;
  };
  char* base_ = nullptr;
  long long size_ = 0;
  std::vector<Slot> slots_;
};

// Routing workspace (device) for P processes x S tokens, N experts, top-k.
struct RouteWorkspace {
  RouteDims dims{};
  RouteBuffers buf{};
  int* caps = nullptr;  // [P*N] int32
  void reserve(Arena& a, int P, int S, int N, int k, bool with_gate64 = false);
  void upload_caps(const long long* caps_host, cudaStream_t s);
  // gate outputs view of the workspace
  RowRouteOut row_out(float* logits, double* probs, int* bad_host = nullptr) const {
    return RowRouteOut{buf.idx, buf.gate, buf.score, buf.hist4, buf.msum4, logits, probs, buf.bad, buf.gate64, bad_host};
  }
  void finish(int mode, cudaStream_t s) const;  // bucket + capacity
};

// Standalone router (the reference's topk_route / gate_forward operator API on device).
struct Router {
  Arena arena;
  RouteWorkspace rw;
  Router(int P, int S, int N, int k);
};

struct LayerConfig {
  int P, S, d, d_out, N, k, f, act;
  int cap_mode;
  double cf;
  int aux_kind;
  double aux_weight;
  int penalty_norm;
  double temperature;
  int need_dx;
  int world_size, rank;
};

struct LayerIO {
  const __nv_bfloat16* x;
  const __nv_bfloat16* y;
  const __nv_bfloat16* wg;
  const __nv_bfloat16* w1;
  const __nv_bfloat16* w2;
  float* dwg;
  __nv_bfloat16* dw1;
  __nv_bfloat16* dw2;
  __nv_bfloat16* dx;
  __nv_bfloat16* y_hat;
  double* losses;
};

// Per-launch timing of the step: CUDA events recorded on the step's stream with no
// host synchronisation inside the step; folded into per-launch totals on read.
struct PhaseTimer {
  static constexpr int kMax = 24;
  bool enabled = false;
  int n = 0;  // launch slots in a step
  const char* names[kMax] = {};
  double total_ms[kMax] = {};
  int steps = 0;
  std::vector<std::vector<cudaEvent_t>> pending;  // one event set per step not yet folded
  std::vector<std::vector<cudaEvent_t>> pool;
  std::vector<cudaEvent_t>* cur = nullptr;
  void begin(cudaStream_t s);
  void mark(const char* name, cudaStream_t s);
  void end(cudaStream_t s);
  void fold();  // synchronises on the recorded events
  void reset();
  ~PhaseTimer();
};

class Layer {
 public:
  // ep == nullptr: all N experts on this device (cfg.world_size must be 1).  Otherwise expert parallel:
  // this rank owns experts [rank*E, (rank+1)*E), E = N / world_size, one logical process per rank.
  Layer(const LayerConfig& cfg, const double* c_hat, std::unique_ptr<EpComm> ep = nullptr);
  ~Layer();
  // off-rank payload bytes of the last step: dispatch stores, combine loads, dO stores, dX loads
  void a2a_bytes(long long* out4);
  void step(const LayerIO& io, cudaStream_t s);
  // Auxiliary-loss kind of the following steps (train()'s topo -> balance switch, trainer.cpp:254-256);
  // the routing keeps the c_hat it was created with.  Drops the captured step graphs.
  void set_aux_kind(int kind);
  EpComm* ep() { return ep_.get(); }
  const LayerConfig& cfg() const { return cfg_; }
  RouteWorkspace& route() { return rw_; }
  int n_pad() const { return n_pad_; }
  int r_max() const { return r_max_; }
  const float* logits() const { return logits_; }
  PhaseTimer& timer() { return timer_; }
  int launches_per_step() const;
  // Non-finite gate logits (the reference throws ValidationError, gate.cpp:16-17) are detected on the
  // device without a host synchronisation inside the step: the flag is copied into pinned host memory at
  // the end of every step and reported (ValidationError) by the next step() once that step has completed,
  // or at once by status(), which waits for the last step.
  void status();
  // expert parallelism with the external bootstrap: this rank's 128-byte blob, then every rank's blobs
  PeerBlob blob() const;
  void connect(const PeerBlob* all);
  bool connected() const { return connected_; }
  // Expert parallelism, outside the step: every rank's n doubles (host) -> all ranks' [world x n] (host, rank
  // order), through peer stores into the mapped workspaces and one device barrier (train()'s per-step report).
  // n <= gather_cap().  Synchronises the stream.
  void allgather_host(const double* mine, int n, double* all, cudaStream_t s);
  int gather_cap() const { return gather_cap_; }

 private:
  void step_local(const LayerIO& io, cudaStream_t s);
  void step_ep(const LayerIO& io, cudaStream_t s);
  void experts_forward(const LayerIO& io, int G, int E, int nsub, const int* seg_start, const int* seg_rows, int rows,
                       cudaStream_t s);
  void experts_backward(const LayerIO& io, int G, int E, int nsub, const int* seg_start, const int* seg_rows, int rows,
                        cudaStream_t s);
  void gate_backward(const LayerIO& io, cudaStream_t s);  // dz + dWg (local inputs only)
  GateDzArgs dz_args(const LayerIO& io) const;
  void gate_backward_dx(const LayerIO& io, cudaStream_t s);  // dX (needs the expert-path gradients)
  void combine(const LayerIO& io, cudaStream_t s);
  PeerBufs peers(__nv_bfloat16* local) const;

  LayerConfig cfg_;
  Arena arena_;
  RouteWorkspace rw_;
  // expert-parallel global capacity (gate.cpp:157-164 across ranks): every rank's picks gathered into a
  // W-process view (peer stores), the global select run on it redundantly, this rank's flags applied locally
  bool global_ep_ = false;
  RouteWorkspace gw_;
  PeerWords gw_idx_{}, gw_score_{}, gw_hist_{};
  std::unique_ptr<EpComm> ep_;
  // expert parallelism: device plan, peer-mapped arena bases, row map
  EpPlanDev plan_{};
  EpSignal sig_{};
  // return codes of this rank's receive rows (written by the permute of the rows' home ranks) and their
  // peer views; expert outputs / input gradients are stored back at row token * k + slot of the home
  int* ret_code_ = nullptr;
  PeerInts ret_codes_{};
  int trash_row_ = 0;                   // device barrier (counts publish + phase barriers)
  unsigned int* sig_slots_ = nullptr;  // [kMaxRanks] in the peer-mapped arena
  unsigned int* sig_epoch_ = nullptr;
  void ep_barrier(cudaStream_t s, bool publish_counts);
  std::vector<char*> bases_;
  RowMap map_{};
  int link_rep_[kMaxRanks] = {};  // emulated link throttle per destination rank (LinkEmulation at creation)
  int r_local_ = 0;  // rows of this rank's own padded layout
  int n_pad_ = 0, n64_ = 0, r_max_ = 0, dw_splits_ = 1, P_global_ = 1;
  // activations (expert order, padded segments)
  // A_ keeps act'(pre-activation) from the forward (all the backward needs of the pre-activation)
  __nv_bfloat16 *xp_ = nullptr, *O_ = nullptr, *dO_ = nullptr, *H_ = nullptr, *A_ = nullptr, *dA_ = nullptr,
                *dxp_ = nullptr, *dz_ = nullptr;
  float *logits_ = nullptr, *dldg_ = nullptr, *dw_part_ = nullptr;
  int* chain_ready_ = nullptr;  // chained FFN GEMMs' readiness counters (null: separate launches)
  double *penalties_ = nullptr, *loss_part_ = nullptr;
  int n_loss_part_ = 0;
  bool topo_ready_ = false;
  // compulsory-quota routing (aux_kind 2): quotas [P x N], fp64 probabilities [P*S x N], sort workspace
  int* quota_ = nullptr;
  double* probs_ = nullptr;
  char* comp_ws_ = nullptr;
  size_t comp_ws_bytes_ = 0;  // penalties p = Norm(1/c_hat) computed at creation (created with the topo loss)
  PhaseTimer timer_;
  bool connected_ = false, stepped_ = false;
  double* gather_buf_ = nullptr;  // [world x gather_cap_] (peer-mapped)
  double* gather_src_ = nullptr;  // [gather_cap_]
  int gather_cap_ = 0;
  PeerWords gather_peers_{};
  unsigned long long fingerprint() const;
  void init_topology(const double* c_hat);
  int* bad_host_ = nullptr;            // mapped pinned: set by the router on a non-finite logit
  int* bad_host_dev_ = nullptr;        // its device address
  cudaEvent_t step_done_ = nullptr;    // recorded on the caller's stream after every step
  bool step_pending_ = false;
  void check_deferred(bool wait);
  // CUDA graphs of one step keyed by the step's buffers (LayerIO), a few cached (double-buffered inputs
  // alternate), captured and launched on a private stream joined to the caller's with two events.
  // TAMOE_GRAPHS=0 or phase timing: eager.
  struct StepGraph {
    static constexpr int kCache = 4;
    bool warm = false;
    LayerIO io[kCache]{};
    cudaGraphExec_t exec[kCache] = {};
    unsigned long long used[kCache] = {};
    unsigned long long tick = 0;
    int misses = 0, calls = 0;  // captures vs replays: mostly misses -> buffers change every step -> eager
    bool disabled = false;
    cudaStream_t stream = nullptr;
    cudaEvent_t in = nullptr, out = nullptr;
    ~StepGraph();
  } graph_;
  void run_step(const LayerIO& io, cudaStream_t s);
  void step_graph(const LayerIO& io, cudaStream_t s);
  void route_front(const LayerIO& io, cudaStream_t s);
};

}  // namespace tamoe
