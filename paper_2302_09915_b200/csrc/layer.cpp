// TA-MoE layer step orchestration (trainer.cpp:371-482 on the device):
//   gate (tcgen05) -> bucket -> capacity -> permute -> expert FFN (tcgen05 grouped) ->
//   combine + MSE + dO -> expert dgrad / wgrad (tcgen05 grouped) -> gate backward.
#include "layer.hpp"

#include <algorithm>
#include <climits>
#include <cstring>
#include <vector>

#include "combine.hpp"
#include "common.hpp"
#include "expert.hpp"
#include "gate.hpp"
#include "gate_bwd.hpp"
#include "host_topology.hpp"

namespace tamoe {

// Chained FFN GEMMs (fwd1+fwd2, dgrad2+dgrad1 as one persistent launch each; TAMOE_CHAIN=1).  Off by default: ncu
// shows 12 us less GEMM time per step, but the graph-replayed step is unchanged (1.099-1.109 vs 1.100-1.104 ms,
// same box): the chained launch runs its second GEMM with one pipeline stage less (the first GEMM's epilogue smem)
// and graph replay already hides most of the kernel boundary.
static bool chain_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("TAMOE_CHAIN");
    return v && v[0] == '1';
  }();
  return on;
}

LinkEmulation& link_emulation() {
  static LinkEmulation e;
  return e;
}


Arena::~Arena() {
  if (base_) cudaFree(base_);
}

void Arena::commit() {
  require(base_ == nullptr, "arena committed twice");
  TAMOE_CUDA(cudaMalloc(&base_, static_cast<size_t>(size_ > 0 ? size_ : 256)));
  for (const Slot& s : slots_) *s.ptr = base_ + s.off;
}

void RouteWorkspace::reserve(Arena& a, int P, int S, int N, int k, bool with_gate64) {
  require(P >= 1 && S >= 1, "P and S must be positive");
  require(N >= 1 && N <= 1024, "N must be in [1, 1024]");
  require(k >= 1 && k <= N, "k must be in [1, N]");
  require(k <= kMaxTopK, "device routing supports k <= 8");
  dims = RouteDims{P, S, N, k, (S + kRouteTile - 1) / kRouteTile};
  const long long picks = dims.picks();
  const long long tw = static_cast<long long>(dims.tiles()) * 4 * N;
  a.reserve(buf.idx, picks);
  a.reserve(buf.gate, picks);
  a.reserve(buf.score, picks);
  a.reserve(buf.kept, picks);
  a.reserve(buf.pos, picks);
  a.reserve(buf.hist4, tw);
  a.reserve(buf.msum4, tw);
  a.reserve(buf.base4, tw);
  a.reserve(buf.list_pick, picks);
  a.reserve(buf.list_score, picks);
  a.reserve(buf.clist, picks);
  a.reserve(buf.list_keep, picks);
  a.reserve(buf.list_start, N);
  a.reserve(buf.list_count, N);
  a.reserve(buf.bucket_start, static_cast<long long>(P) * N);
  a.reserve(buf.bucket_count, static_cast<long long>(P) * N);
  a.reserve(buf.counts, static_cast<long long>(P) * N);
  a.reserve(buf.dropped, static_cast<long long>(P) * N);
  a.reserve(buf.mean_probs, static_cast<long long>(P) * N);
  a.reserve(buf.seg_start, N);
  a.reserve(buf.seg_rows, N);
  a.reserve(buf.total_rows, 1);
  a.reserve(buf.bad, 1);
  a.reserve(buf.logits, static_cast<long long>(P) * S * N);
  a.reserve(caps, static_cast<long long>(P) * N);
  if (with_gate64) a.reserve(buf.gate64, picks);
}

void RouteWorkspace::upload_caps(const long long* caps_host, cudaStream_t s) {
  const int n = dims.P * dims.N;
  std::vector<int> c(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) c[i] = static_cast<int>(std::min<long long>(std::max<long long>(caps_host[i], 0), INT_MAX));
  TAMOE_CUDA(cudaMemcpyAsync(caps, c.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s));
  TAMOE_CUDA(cudaStreamSynchronize(s));  // c is a stack temporary
}

void RouteWorkspace::finish(int mode, cudaStream_t s) const {
  route_bucket(dims, buf, s, mode == 0);
  if (mode != 0) route_capacity(dims, buf, mode, caps, s);
}

Router::Router(int P, int S, int N, int k) {
  rw.reserve(arena, P, S, N, k, /*with_gate64=*/true);
  arena.commit();
}

// ------------------------------------------------------------------------------------ timing
void PhaseTimer::begin(cudaStream_t s) {
  if (!enabled) return;
  std::vector<cudaEvent_t> set;
  if (!pool.empty()) {
    set = std::move(pool.back());
    pool.pop_back();
  } else {
    set.resize(kMax + 1);
    for (auto& e : set) TAMOE_CUDA(cudaEventCreate(&e));
  }
  pending.push_back(std::move(set));
  cur = &pending.back();
  n = 0;
  TAMOE_CUDA(cudaEventRecord((*cur)[0], s));
}

void PhaseTimer::mark(const char* name, cudaStream_t s) {
  if (!enabled || cur == nullptr || n >= kMax) return;
  names[n] = name;
  TAMOE_CUDA(cudaEventRecord((*cur)[++n], s));
}

void PhaseTimer::end(cudaStream_t) {
  cur = nullptr;
  if (enabled && pending.size() >= 64) fold();
}

void PhaseTimer::fold() {
  for (auto& set : pending) {
    TAMOE_CUDA(cudaEventSynchronize(set[n]));
    for (int i = 0; i < n; ++i) {
      float ms = 0.f;
      TAMOE_CUDA(cudaEventElapsedTime(&ms, set[i], set[i + 1]));
      total_ms[i] += ms;
    }
    ++steps;
    pool.push_back(std::move(set));
  }
  pending.clear();
}

void PhaseTimer::reset() {
  fold();
  steps = 0;
  for (double& v : total_ms) v = 0.0;
}

PhaseTimer::~PhaseTimer() {
  for (auto* v : {&pending, &pool})
    for (auto& set : *v)
      for (auto e : set) cudaEventDestroy(e);
}

// ------------------------------------------------------------------------------------ Layer
Layer::Layer(const LayerConfig& c, const double* c_hat, std::unique_ptr<EpComm> ep) : cfg_(c), ep_(std::move(ep)) {
  require(c.world_size >= 1 && c.rank >= 0 && c.rank < c.world_size, "bad world_size / rank");
  require(c.world_size == 1 || ep_ != nullptr, "expert parallelism needs a communicator (tamoe_layer_create_ep)");
  require(c.world_size == 1 || c.P == 1, "expert parallelism runs one logical process per rank (P = 1)");
  require(c.N % c.world_size == 0, "N must be divisible by world_size");
  require(c.d % 256 == 0, "layer: d must be a multiple of 256");
  require(c.d_out % 128 == 0, "layer: d_out must be a multiple of 128");
  require(c.f == 0 || (c.f % 256 == 0), "layer: f must be 0 (linear expert) or a multiple of 256");
  require(c.P == 1 || c.S % 16 == 0, "layer: S must be a multiple of 16 when P > 1 processes share a device");
  require(c.cap_mode >= 0 && c.cap_mode <= 3, "unknown capacity mode");
  require(c.aux_kind >= 0 && c.aux_kind <= 2, "unknown aux loss kind (0 balance, 1 topo, 2 compulsory)");
  require(c.aux_kind != 2 || c.k == 1, "compulsory routing supports top-1 only");
  require(c.N <= 256, "layer: N must be <= 256");
  P_global_ = c.P * c.world_size;
  n_pad_ = (c.N + 15) & ~15;
  n64_ = expert_pad64(c.N);
  const int E = c.N / c.world_size;
  const long long T = static_cast<long long>(c.P) * c.S;
  // receive side: worst case every token of every rank picks this rank's experts
  const long long r_max = static_cast<long long>(c.world_size) * (T * c.k + 16LL * E);
  require(r_max <= INT_MAX, "layer: world_size * (P*S*k + 16*E) rows exceed the int32 row index");
  require(T * c.k < (1LL << 27), "layer: P*S*k must be < 2^27 (row field of the expert-parallel return codes)");
  r_max_ = static_cast<int>(r_max);
  rw_.reserve(arena_, c.P, c.S, c.N, c.k);
  global_ep_ = ep_ != nullptr && c.cap_mode == 1;
  if (global_ep_) gw_.reserve(arena_, c.world_size, c.S, c.N, c.k);
  arena_.reserve(xp_, static_cast<long long>(r_max_) * c.d);
  arena_.reserve(O_, static_cast<long long>(r_max_) * c.d_out);
  arena_.reserve(dO_, static_cast<long long>(r_max_) * c.d_out);
  if (c.f > 0) {
    arena_.reserve(H_, static_cast<long long>(r_max_) * c.f);
    arena_.reserve(A_, static_cast<long long>(r_max_) * c.f);
    arena_.reserve(dA_, static_cast<long long>(r_max_) * c.f);
  }
  if (c.need_dx) arena_.reserve(dxp_, static_cast<long long>(r_max_) * c.d);
  // chained FFN GEMMs (TAMOE_CHAIN=1): readiness counters per (group, token tile)
  if (c.f > 0 && chain_enabled() && c.f % 256 == 0 && c.d % 256 == 0 && c.d_out % 256 == 0)
    arena_.reserve(chain_ready_, static_cast<long long>(c.N) * chain_ready_stride(r_max_));
  r_local_ = static_cast<int>(T * c.k + 16LL * c.N);
  if (ep_) {
    const int W = c.world_size;
    arena_.reserve(plan_.all_counts, static_cast<long long>(W) * c.N);
    arena_.reserve(plan_.seg_start, E);
    arena_.reserve(plan_.seg_rows, E);
    arena_.reserve(plan_.dst_off, c.N);
    arena_.reserve(plan_.recv_rows, 1);
    arena_.reserve(plan_.flag, 1);
    arena_.reserve(plan_.push_row, r_max_);
    arena_.reserve(sig_slots_, kMaxRanks);
    arena_.reserve(sig_epoch_, 1);
    gather_cap_ = 8 + 2 * c.P * c.N;
    arena_.reserve(gather_buf_, static_cast<long long>(W) * gather_cap_);
    arena_.reserve(gather_src_, gather_cap_);
  }
  if (c.aux_kind == 2) {
    arena_.reserve(quota_, static_cast<long long>(c.P) * c.N);
    arena_.reserve(probs_, T * c.N);
    comp_ws_bytes_ = compulsory_workspace_bytes(c.P, c.S);
    arena_.reserve(comp_ws_, static_cast<long long>(comp_ws_bytes_));
  }
  if (!ep_) arena_.reserve(ret_code_, r_max_);
  trash_row_ = static_cast<int>(T * c.k);  // pick-ordered buffers: T*k rows + one trash row (<= r_max)
  require(static_cast<long long>(trash_row_) < r_max_, "layer: receive buffers too small for the return rows");
  arena_.reserve(dz_, T * n64_);
  arena_.reserve(logits_, T * c.N);
  arena_.reserve(dldg_, T * c.k);
  dw_splits_ = gate_dw_splits(c.P, c.S, c.d, n64_);
  arena_.reserve(dw_part_, static_cast<long long>(dw_splits_) * c.P * n64_ * c.d);
  arena_.reserve(penalties_, static_cast<long long>(c.P) * c.N);
  n_loss_part_ = combine_blocks(T);
  arena_.reserve(loss_part_, n_loss_part_);
  arena_.commit();
  TAMOE_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&bad_host_), sizeof(int), cudaHostAllocMapped));
  *bad_host_ = 0;
  TAMOE_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&bad_host_dev_), bad_host_, 0));
  TAMOE_CUDA(cudaEventCreateWithFlags(&step_done_, cudaEventDisableTiming));
  if (!ep_) ret_codes_.p[0] = ret_code_;
  if (ep_) {
    // barrier slots start at zero on every rank before any peer can signal: zeroed (and synchronised)
    // before this rank's handle leaves the process
    TAMOE_CUDA(cudaMemset(sig_slots_, 0, sizeof(unsigned int) * kMaxRanks));
    TAMOE_CUDA(cudaMemset(sig_epoch_, 0, sizeof(unsigned int)));
    if (global_ep_)
      TAMOE_CUDA(cudaMemset(gw_.buf.msum4, 0, sizeof(double) * static_cast<size_t>(gw_.dims.tiles()) * 4 * c.N));
    TAMOE_CUDA(cudaDeviceSynchronize());
    if (ep_->has_nccl()) {
      const std::vector<PeerBlob> all = ep_->allgather_blobs(blob());
      connect(all.data());
    }
  }
  init_topology(c_hat);
}

unsigned long long Layer::fingerprint() const {
  // FNV-1a over everything that shapes the workspace layout (not the rank)
  const LayerConfig& c = cfg_;
  const long long f[] = {c.P, c.S, c.d, c.d_out, c.N, c.k, c.f, c.act, c.cap_mode, c.aux_kind, c.need_dx,
                         c.world_size, static_cast<long long>(c.cf * 1e9), r_max_, dw_splits_};
  unsigned long long h = 1469598103934665603ull;
  for (long long v : f)
    for (int b = 0; b < 8; ++b) {
      h ^= static_cast<unsigned long long>(v >> (8 * b)) & 0xffull;
      h *= 1099511628211ull;
    }
  return h;
}

PeerBlob Layer::blob() const {
  require(ep_ != nullptr, "blob: not an expert-parallel layer");
  return ep_->make_blob(arena_.base(), arena_.bytes(), fingerprint());
}

// Map every rank's workspace (identical layouts: every peer pointer is this rank's offset applied to the
// peer's base) and derive the peer views of the exchange buffers and barrier slots.
void Layer::connect(const PeerBlob* all) {
  const LayerConfig& c = cfg_;
  require(ep_ != nullptr, "connect: not an expert-parallel layer");
  require(!connected_, "connect: peers already mapped");
  const int E = c.N / c.world_size;
  {
    ep_->open_peers(all, arena_.base(), bases_);
    for (int j = 0; j < c.world_size; ++j) link_rep_[j] = link_emulation().factor(c.rank, j);
    sig_.P = c.world_size;
    sig_.me = c.rank;
    sig_.N = c.N;
    sig_.epoch = sig_epoch_;
    const long long soff = reinterpret_cast<char*>(sig_slots_) - arena_.base();
    const long long coff = reinterpret_cast<char*>(plan_.all_counts) - arena_.base();
    for (int j = 0; j < c.world_size; ++j) {
      sig_.sig[j] = reinterpret_cast<unsigned int*>(bases_[j] + soff);
      sig_.counts_dst[j] = reinterpret_cast<int*>(bases_[j] + coff);
    }
    ret_code_ = plan_.push_row;
    {
      const long long roff = reinterpret_cast<char*>(plan_.push_row) - arena_.base();
      for (int j = 0; j < c.world_size; ++j) ret_codes_.p[j] = reinterpret_cast<int*>(bases_[j] + roff);
    }
    if (global_ep_) {
      auto peer_of = [&](const void* local, int j) {
        return reinterpret_cast<unsigned int*>(bases_[j] + (static_cast<const char*>(local) - arena_.base()));
      };
      for (int j = 0; j < c.world_size; ++j) {
        gw_idx_.p[j] = peer_of(gw_.buf.idx, j);
        gw_score_.p[j] = peer_of(gw_.buf.score, j);
        gw_hist_.p[j] = peer_of(gw_.buf.hist4, j);
      }
    }
    map_.P = c.world_size;
    map_.E = E;
    map_.local_start = rw_.buf.seg_start;
    map_.dst_off = plan_.dst_off;
    const long long goff = reinterpret_cast<char*>(gather_buf_) - arena_.base();
    for (int j = 0; j < c.world_size; ++j) gather_peers_.p[j] = reinterpret_cast<unsigned int*>(bases_[j] + goff);
  }
  connected_ = true;
}

void Layer::init_topology(const double* c_hat) {
  const LayerConfig& c = cfg_;
  // host-side, once per topology: penalties p = Norm(1/c_hat) and capacities (gate.cpp:151-180, 222-246)
  std::vector<double> pen(static_cast<size_t>(c.P) * c.N, 1.0 / c.N);
  if (c.aux_kind == 1) {
    require(c_hat != nullptr, "topo loss requires a target pattern (c_hat)");
    topo_ready_ = true;
    for (int i = 0; i < c.P; ++i) {
      auto p = penalty_weights(c_hat + static_cast<size_t>(c.rank * c.P + i) * c.N, c.N, c.penalty_norm,
                               c.temperature);
      std::copy(p.begin(), p.end(), pen.begin() + static_cast<size_t>(i) * c.N);
    }
  }
  TAMOE_CUDA(cudaMemcpy(penalties_, pen.data(), sizeof(double) * pen.size(), cudaMemcpyHostToDevice));
  // the reference withholds c_hat from balance routing (trainer.cpp:250): proportional capacity then throws
  const double* ch = (c.aux_kind == 0) ? nullptr : c_hat;
  auto caps = capacity_caps(c.cap_mode, c.cf, c.k, c.S, c.N, P_global_, ch);
  if (c.aux_kind == 2) {  // quota_i = LRR(c_hat_i / sum(c_hat_i) * S, S)  (trainer.cpp:128-134)
    require(c_hat != nullptr, "compulsory routing requires a target pattern (c_hat)");
    std::vector<int> q(static_cast<size_t>(c.P) * c.N);
    for (int i = 0; i < c.P; ++i) {
      const double* row = c_hat + static_cast<size_t>(c.rank * c.P + i) * c.N;
      double sum = 0.0;
      for (int e = 0; e < c.N; ++e) sum += row[e];
      std::vector<double> share(static_cast<size_t>(c.N));
      for (int e = 0; e < c.N; ++e) share[static_cast<size_t>(e)] = row[e] / sum * static_cast<double>(c.S);
      const auto lrr = largest_remainder_round(share.data(), c.N, c.S);
      for (int e = 0; e < c.N; ++e) q[static_cast<size_t>(i) * c.N + e] = static_cast<int>(lrr[static_cast<size_t>(e)]);
    }
    TAMOE_CUDA(cudaMemcpy(quota_, q.data(), sizeof(int) * q.size(), cudaMemcpyHostToDevice));
  }
  rw_.upload_caps(caps.data() + static_cast<size_t>(c.rank) * c.P * c.N, nullptr);
  if (global_ep_) gw_.upload_caps(caps.data(), nullptr);  // one global cap per expert, every rank's row
}

Layer::~Layer() {
  if (step_done_) {
    cudaEventSynchronize(step_done_);
    cudaEventDestroy(step_done_);
  }
  if (bad_host_) cudaFreeHost(bad_host_);
  if (ep_ && connected_ && stepped_) {
    // nobody unmaps or frees its workspace while a peer may still store into it: a (soft) device barrier,
    // then unmap the peers, then the arena is freed (member destruction)
    try {
      EpSignal a = sig_;
      a.my_counts = nullptr;
      a.soft = 1;
      ep_signal_barrier(a, nullptr);
      cudaStreamSynchronize(nullptr);
    } catch (...) {
    }
  }
  if (ep_) ep_->close_peers();
}

void Layer::check_deferred(bool wait) {
  if (!step_pending_) return;
  if (wait) TAMOE_CUDA(cudaEventSynchronize(step_done_));
  else if (cudaEventQuery(step_done_) != cudaSuccess) {
    (void)cudaGetLastError();  // cudaErrorNotReady is not sticky; clear it
    return;
  }
  step_pending_ = false;
  if (*reinterpret_cast<volatile int*>(bad_host_) != 0) {
    *reinterpret_cast<volatile int*>(bad_host_) = 0;
    throw ValidationError("non-finite gate logit");
  }
}

void Layer::status() { check_deferred(true); }

void Layer::allgather_host(const double* mine, int n, double* all, cudaStream_t s) {
  const int W = cfg_.world_size;
  if (!ep_) {
    std::copy(mine, mine + n, all);
    return;
  }
  require(connected_, "allgather: expert-parallel peers not connected");
  require(n >= 1 && n <= gather_cap_, "allgather: record larger than the gather buffer");
  TAMOE_CUDA(cudaMemcpyAsync(gather_src_, mine, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  peer_broadcast_words(gather_peers_, static_cast<long long>(cfg_.rank) * gather_cap_ * 2, gather_src_, 2LL * n, W,
                       s);
  ep_barrier(s, false);
  for (int r = 0; r < W; ++r)
    TAMOE_CUDA(cudaMemcpyAsync(all + static_cast<size_t>(r) * n, gather_buf_ + static_cast<size_t>(r) * gather_cap_,
                               sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  TAMOE_CUDA(cudaStreamSynchronize(s));
}

PeerBufs Layer::peers(__nv_bfloat16* local) const {
  PeerBufs pb{};
  if (!ep_) {
    pb.p[0] = local;
    return pb;
  }
  const long long off = reinterpret_cast<char*>(local) - arena_.base();
  for (size_t j = 0; j < bases_.size(); ++j) {
    pb.p[j] = reinterpret_cast<__nv_bfloat16*>(bases_[j] + off);
    pb.rep[j] = static_cast<unsigned char>(link_rep_[j]);
  }
  return pb;
}

void Layer::a2a_bytes(long long* out4) {
  for (int i = 0; i < 4; ++i) out4[i] = 0;
  if (!ep_) return;
  const LayerConfig& c = cfg_;
  const int W = c.world_size, E = c.N / W, me = c.rank;
  std::vector<int> all(static_cast<size_t>(W) * c.N);
  TAMOE_CUDA(cudaMemcpy(all.data(), plan_.all_counts, sizeof(int) * all.size(), cudaMemcpyDeviceToHost));
  long long rows_pad = 0, rows = 0;
  for (int e = 0; e < c.N; ++e) {
    if (e / E == me) continue;
    const long long cnt = all[static_cast<size_t>(me) * c.N + e];
    rows += cnt;
    rows_pad += (cnt + 15) / 16 * 16;
  }
  out4[0] = rows_pad * c.d * 2;     // dispatch stores (incl. zero pad rows)
  out4[1] = rows_pad * c.d_out * 2;  // expert outputs returned (owners' fwd2 epilogue stores, incl. pad rows)
  out4[2] = rows * c.d_out * 2;      // dO stores (combine kernel)
  out4[3] = c.need_dx ? rows_pad * c.d * 2 : 0;  // dX returns (owners' dgrad1 epilogue stores)
}

// Segments: G groups; group g uses weight g % E (E = G when nsub == 1).  For wgrad the E experts'
// K ranges are the nsub = G / E sub-segments s*E + e.
void Layer::experts_forward(const LayerIO& io, int G, int E, int /*nsub*/, const int* seg_start, const int* seg_rows,
                            int rows, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  PhaseTimer& tm = timer_;
  const int wm = G == E ? 0 : E;
  // expert outputs go straight back to row token * k + slot of their home rank (peer stores under EP)
  SwapPush push{peers(O_), ret_code_};
  const SwapPush* pp = &push;
  if (c.f == 0) {
    grouped_fwd(xp_, io.w1, G, c.d_out, c.d, rows, seg_start, seg_rows, O_, nullptr, kActNone, s, wm, pp);
    tm.mark("expert_fwd", s);
  } else if (chain_ready_) {  // both FFN GEMMs in one persistent launch
    grouped_ffn_fwd_chain(xp_, io.w1, io.w2, G, c.f, c.d, c.d_out, rows, seg_start, seg_rows, H_, A_, O_, c.act,
                          chain_ready_, s, wm, pp);
    tm.mark("expert_fwd12", s);
  } else {
    grouped_fwd(xp_, io.w1, G, c.f, c.d, rows, seg_start, seg_rows, H_, A_, c.act, s, wm);
    tm.mark("expert_fwd1", s);
    grouped_fwd(H_, io.w2, G, c.d_out, c.f, rows, seg_start, seg_rows, O_, nullptr, kActNone, s, wm, pp);
    tm.mark("expert_fwd2", s);
  }
}

void Layer::experts_backward(const LayerIO& io, int G, int E, int nsub, const int* seg_start, const int* seg_rows,
                             int rows, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  PhaseTimer& tm = timer_;
  const int wm = G == E ? 0 : E;
  // expert-path input gradients go straight back to row token * k + slot of their home rank
  SwapPush push{peers(dxp_), ret_code_};
  const SwapPush* pp = &push;
  if (c.f == 0) {
    grouped_wgrad(dO_, xp_, E, c.d_out, c.d, rows, seg_start, seg_rows, io.dw1, s, nsub);
    tm.mark("expert_wgrad", s);
    if (c.need_dx) {
      grouped_dgrad(dO_, io.w1, G, c.d, c.d_out, rows, seg_start, seg_rows, dxp_, nullptr, kActNone, s, wm, pp);
      tm.mark("expert_dgrad", s);
    }
  } else if (chain_ready_ && c.need_dx) {  // dgrad2 -> dgrad1 in one persistent launch, then the weight gradients
    grouped_ffn_dgrad_chain(dO_, io.w2, io.w1, G, c.f, c.d, c.d_out, rows, seg_start, seg_rows, dA_, A_, dxp_, c.act,
                            chain_ready_, s, wm, pp);
    tm.mark("expert_dgrad21", s);
    grouped_wgrad(dO_, H_, E, c.d_out, c.f, rows, seg_start, seg_rows, io.dw2, s, nsub);
    tm.mark("expert_wgrad2", s);
    grouped_wgrad(dA_, xp_, E, c.f, c.d, rows, seg_start, seg_rows, io.dw1, s, nsub);
    tm.mark("expert_wgrad1", s);
  } else {
    grouped_dgrad(dO_, io.w2, G, c.f, c.d_out, rows, seg_start, seg_rows, dA_, A_, c.act, s, wm);
    tm.mark("expert_dgrad2", s);
    grouped_wgrad(dO_, H_, E, c.d_out, c.f, rows, seg_start, seg_rows, io.dw2, s, nsub);
    tm.mark("expert_wgrad2", s);
    grouped_wgrad(dA_, xp_, E, c.f, c.d, rows, seg_start, seg_rows, io.dw1, s, nsub);
    tm.mark("expert_wgrad1", s);
    if (c.need_dx) {
      grouped_dgrad(dA_, io.w1, G, c.d, c.f, rows, seg_start, seg_rows, dxp_, nullptr, kActNone, s, wm, pp);
      tm.mark("expert_dgrad1", s);
    }
  }
}

Layer::StepGraph::~StepGraph() {
  for (auto e : exec)
    if (e) cudaGraphExecDestroy(e);
  if (in) cudaEventDestroy(in);
  if (out) cudaEventDestroy(out);
  if (stream) cudaStreamDestroy(stream);
}

static bool fused_dz_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("TAMOE_FUSED_DZ");
    return !(v && v[0] == '0');
  }();
  return on;
}

static bool graphs_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("TAMOE_GRAPHS");
    return !(v && v[0] == '0');
  }();
  return on;
}

void Layer::set_aux_kind(int kind) {
  require(kind == 0 || kind == 1, "aux kind must be 0 (balance) or 1 (topo)");
  require(kind == 0 || topo_ready_, "switching to the topo loss needs a layer created with it (penalties)");
  if (kind == cfg_.aux_kind) return;
  cfg_.aux_kind = kind;
  for (auto& e : graph_.exec)
    if (e) {
      TAMOE_CUDA(cudaGraphExecDestroy(e));
      e = nullptr;
    }
}

void Layer::run_step(const LayerIO& io, cudaStream_t s) {
  if (ep_) step_ep(io, s);
  else step_local(io, s);
}

// The first step runs eagerly (one-time kernel attribute setup); later steps replay a captured graph
// of the whole step (17-19 launches, tensor maps baked in), re-captured whenever a buffer pointer changes.
void Layer::step(const LayerIO& io, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  require(io.x && io.y && io.wg && io.w1 && io.dwg && io.dw1 && io.losses, "layer step: missing buffer");
  require(c.f == 0 || (io.w2 && io.dw2), "layer step: FFN experts need w2 / dw2");
  require(!c.need_dx || io.dx, "layer step: need_dx set but dx is null");
  require(!ep_ || connected_, "layer step: expert-parallel peers not connected (tamoe_layer_ep_connect)");
  check_deferred(false);  // a completed earlier step that saw a non-finite logit raises here
  stepped_ = true;
  step_graph(io, s);
  TAMOE_CUDA(cudaEventRecord(step_done_, s));
  step_pending_ = true;
}

void Layer::step_graph(const LayerIO& io, cudaStream_t s) {
  StepGraph& g = graph_;
  if (timer_.enabled || !graphs_enabled() || !g.warm || g.disabled) {
    run_step(io, s);
    g.warm = true;
    return;
  }
  if (!g.stream) {
    TAMOE_CUDA(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
    TAMOE_CUDA(cudaEventCreateWithFlags(&g.in, cudaEventDisableTiming));
    TAMOE_CUDA(cudaEventCreateWithFlags(&g.out, cudaEventDisableTiming));
  }
  TAMOE_CUDA(cudaEventRecord(g.in, s));
  TAMOE_CUDA(cudaStreamWaitEvent(g.stream, g.in, 0));
  int slot = -1;
  for (int i = 0; i < StepGraph::kCache; ++i)
    if (g.exec[i] && std::memcmp(&g.io[i], &io, sizeof(LayerIO)) == 0) slot = i;
  ++g.calls;
  if (slot < 0 && ++g.misses > 8 && 2 * g.misses > g.calls) {
    // the caller hands new buffers nearly every step: capturing costs more than it saves
    g.disabled = true;
    run_step(io, s);
    return;
  }
  if (slot < 0) {
    slot = 0;  // least recently used
    for (int i = 1; i < StepGraph::kCache; ++i)
      if (g.used[i] < g.used[slot]) slot = i;
    if (g.exec[slot]) {
      TAMOE_CUDA(cudaGraphExecDestroy(g.exec[slot]));
      g.exec[slot] = nullptr;
    }
    cudaGraph_t graph = nullptr;
    TAMOE_CUDA(cudaStreamBeginCapture(g.stream, cudaStreamCaptureModeThreadLocal));
    try {
      run_step(io, g.stream);
    } catch (...) {
      cudaStreamEndCapture(g.stream, &graph);
      if (graph) cudaGraphDestroy(graph);
      throw;
    }
    TAMOE_CUDA(cudaStreamEndCapture(g.stream, &graph));
    const cudaError_t e = cudaGraphInstantiate(&g.exec[slot], graph, 0);
    cudaGraphDestroy(graph);
    TAMOE_CUDA(e);
    g.io[slot] = io;
  }
  g.used[slot] = ++g.tick;
  TAMOE_CUDA(cudaGraphLaunch(g.exec[slot], g.stream));
  TAMOE_CUDA(cudaEventRecord(g.out, g.stream));
  TAMOE_CUDA(cudaStreamWaitEvent(s, g.out, 0));
}

// Shared front: gate + histogram/scan + capacity.
void Layer::route_front(const LayerIO& io, cudaStream_t s) {
  RouteWorkspace& rw = rw_;
  PhaseTimer& tm = timer_;
  const RouteBuffers& b = rw.buf;
  const bool compulsory = cfg_.aux_kind == 2;
  TAMOE_CUDA(cudaMemsetAsync(b.bad, 0, sizeof(int), s));
  gate_forward(io.x, io.wg, n_pad_, rw.dims, cfg_.d, rw.row_out(logits_, compulsory ? probs_ : nullptr, bad_host_dev_),
               s);
  tm.mark("gate_fwd", s);
  if (compulsory) {  // quota claims replace the top-k / capacity outcome; every token is kept
    route_compulsory(rw.dims, b, probs_, quota_, comp_ws_, comp_ws_bytes_, s);
    tm.mark("route_compulsory", s);
  }
  const int mode = compulsory ? 0 : cfg_.cap_mode;
  route_bucket(rw.dims, b, s, mode == 0);  // mode 0: kept lists directly, no capacity pass
  tm.mark("route_bucket", s);
  if (global_ep_) {
    // every rank's picks (expert, score) and 32-token histograms -> every rank's global view, then the
    // global select over (score desc, process asc, token asc) on that view and this rank's flags back
    const int W = cfg_.world_size, me = cfg_.rank;
    const long long picks = rw.dims.picks(), hist = static_cast<long long>(rw.dims.tiles()) * 4 * cfg_.N;
    peer_broadcast_words(gw_idx_, me * picks, b.idx, picks, W, s);
    peer_broadcast_words(gw_score_, me * picks * 2, b.score, picks * 2, W, s);
    peer_broadcast_words(gw_hist_, me * hist, b.hist4, hist, W, s);
    ep_barrier(s, false);
    route_bucket(gw_.dims, gw_.buf, s);
    route_capacity(gw_.dims, gw_.buf, 1, gw_.caps, s);
    TAMOE_CUDA(cudaMemcpyAsync(b.kept, gw_.buf.kept + me * picks, static_cast<size_t>(picks), cudaMemcpyDeviceToDevice, s));
    route_capacity(rw.dims, b, 4, rw.caps, s);
    tm.mark("route_capacity_global", s);
    return;
  }
  if (mode != 0) {
    route_capacity(rw.dims, b, mode, rw.caps, s);
    tm.mark("route_capacity", s);
  }
}

void Layer::step_local(const LayerIO& io, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  const RouteBuffers& b = rw_.buf;
  PhaseTimer& tm = timer_;
  tm.begin(s);
  route_front(io, s);
  const PeerBufs zb = peers(dO_);
  route_permute(rw_.dims, b, io.x, c.d, peers(xp_), r_max_, &zb, c.d_out, map_, s, &ret_codes_, 0, trash_row_);
  tm.mark("permute", s);
  experts_forward(io, c.N, c.N, 1, b.seg_start, b.seg_rows, r_max_, s);
  combine(io, s);
  gate_backward(io, s);
  experts_backward(io, c.N, c.N, 1, b.seg_start, b.seg_rows, r_max_, s);
  gate_backward_dx(io, s);
  tm.end(s);
}

// Expert parallel step: NCCL carries only the counts all-gather and barriers; every payload moves over
// NVLink through peer-mapped memory inside the compute kernels.
void Layer::step_ep(const LayerIO& io, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  const RouteBuffers& b = rw_.buf;
  PhaseTimer& tm = timer_;
  const int W = c.world_size, E = c.N / W;
  tm.begin(s);
  route_front(io, s);
  ep_barrier(s, true);  // counts all-gather; also: every rank finished its previous step
  {
    EpPlanDev plan = plan_;
    plan.push_row = nullptr;  // the return codes come from the sources' permute kernels
    ep_plan_device(plan, W, E, c.rank, s);
  }
  tm.mark("a2a_counts", s);
  // fused permute + dispatch: rows (and the owners' zero pad rows of dO) stored straight into the owners
  const PeerBufs zb = peers(dO_);
  route_permute(rw_.dims, b, io.x, c.d, peers(xp_), r_local_, &zb, c.d_out, map_, s, &ret_codes_, c.rank,
                trash_row_);
  ep_barrier(s, false);
  tm.mark("a2a_dispatch", s);
  experts_forward(io, E, E, 1, plan_.seg_start, plan_.seg_rows, r_max_, s);
  ep_barrier(s, false);
  tm.mark("a2a_barrier_fwd", s);
  combine(io, s);  // reads the returned expert outputs, stores dO into the owners
  gate_backward(io, s);  // dz + dWg need only local data: they overlap the dO stores' NVLink drain
  ep_barrier(s, false);
  tm.mark("a2a_barrier_combine", s);
  experts_backward(io, E, E, 1, plan_.seg_start, plan_.seg_rows, r_max_, s);
  if (c.need_dx) {
    ep_barrier(s, false);
    tm.mark("a2a_barrier_bwd", s);
  }
  gate_backward_dx(io, s);  // the expert-path gradients were pushed back by the owners' dgrad1
  tm.end(s);
}

static bool nccl_barrier() {
  static const bool on = [] {
    const char* v = std::getenv("TAMOE_NCCL_BARRIER");
    return v && v[0] == '1';
  }();
  return on;
}

// Phase barrier of the expert-parallel step: device signal slots over NVLink by default,
// NCCL (all-gather of counts / 1-int all-reduce) with TAMOE_NCCL_BARRIER=1.
void Layer::ep_barrier(cudaStream_t s, bool publish_counts) {
  if (nccl_barrier()) {
    if (publish_counts) ep_->allgather_counts(rw_.buf.counts, plan_.all_counts, cfg_.N, s);
    else ep_->barrier(plan_.flag, s);
    return;
  }
  EpSignal a = sig_;
  a.my_counts = publish_counts ? rw_.buf.counts : nullptr;
  ep_signal_barrier(a, s);
}

void Layer::combine(const LayerIO& io, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  const RouteBuffers& b = rw_.buf;
  CombineArgs ca{};
  ca.T = static_cast<long long>(c.P) * c.S;
  ca.k = c.k;
  ca.dout = c.d_out;
  ca.mse_scale = static_cast<float>(2.0 / (static_cast<double>(P_global_) * c.S * c.d_out));
  ca.pos = b.pos;
  ca.idx = b.idx;
  ca.gate = b.gate;
  ca.O = PeerBufs{};
  ca.O.p[0] = O_;  // fwd2 stored the expert outputs at row token * k + slot of this rank (local pointer)
  ca.o_home = 1;
  ca.y = io.y;
  ca.y_hat = io.y_hat;
  ca.dO = peers(dO_);
  ca.map = map_;
  ca.dldg = dldg_;
  ca.loss_part = loss_part_;
  ca.fuse_dz = fused_dz_enabled() ? 1 : 0;
  ca.gz = dz_args(io);
  combine_loss(ca, s);
  timer_.mark("combine_loss", s);
}

GateDzArgs Layer::dz_args(const LayerIO& io) const {
  const LayerConfig& c = cfg_;
  const RouteBuffers& b = rw_.buf;
  GateDzArgs ga{};
  ga.P = c.P;
  ga.S = c.S;
  ga.N = c.N;
  ga.k = c.k;
  ga.n64 = n64_;
  ga.dout = c.d_out;
  ga.P_global = P_global_;
  ga.aux_kind = c.aux_kind == 2 ? 0 : c.aux_kind;  // compulsory trains with the balance loss (trainer.cpp:253)
  ga.aux_weight = c.aux_weight;
  ga.logits = logits_;
  ga.idx = b.idx;
  ga.score = b.score;
  ga.dldg = dldg_;
  ga.counts = b.counts;
  ga.mean_probs = b.mean_probs;
  ga.penalties = penalties_;
  ga.loss_part = loss_part_;
  ga.n_loss_part = n_loss_part_;
  ga.losses = io.losses;
  ga.dz = dz_;
  return ga;
}

void Layer::gate_backward(const LayerIO& io, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  PhaseTimer& tm = timer_;
  const GateDzArgs ga = dz_args(io);
  if (fused_dz_enabled()) {  // dz came from the combine kernel; the gate dW GEMM finalises the losses
    gate_dw(io.x, dz_, c.P, c.S, c.d, n64_, n_pad_, c.N, dw_part_, dw_splits_, io.dwg, s, &ga);
    tm.mark("gate_dw", s);
    return;
  }
  gate_dz(ga, s);
  tm.mark("gate_dz", s);
  gate_dw(io.x, dz_, c.P, c.S, c.d, n64_, n_pad_, c.N, dw_part_, dw_splits_, io.dwg, s);
  tm.mark("gate_dw", s);
}

void Layer::gate_backward_dx(const LayerIO& io, cudaStream_t s) {
  const LayerConfig& c = cfg_;
  const RouteBuffers& b = rw_.buf;
  PhaseTimer& tm = timer_;
  if (c.need_dx) {
    // expert-path gradients are in this rank's layout (pushed back by the owners' dgrad1 in EP)
    PeerBufs home{};
    home.p[0] = dxp_;
    gate_dx(dz_, io.wg, c.P, c.S, c.d, n64_, n_pad_, home, b.pos, b.idx, RowMap{}, c.k, io.dx, s);
    tm.mark("gate_dx", s);
  }
}

int Layer::launches_per_step() const {
  // gate, scan, bucket, capacity, permute, combine, dz, dW GEMM + reduce
  int n = gate_is_fused(cfg_.N, cfg_.aux_kind == 2) ? 9 : 10;  // gate: one fused launch, or logits GEMM + router
  if (!global_ep_ && (cfg_.cap_mode == 0 || cfg_.aux_kind == 2)) n -= 1;  // no capacity pass
  if (fused_dz_enabled()) n -= 1;  // gate dz inside the combine kernel
  // EP: + plan and return-map kernels + the device barriers (counts publish, dispatch, forward, combine, [dX])
  if (ep_) n += 1 + (nccl_barrier() ? 0 : 4 + (cfg_.need_dx ? 1 : 0));  // + the device plan
  if (global_ep_) n += 3 + (nccl_barrier() ? 0 : 1) + 3;  // broadcasts, barrier, global scan/bucket/capacity
  n += cfg_.f == 0 ? (1 + 1 + (cfg_.need_dx ? 1 : 0))
                    : (chain_ready_ ? (1 + 2 + (cfg_.need_dx ? 1 : 1)) : (2 + 3 + (cfg_.need_dx ? 1 : 0)));
  if (cfg_.need_dx) n += 1;
  return n;
}

}  // namespace tamoe
