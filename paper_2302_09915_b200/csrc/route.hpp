// Routing state shared by the gate epilogue, the histogram/scan/capacity/permute
// kernels and the combine / backward kernels.  All buffers are device memory.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace tamoe {

constexpr int kMaxTopK = 8;
constexpr int kMaxRanks = 16;

// Maps a row of this rank's padded expert-major layout to the row it occupies in the owner rank's receive
// layout (expert parallelism over peer memory).  The owner's layout is expert-major too: for each of its
// experts, one 16-row-padded segment per source rank in rank order.  P == 1: identity (everything local).
struct RowMap {
  int P = 1, E = 1;                  // ranks, experts per rank
  const int* local_start = nullptr;  // [N] segment start of expert e in this rank's padded layout
  const int* dst_off = nullptr;      // [N] start of this rank's segment for expert e at the owner
  __device__ __forceinline__ int rank_of(int expert) const { return P == 1 ? 0 : expert / E; }
  __device__ __forceinline__ long long row(int local_row, int expert) const {
    return P == 1 ? local_row : static_cast<long long>(local_row) - local_start[expert] + dst_off[expert];
  }
};

// Return codes: the expert GEMMs store output row y of a rank's receive layout into rank (code >> 27) at row
// (code & (2^27 - 1)) of its pick-ordered buffers (row = token * k + slot; pad rows go to a trash row).
constexpr int kPushRowBits = 27;
struct PeerInts {
  int* p[kMaxRanks];
};

// The same buffer in every rank's address space (peer-mapped over NVLink; p[0] only when P == 1).
// rep[r] > 1: emulated slow link to rank r (set_link_emulation) -- every payload store to r is issued rep[r]
// times, so that link delivers 1/rep of its bandwidth (the extra copies rewrite identical bytes).
struct PeerBufs {
  __nv_bfloat16* p[kMaxRanks];
  unsigned char rep[kMaxRanks];
};

// Heterogeneous-topology emulation (BASELINE C5): ranks r, j in different groups of `group_size` consecutive
// ranks talk over a link throttled by `repeat`.  Process-wide; off by default (group_size 0 / repeat <= 1).
struct LinkEmulation {
  int group_size = 0, repeat = 1;
  int factor(int src, int dst) const {
    return (group_size > 0 && repeat > 1 && src / group_size != dst / group_size) ? repeat : 1;
  }
};
LinkEmulation& link_emulation();

#ifdef __CUDACC__
// The throttle's extra copies: volatile stores, so none is merged with the payload store it repeats.
__device__ __forceinline__ void store_repeat(void* p, const uint4& v, int rep) {
  for (int r = 1; r < rep; ++r)
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
#endif
constexpr int kRouteTile = 128;  // tokens per routing tile (= GEMM M tile), 4 warps of 32

struct RouteDims {
  int P;      // logical processes on this device
  int S;      // tokens per process
  int N;      // experts
  int k;      // experts per token
  int TB;     // 128-token tiles per process = ceil(S / 128)
  __host__ __device__ int tiles() const { return P * TB; }
  __host__ __device__ long long picks() const { return static_cast<long long>(P) * S * k; }
};

struct RouteBuffers {
  // per pick [P*S*k], pick id = token * k + slot (token = proc * S + s)
  int* idx = nullptr;
  float* gate = nullptr;
  double* score = nullptr;
  uint8_t* kept = nullptr;
  int* pos = nullptr;  // row of the pick in the expert-sorted buffer, -1 if dropped
  // per (tile, warp, expert) [tiles*4*N]
  int* hist4 = nullptr;
  double* msum4 = nullptr;
  int* base4 = nullptr;  // exclusive prefix of hist4 per expert (route_scan)
  // expert lists [P*S*k]
  int* list_pick = nullptr;     // pre-capacity, expert-major, (process, token) order inside
  double* list_score = nullptr;
  int* clist = nullptr;         // kept picks compacted at the front of each expert range
  uint8_t* list_keep = nullptr;
  // per expert / bucket
  int* list_start = nullptr;  // [N]
  int* list_count = nullptr;  // [N]
  int* bucket_start = nullptr;  // [P*N] offset inside the expert list
  int* bucket_count = nullptr;  // [P*N]
  int* counts = nullptr;      // [P*N] kept
  int* dropped = nullptr;     // [P*N]
  double* mean_probs = nullptr;  // [P*N]
  int* seg_start = nullptr;   // [N] padded row segment per expert
  int* seg_rows = nullptr;    // [N]
  int* total_rows = nullptr;  // [1]
  int* bad = nullptr;         // [1] non-finite logit flag
  float* logits = nullptr;    // [P*S*N] gate logits scratch (router API without a caller buffer)
  double* gate64 = nullptr;   // [P*S*k] fp64 gate values (standalone router only; the layer uses fp32 gate)
};

// Gate epilogue / standalone router outputs (per-row routing, see gate.cu).
struct RowRouteOut {
  int* idx;
  float* gate;
  double* score;
  int* hist4;
  double* msum4;
  float* logits;  // optional [P*S*N]
  double* probs;  // optional [P*S*N]
  int* bad;
  double* gate64 = nullptr;  // optional [P*S*k] fp64 gate values (reference Assignment::gate_value)
  int* bad_host = nullptr;   // optional: mapped pinned host flag, set to 1 on a non-finite logit
};

// Top-k selection from fp64 probabilities (P x S x N), the reference's topk_route input.
void route_rows_from_probs(const double* probs, const RouteDims& d, const RowRouteOut& o, cudaStream_t s);
// Same per-token routing over fp32 gate logits (softmax in fp64 first), N <= 256.
void route_from_logits(const float* logits, const RouteDims& d, const RowRouteOut& o, cudaStream_t s);

// Compulsory-quota re-routing of top-1 picks (trainer.cpp:121-169): rewrites idx / score / gate from the
// fp64 probabilities [P*S x N] and the per-(process, expert) quotas (device int32 [P*N], rows sum to S),
// rebuilds the 32-token histograms; follow with route_bucket + route_capacity(mode 0).
size_t compulsory_workspace_bytes(int P, int S);
void route_compulsory(const RouteDims& d, const RouteBuffers& b, const double* probs, const int* quota, void* ws,
                      size_t ws_bytes, cudaStream_t s);

// histogram scan + stable bucket lists (gate.cpp:160-164 / 181-185 order)
// direct = no capacity (mode 0): the bucket lists are written as the kept lists (clist, kept, counts, mean
// probabilities) and route_capacity is not needed
void route_bucket(const RouteDims& d, const RouteBuffers& b, cudaStream_t s, bool direct = false);
// capacity enforcement + compaction + counts + mean probs (gate.cpp:115, 138-199)
// caps: device int32 [P*N] (INT32_MAX = unlimited); mode: 0 none, 1 global, 2 local, 3 proportional,
// 4 external (b.kept already holds the keep flag of every pick: the expert-parallel global decision)
void route_capacity(const RouteDims& d, const RouteBuffers& b, int mode, const int* caps, cudaStream_t s);
// padded expert segments + gather of token rows into the expert-sorted buffer.
// x: [P*S x dx] bf16; xp: [R_max x dx]; zero_rows (optional): second buffer whose pad rows are zeroed.
// Gather kept token rows into the padded expert-major layout (16-row segments, pad rows zeroed) and write
// each row to wherever its owner expects it: `map`/`xp` (and the pad rows of `zrows`) may point into peer
// ranks' memory, which fuses the dispatch all-to-all into the permute (NVLink stores).
// codes (optional): for every row it writes, the permute also stores the row's return code into the owner's
// code array (me << 27 | pick, pad rows -> me << 27 | trash_row).
void route_permute(const RouteDims& d, const RouteBuffers& b, const __nv_bfloat16* x, int dx, const PeerBufs& xp,
                   int r_max, const PeerBufs* zrows, int zdim, const RowMap& map, cudaStream_t s,
                   const PeerInts* codes = nullptr, int me = 0, int trash_row = 0);
// Zero rows [seg_start + seg_real, seg_start + seg_rows) of each of G segments in buffers a and b.
void zero_pad_rows(const int* seg_start, const int* seg_rows, const int* seg_real, int G, __nv_bfloat16* a, int wa,
                   __nv_bfloat16* b, int wb, cudaStream_t s);

}  // namespace tamoe
