#include "ep.hpp"

#include <unistd.h>

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

EpComm::EpComm(int world, int rank) : world_(world), rank_(rank) {
  require(world >= 1 && world <= kMaxRanks && rank >= 0 && rank < world, "bad expert-parallel world / rank");
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
  require(comm_ != nullptr, "NCCL barriers need the NCCL bootstrap (tamoe_layer_create_ep)");
  TAMOE_NCCL(ncclAllGather(my_counts, all_counts, N, ncclInt32, comm_, s));
}

void EpComm::barrier(int* flag, cudaStream_t s) {
  require(comm_ != nullptr, "NCCL barriers need the NCCL bootstrap (tamoe_layer_create_ep)");
  TAMOE_NCCL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, comm_, s));
}

void EpComm::allreduce_sum(double* buf, size_t n, cudaStream_t s) {
  require(comm_ != nullptr, "NCCL all-reduce needs the NCCL bootstrap");
  TAMOE_NCCL(ncclAllReduce(buf, buf, n, ncclFloat64, ncclSum, comm_, s));
}

PeerBlob EpComm::make_blob(void* local_base, long long bytes, unsigned long long fingerprint) const {
  PeerBlob b;
  std::memset(&b, 0, sizeof(b));
  TAMOE_CUDA(cudaIpcGetMemHandle(&b.handle, local_base));
  b.bytes = bytes;
  b.fingerprint = fingerprint;
  b.world = world_;
  b.rank = rank_;
  b.pid = static_cast<int>(getpid());
  TAMOE_CUDA(cudaGetDevice(&b.device));
  return b;
}

std::vector<PeerBlob> EpComm::allgather_blobs(const PeerBlob& mine) {
  require(comm_ != nullptr, "blob all-gather needs the NCCL bootstrap");
  const size_t hs = sizeof(PeerBlob);
  char* d_buf = nullptr;
  TAMOE_CUDA(cudaMalloc(&d_buf, hs * (world_ + 1)));
  TAMOE_CUDA(cudaMemcpy(d_buf + hs * world_, &mine, hs, cudaMemcpyHostToDevice));
  TAMOE_NCCL(ncclAllGather(d_buf + hs * world_, d_buf, hs, ncclChar, comm_, nullptr));
  TAMOE_CUDA(cudaStreamSynchronize(nullptr));
  std::vector<PeerBlob> all(world_);
  TAMOE_CUDA(cudaMemcpy(all.data(), d_buf, hs * world_, cudaMemcpyDeviceToHost));
  TAMOE_CUDA(cudaFree(d_buf));
  return all;
}

void EpComm::open_peers(const PeerBlob* all, void* local_base, std::vector<char*>& bases) {
  require(opened_.empty(), "expert-parallel peers are already mapped");
  const PeerBlob& me = all[rank_];
  for (int j = 0; j < world_; ++j) {
    const PeerBlob& b = all[j];
    require(b.world == world_ && b.rank == j,
            "expert-parallel bootstrap: blob " + std::to_string(j) + " is not rank " + std::to_string(j) + " of " +
                std::to_string(world_));
    require(b.bytes == me.bytes && b.fingerprint == me.fingerprint,
            "expert-parallel bootstrap: rank " + std::to_string(j) +
                " was created with a different configuration / workspace layout than rank " +
                std::to_string(rank_));
  }
  bases.assign(world_, nullptr);
  for (int j = 0; j < world_; ++j) {
    if (j == rank_) {
      bases[j] = static_cast<char*>(local_base);
    } else {
      void* p = nullptr;
      TAMOE_CUDA(cudaIpcOpenMemHandle(&p, all[j].handle, cudaIpcMemLazyEnablePeerAccess));
      opened_.push_back(p);
      bases[j] = static_cast<char*>(p);
    }
  }
}

namespace {
constexpr size_t kProbeSig = 256;  // signal slots [kMaxRanks] + epoch at the head of the probe buffer
}

P2PProbe::P2PProbe(std::unique_ptr<EpComm> comm, size_t max_bytes) : comm_(std::move(comm)), max_bytes_(max_bytes) {
  require(max_bytes >= 16, "p2p probe buffer too small");
  TAMOE_CUDA(cudaMalloc(&buf_, kProbeSig + 2 * max_bytes_));
  TAMOE_CUDA(cudaMemset(buf_, 0, kProbeSig));
  TAMOE_CUDA(cudaMemset(buf_ + kProbeSig, 1, 2 * max_bytes_));
  TAMOE_CUDA(cudaDeviceSynchronize());  // slots zeroed before any peer can see the handle
  TAMOE_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  if (comm_->has_nccl()) {
    const std::vector<PeerBlob> all = comm_->allgather_blobs(blob());
    connect(all.data());
  }
}

PeerBlob P2PProbe::blob() const {
  return comm_->make_blob(buf_, static_cast<long long>(kProbeSig + 2 * max_bytes_), 0x70327050726f6265ull);
}

void P2PProbe::connect(const PeerBlob* all) {
  comm_->open_peers(all, buf_, bases_);
  sig_.P = comm_->world();
  sig_.me = comm_->rank();
  sig_.N = 0;
  sig_.my_counts = nullptr;
  sig_.epoch = reinterpret_cast<unsigned int*>(buf_ + sizeof(unsigned int) * kMaxRanks);
  for (int j = 0; j < sig_.P; ++j) sig_.sig[j] = reinterpret_cast<unsigned int*>(bases_[static_cast<size_t>(j)]);
  connected_ = true;
}

void P2PProbe::barrier(bool soft) {
  EpSignal a = sig_;
  a.soft = soft ? 1 : 0;
  ep_signal_barrier(a, stream_);
}

P2PProbe::~P2PProbe() {
  // nobody unmaps or frees before every rank finished its last transfer
  if (connected_ && stream_) {
    try {
      barrier(true);
      cudaStreamSynchronize(stream_);
    } catch (...) {
    }
  }
  comm_->close_peers();
  if (stream_) cudaStreamDestroy(stream_);
  if (buf_) cudaFree(buf_);
}

std::vector<double> P2PProbe::sweep(const double* sizes_mb, int nsizes, int reps, int warmup) {
  require(connected_, "p2p sweep: peers not connected (tamoe_p2p_probe_connect)");
  const int W = comm_->world(), me = comm_->rank();
  require(nsizes >= 1 && reps >= 1 && warmup >= 0, "p2p sweep: bad sizes / reps");
  for (int s = 0; s < nsizes; ++s)
    require(sizes_mb[s] > 0.0 && sizes_mb[s] * 1e6 <= static_cast<double>(max_bytes_),
            "p2p sweep: message size outside the probe buffer");
  std::vector<double> out(static_cast<size_t>(W) * W * nsizes * reps, 0.0);
  cudaEvent_t e0, e1;
  TAMOE_CUDA(cudaEventCreate(&e0));
  TAMOE_CUDA(cudaEventCreate(&e1));
  char* src_buf = buf_ + kProbeSig;
  for (int src = 0; src < W; ++src)
    for (int dst = 0; dst < W; ++dst)
      for (int si = 0; si < nsizes; ++si) {
        const size_t bytes = (static_cast<size_t>(sizes_mb[si] * 1e6) + 15) & ~static_cast<size_t>(15);
        for (int r = -warmup; r < reps; ++r) {
          barrier();  // everybody idle, previous transfer done
          if (me == src) {
            TAMOE_CUDA(cudaEventRecord(e0, stream_));
            p2p_copy(bases_[static_cast<size_t>(dst)] + kProbeSig + max_bytes_, src_buf, bytes, stream_,
                     link_emulation().factor(src, dst));
            TAMOE_CUDA(cudaEventRecord(e1, stream_));
            TAMOE_CUDA(cudaEventSynchronize(e1));
            float ms = 0.f;
            TAMOE_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (r >= 0) out[((static_cast<size_t>(src) * W + dst) * nsizes + si) * reps + r] = ms * 1e3;
          }
        }
      }
  barrier();
  TAMOE_CUDA(cudaStreamSynchronize(stream_));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (comm_->has_nccl()) {
    // every entry was written by exactly one rank: a sum all-reduce gathers them
    double* d = nullptr;
    TAMOE_CUDA(cudaMalloc(&d, sizeof(double) * out.size()));
    TAMOE_CUDA(cudaMemcpy(d, out.data(), sizeof(double) * out.size(), cudaMemcpyHostToDevice));
    comm_->allreduce_sum(d, out.size(), stream_);
    TAMOE_CUDA(cudaStreamSynchronize(stream_));
    TAMOE_CUDA(cudaMemcpy(out.data(), d, sizeof(double) * out.size(), cudaMemcpyDeviceToHost));
    cudaFree(d);
  }
  return out;
}

}  // namespace tamoe
