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
  for (void* p : opened_) cudaIpcCloseMemHandle(p);
  if (comm_) ncclCommDestroy(comm_);
}

void EpComm::allgather_counts(const int* my_counts, int* all_counts, int N, cudaStream_t s) {
  TAMOE_NCCL(ncclAllGather(my_counts, all_counts, N, ncclInt32, comm_, s));
}

void EpComm::barrier(int* flag, cudaStream_t s) {
  TAMOE_NCCL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclSum, comm_, s));
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

}  // namespace tamoe
