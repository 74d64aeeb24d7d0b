// comm.cu — the two collectives the kernel split creates, over NCCL on NVLink/NVSwitch.
//
//  * forward: channel AllGather of the per-rank output blocks (the paper's gather +
//    "reshapes and rearranges", Alg. 1 L19-22).  Because the gather
//    layout stores each rank's channels as one contiguous block in rank order, equal
//    block widths make this ONE in-place ncclAllGather; unequal widths (Eq. 1 maps) are a
//    grouped set of ncclBroadcast calls, one per root (allgather-v).
//  * backward: sum of the per-rank partial dX (north_star) as in-place ncclAllReduce, or
//    ncclReduceScatter delivering each rank exactly its own input block (grouped
//    ncclReduce per root for unequal widths).
#include <nccl.h>

#include <string>
#include <vector>

#include "kernels.cuh"

struct cp_comm_s {
  ncclComm_t comm;
  int rank, world;
};

#define CP_NCCL(call)                                                                      \
  do {                                                                                     \
    ncclResult_t r__ = (call);                                                             \
    if (r__ != ncclSuccess) {                                                              \
      ::cp::set_error(std::string(#call) + ": " + ncclGetErrorString(r__));               \
      return CP_ERR_NCCL;                                                                  \
    }                                                                                      \
  } while (0)

extern "C" int cp_comm_unique_id(uint8_t id_out[128]) {
  if (!id_out) CP_FAIL(CP_ERR_ARG, "cp_comm_unique_id: null pointer");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId must be 128 bytes");
  ncclUniqueId id;
  CP_NCCL(ncclGetUniqueId(&id));
  memcpy(id_out, &id, 128);
  return CP_OK;
}

extern "C" int cp_comm_create(const uint8_t id[128], int32_t rank, int32_t world, cp_comm* out) {
  if (!id || !out) CP_FAIL(CP_ERR_ARG, "cp_comm_create: null pointer");
  if (world < 1 || world > CP_MAX_RANKS || rank < 0 || rank >= world)
    CP_FAIL(CP_ERR_CONFIG, "cp_comm_create: bad rank/world " + std::to_string(rank) + "/" + std::to_string(world));
  ncclUniqueId uid;
  memcpy(&uid, id, 128);
  auto* c = new cp_comm_s{};
  c->rank = rank;
  c->world = world;
  ncclResult_t r = ncclCommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    CP_FAIL(CP_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  *out = c;
  return CP_OK;
}

extern "C" int cp_comm_destroy(cp_comm c) {
  if (!c) return CP_OK;
  ncclResult_t r = ncclCommDestroy(c->comm);
  delete c;
  if (r != ncclSuccess) CP_FAIL(CP_ERR_NCCL, std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
  return CP_OK;
}

extern "C" int cp_allreduce_sum(cp_comm c, float* buf, int64_t n, void* stream) {
  if (!c || c->world == 1 || n == 0) return CP_OK;
  if (!buf || n < 0) CP_FAIL(CP_ERR_ARG, "cp_allreduce_sum: bad arguments");
  CP_NCCL(ncclAllReduce(buf, buf, (size_t)n, ncclFloat, ncclSum, c->comm, (cudaStream_t)stream));
  return CP_OK;
}

namespace cp {

static int async_error(cp_comm c) {
  ncclResult_t ar;
  CP_NCCL(ncclCommGetAsyncError(c->comm, &ar));
  if (ar != ncclSuccess) CP_FAIL(CP_ERR_NCCL, std::string("NCCL async error: ") + ncclGetErrorString(ar));
  return CP_OK;
}

// Every rank must hold the same partition maps: compare min and max of a hash.
int comm_check_plan(cp_comm c, const Layer& L) {
  if (!c || c->world == 1) return CP_OK;
  if (c->world != L.d.world || c->rank != L.d.rank)
    CP_FAIL(CP_ERR_CONFIG, "conv_part_create: desc rank/world " + std::to_string(L.d.rank) + "/" +
                               std::to_string(L.d.world) + " vs communicator " + std::to_string(c->rank) +
                               "/" + std::to_string(c->world));
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](int64_t v) { h = (h ^ (uint64_t)v) * 1099511628211ull; };
  const cp_partition* ps[2] = {&L.d.out_part, &L.d.in_part};
  for (int t = 0; t < (L.images ? 1 : 2); ++t) {
    mix(ps[t]->n_ranks);
    mix(ps[t]->num_k);
    for (int r = 0; r < ps[t]->n_ranks; ++r) {
      mix(ps[t]->k_begin[r]);
      mix(ps[t]->k_count[r]);
      mix(ps[t]->k_width[r]);
    }
  }
  mix(L.B); mix(L.C); mix(L.H); mix(L.W); mix(L.K); mix(L.R); mix(L.S); mix(L.d.math);
  // split into two non-negative int64 halves so min/max comparisons are exact
  int64_t host[4] = {(int64_t)(h >> 32), (int64_t)(h & 0xffffffffu), -(int64_t)(h >> 32), -(int64_t)(h & 0xffffffffu)};
  int64_t* dev = nullptr;
  CP_CUDA(cudaMalloc(&dev, sizeof(host)));
  CP_CUDA(cudaMemcpy(dev, host, sizeof(host), cudaMemcpyHostToDevice));
  // max over ranks of (h, -h) == (h, -h) on every rank  <=>  all equal
  ncclResult_t r = ncclAllReduce(dev, dev, 4, ncclInt64, ncclMax, c->comm, 0);
  int64_t got[4];
  cudaError_t e = cudaSuccess;
  if (r == ncclSuccess) e = cudaMemcpy(got, dev, sizeof(got), cudaMemcpyDeviceToHost);
  cudaFree(dev);
  if (r != ncclSuccess) CP_FAIL(CP_ERR_NCCL, std::string("plan check: ") + ncclGetErrorString(r));
  if (e != cudaSuccess) CP_FAIL(CP_ERR_CUDA, std::string("plan check: ") + cudaGetErrorString(e));
  for (int i = 0; i < 4; ++i)
    if (got[i] != host[i]) CP_FAIL(CP_ERR_CONFIG, "conv_part_create: ranks hold different partition maps");
  return CP_OK;
}

static bool equal_widths(const Blocks& g) {
  for (int r = 1; r < g.n; ++r)
    if (g.kw[r] != g.kw[0]) return false;
  return true;
}

int comm_allgather_blocks(cp_comm c, float* buf, const Blocks& g, cudaStream_t s) {
  if (!c || c->world == 1) return CP_OK;
  CP_TRY(async_error(c));
  if (equal_widths(g)) {
    const size_t cnt = (size_t)(g.start[1] - g.start[0]);
    if (cnt == 0) return CP_OK;
    CP_NCCL(ncclAllGather(buf + g.start[c->rank], buf, cnt, ncclFloat, c->comm, s));
    return CP_OK;
  }
  CP_NCCL(ncclGroupStart());
  for (int r = 0; r < g.n; ++r) {
    const size_t cnt = (size_t)(g.start[r + 1] - g.start[r]);
    if (cnt == 0) continue;
    ncclResult_t rr = ncclBroadcast(buf + g.start[r], buf + g.start[r], cnt, ncclFloat, r, c->comm, s);
    if (rr != ncclSuccess) {
      ncclGroupEnd();
      CP_FAIL(CP_ERR_NCCL, std::string("ncclBroadcast: ") + ncclGetErrorString(rr));
    }
  }
  CP_NCCL(ncclGroupEnd());
  return CP_OK;
}

int comm_sum_blocks(cp_comm c, float* buf, const Blocks& g, int dx_mode, cudaStream_t s) {
  if (!c || c->world == 1 || dx_mode == CP_DX_LOCAL) return CP_OK;
  CP_TRY(async_error(c));
  if (dx_mode == CP_DX_ALLREDUCE) {
    CP_NCCL(ncclAllReduce(buf, buf, (size_t)g.start[g.n], ncclFloat, ncclSum, c->comm, s));
    return CP_OK;
  }
  if (equal_widths(g)) {
    const size_t cnt = (size_t)(g.start[1] - g.start[0]);
    if (cnt == 0) return CP_OK;
    CP_NCCL(ncclReduceScatter(buf, buf + g.start[c->rank], cnt, ncclFloat, ncclSum, c->comm, s));
    return CP_OK;
  }
  CP_NCCL(ncclGroupStart());
  for (int r = 0; r < g.n; ++r) {
    const size_t cnt = (size_t)(g.start[r + 1] - g.start[r]);
    if (cnt == 0) continue;
    ncclResult_t rr = ncclReduce(buf + g.start[r], buf + g.start[r], cnt, ncclFloat, ncclSum, r, c->comm, s);
    if (rr != ncclSuccess) {
      ncclGroupEnd();
      CP_FAIL(CP_ERR_NCCL, std::string("ncclReduce: ") + ncclGetErrorString(rr));
    }
  }
  CP_NCCL(ncclGroupEnd());
  return CP_OK;
}

}  // namespace cp
