// layer.cu — the C-ABI entry points of a kernel-partitioned conv layer (convpart.h).
//
// Orchestration of one rank's share of the method (Alg. 1/2) as SPMD:
// every rank is a peer holding the same input and its own contiguous kernel slice; the
// master/slave socket protocol becomes stream-ordered kernels plus NCCL collectives.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace cp {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
std::atomic<int64_t>& launch_counter() {
  static std::atomic<int64_t> c{0};
  return c;
}

static std::string shp(std::initializer_list<int64_t> v) {
  std::string s = "[";
  bool first = true;
  for (auto x : v) {
    s += (first ? "" : ",") + std::to_string(x);
    first = false;
  }
  return s + "]";
}

static int validate_part(const cp_partition& p, const char* what) {
  if (p.n_ranks < 1 || p.n_ranks > CP_MAX_RANKS)
    CP_FAIL(CP_ERR_CONFIG, std::string(what) + ": n_ranks out of [1,16]");
  int b = 0;
  for (int r = 0; r < p.n_ranks; ++r) {
    if (p.k_begin[r] != b || p.k_count[r] < 0 || p.k_width[r] < p.k_count[r] || p.k_width[r] % 8)
      CP_FAIL(CP_ERR_CONFIG, std::string(what) + ": ranges must be contiguous in rank order with widths = "
                                                 "multiples of 8 >= counts");
    b += p.k_count[r];
  }
  if (b != p.num_k) CP_FAIL(CP_ERR_CONFIG, std::string(what) + ": counts do not sum to num_k");
  return CP_OK;
}

static size_t al256(size_t x) { return (x + 255) / 256 * 256; }

static int derive(Layer& L, const cp_conv_desc& d) {
  L.d = d;
  if (d.batch < 1 || d.in_c < 1 || d.in_h < 1 || d.in_w < 1 || d.num_k < 1 || d.k_h < 1 || d.k_w < 1)
    CP_FAIL(CP_ERR_SHAPE, "conv_part_create: nonpositive dimension");
  if (d.in_h < d.k_h || d.in_w < d.k_w)
    CP_FAIL(CP_ERR_SHAPE, "dimension error: input " + shp({d.batch, d.in_c, d.in_h, d.in_w}) + " vs kernels " +
                              shp({d.num_k, d.in_c, d.k_h, d.k_w}));
  if (d.math != CP_MATH_TF32 && d.math != CP_MATH_FP32_SIMT && d.math != CP_MATH_BF16)
    CP_FAIL(CP_ERR_CONFIG, "unknown math mode");
  if (d.input_kind != CP_INPUT_IMAGES && d.input_kind != CP_INPUT_GATHER) CP_FAIL(CP_ERR_CONFIG, "unknown input kind");
  CP_TRY(validate_part(d.out_part, "out_part"));
  if (d.out_part.num_k != d.num_k)
    CP_FAIL(CP_ERR_SHAPE, "out_part.num_k=" + std::to_string(d.out_part.num_k) + " vs num_k=" + std::to_string(d.num_k));
  if (d.world != d.out_part.n_ranks || d.rank < 0 || d.rank >= d.world)
    CP_FAIL(CP_ERR_CONFIG, "rank/world inconsistent with out_part");
  L.images = d.input_kind == CP_INPUT_IMAGES;
  L.B = d.batch;
  L.Bp = roundup(d.batch, 32);
  L.C = d.in_c; L.H = d.in_h; L.W = d.in_w; L.R = d.k_h; L.S = d.k_w;
  L.Ho = L.H - L.R + 1; L.Wo = L.W - L.S + 1;
  if (d.pool && ((L.Ho & 1) || (L.Wo & 1)))
    CP_FAIL(CP_ERR_SHAPE, "dimension error: pooling input " + shp({L.Ho, L.Wo}) + " not divisible by stride 2");
  L.Hp = d.pool ? L.Ho / 2 : L.Ho;
  L.Wp = d.pool ? L.Wo / 2 : L.Wo;
  L.K = d.num_k;
  L.Kr = d.out_part.k_count[d.rank];
  L.Kc = d.out_part.k_width[d.rank];
  L.k0 = d.out_part.k_begin[d.rank];
  if (L.images) {
    L.Kcol = roundup(L.R * L.S * L.C, 8);
    L.Ktot = L.Kcol;
    L.in = Blocks{};
  } else {
    CP_TRY(validate_part(d.in_part, "in_part"));
    if (d.in_part.num_k != d.in_c)
      CP_FAIL(CP_ERR_SHAPE, "in_part.num_k=" + std::to_string(d.in_part.num_k) + " vs in_c=" + std::to_string(d.in_c));
    L.in = make_blocks(d.in_part, L.H, L.W, L.Bp);
    L.Kcol = 0;
    L.Ktot = L.R * L.S * L.in.Cg;
  }
  L.out = make_blocks(d.out_part, L.Hp, L.Wp, L.Bp);
  if (d.math == CP_MATH_BF16) {   // 64-element K-chunks: whole chunks of slots and of images
    if (L.Bp % 64) CP_FAIL(CP_ERR_UNSUPPORTED, "bf16 mode: batch padded to 32 must be a multiple of 64");
    for (int r = 0; r < d.out_part.n_ranks; ++r)
      if (d.out_part.k_width[r] % 64) CP_FAIL(CP_ERR_CONFIG, "bf16 mode: out_part widths must be multiples of 64");
    if (!L.images)
      for (int r = 0; r < d.in_part.n_ranks; ++r)
        if (d.in_part.k_width[r] % 64) CP_FAIL(CP_ERR_CONFIG, "bf16 mode: in_part widths must be multiples of 64");
  }
  if (d.math != CP_MATH_FP32_SIMT) CP_TRY(tc_validate(L));
  // workspace carve-up
  size_t off = 0;
  L.off_xcol = off; L.ws_xcol = L.images ? al256((size_t)L.Ho * L.Wo * L.Bp * L.Kcol * 4) : 0; off += L.ws_xcol;
  L.off_z = off; L.ws_z = d.math == CP_MATH_FP32_SIMT ? al256((size_t)L.Ho * L.Wo * L.Bp * L.Kc * 4) : 0; off += L.ws_z;
  L.off_dy = off; L.ws_dy = al256((size_t)L.Ho * L.Wo * L.Bp * L.Kc * 4); off += L.ws_dy;
  L.off_dbpart = off; L.ws_dbpart = al256((size_t)kBiasSplitMax * std::max(L.Kc, 8) * 4); off += L.ws_dbpart;
  L.off_split = off; L.ws_split = d.math != CP_MATH_FP32_SIMT ? al256(tc_workspace_bytes(L)) : 0; off += L.ws_split;
  L.off_x16 = L.off_w16 = L.off_dy16 = 0;
  if (d.math == CP_MATH_BF16) {
    const int64_t nx = L.images ? (int64_t)L.Ho * L.Wo * L.Bp * L.Kcol : L.in.start[L.in.n];
    L.off_x16 = off; off += al256((size_t)nx * 2 + 256);
    L.off_w16 = off; off += al256((size_t)L.Kr * L.Ktot * 2 + 256);
    L.off_dy16 = off; off += al256((size_t)L.Ho * L.Wo * L.Bp * L.Kc * 2 + 256);
  }
  L.off_stamp = off; off += 256;
  L.off_c1w = off; off += al256(L.images ? c1_wgrad_workspace(L) : 0);
  L.ws_total = off + 256;
  L.dy_ready = 0;
  return CP_OK;
}

static char* WS(void* ws, size_t off) { return (char*)ws + off; }

bool gather_push_in_epilogue() {
  static const bool e = [] {
    const char* v = getenv("CP_GATHER_PUSH");
    return v && std::string(v) == "epilogue";
  }();
  return e;
}

// epilogue backward of this rank's block (shared by backward_data and backward_filter)
static int ensure_dy(Layer& L, const float* dy_g, const uint8_t* saved, const float* y_g, void* ws, cudaStream_t s) {
  if (L.dy_ready && L.dy_key[0] == dy_g && L.dy_key[1] == saved && L.dy_key[2] == y_g) return CP_OK;
  const int64_t o = L.out.start[L.d.rank];
  CP_TRY(launch_unpool(L, dy_g + o, saved, y_g + o, (float*)WS(ws, L.off_dy), (float*)WS(ws, L.off_dbpart),
                       L.d.math == CP_MATH_TF32, s));
  if (L.d.math == CP_MATH_BF16)
    CP_TRY(launch_to_bf16((const float*)WS(ws, L.off_dy), WS(ws, L.off_dy16), (int64_t)L.Ho * L.Wo * L.Bp * L.Kc, s));
  L.dy_ready = 1;
  L.dy_key[0] = dy_g; L.dy_key[1] = saved; L.dy_key[2] = y_g;
  return CP_OK;
}

static int fork_comm(Layer& L, cudaStream_t s, cudaStream_t cs) {
  if (cs == s) return CP_OK;
  CP_CUDA(cudaEventRecord(L.ev_compute, s));
  CP_CUDA(cudaStreamWaitEvent(cs, L.ev_compute, 0));
  return CP_OK;
}
static int join_comm(Layer& L, cudaStream_t s, cudaStream_t cs) {
  if (cs == s) return CP_OK;
  CP_CUDA(cudaEventRecord(L.ev_comm, cs));
  CP_CUDA(cudaStreamWaitEvent(s, L.ev_comm, 0));
  return CP_OK;
}

}  // namespace cp

using namespace cp;

struct cp_layer_s : Layer {};

extern "C" {

const char* cp_last_error(void) { return g_last_error.c_str(); }
int64_t cp_launch_count(void) { return launch_counter().load(); }

int conv_part_create(const cp_conv_desc* desc, cp_comm comm, cp_layer* out) {
  if (!desc || !out) CP_FAIL(CP_ERR_ARG, "conv_part_create: null pointer");
  auto* L = new cp_layer_s();
  int rc = derive(*L, *desc);
  if (rc == CP_OK) {
    L->comm = comm;
    rc = comm_check_plan(comm, *L);
  }
  if (rc == CP_OK && cudaEventCreateWithFlags(&L->ev_compute, cudaEventDisableTiming) != cudaSuccess) {
    set_error("cudaEventCreate failed");
    rc = CP_ERR_CUDA;
  }
  if (rc == CP_OK && cudaEventCreateWithFlags(&L->ev_comm, cudaEventDisableTiming) != cudaSuccess) {
    set_error("cudaEventCreate failed");
    rc = CP_ERR_CUDA;
  }
  if (rc != CP_OK) {
    delete L;
    return rc;
  }
  *out = L;
  return CP_OK;
}

int conv_part_query(cp_layer L, cp_sizes* o) {
  if (!L || !o) CP_FAIL(CP_ERR_ARG, "conv_part_query: null pointer");
  // +256 B read slack on every operand the tensor-core path streams with 32-column atoms
  o->w = (size_t)L->Kr * L->Ktot * 4 + 256;
  o->b = (size_t)L->Kr * 4;
  o->x = (L->images ? (size_t)L->B * L->C * L->H * L->W * 4 : (size_t)L->in.start[L->in.n] * 4) + 256;
  o->y = (size_t)L->out.start[L->out.n] * 4 + 256;
  o->y_block = (size_t)(L->out.start[L->d.rank + 1] - L->out.start[L->d.rank]) * 4;
  o->y_offset = (size_t)L->out.start[L->d.rank] * 4;
  o->saved = L->d.pool ? (size_t)L->Hp * L->Wp * L->Bp * L->Kc : 0;
  o->dx = o->x;
  o->workspace = L->ws_total;
  o->dx_peer = 0;
  if (!L->images) {
    int64_t mb = 0;
    for (int r = 0; r < L->in.n; ++r) mb = std::max(mb, L->in.start[r + 1] - L->in.start[r]);
    o->dx_peer = (size_t)(L->in.start[L->in.n] + (int64_t)L->in.n * mb) * 4 + 256;
  }
  return CP_OK;
}

int conv_part_destroy(cp_layer L) {
  if (!L) return CP_OK;
  tc_release(*L);
  for (int p = 0; p < 5; ++p)
    for (int e = 0; e < 2; ++e)
      if (L->ev_t[p][e]) cudaEventDestroy(L->ev_t[p][e]);
  if (L->ev_compute) cudaEventDestroy(L->ev_compute);
  if (L->ev_comm) cudaEventDestroy(L->ev_comm);
  if (L->ev_bar_fork) cudaEventDestroy(L->ev_bar_fork);
  if (L->ev_bar) cudaEventDestroy(L->ev_bar);
  if (L->ev_gfork) cudaEventDestroy(L->ev_gfork);
  if (L->ev_gjoin) cudaEventDestroy(L->ev_gjoin);
  for (int k = 0; k < CP_MAX_RANKS; ++k)
    if (L->ev_split[k]) cudaEventDestroy(L->ev_split[k]);
  if (L->cs2) cudaStreamDestroy(L->cs2);

  delete L;
  return CP_OK;
}

// gather variant of a tensor-core consumer with a comm stream, read per call: copy engines (default) or
// CP_GATHER_MODE=push (warp 3 of the consuming GEMM pushes the block over NVLink)
static bool gather_on_copy_engines() {
  const char* e = getenv("CP_GATHER_MODE");
  return !(e && strcmp(e, "push") == 0);
}

// fused reduce-scatter variant, read per call (tests switch it between layers): 2 ce (default: the owners'
// copy engines fetch the partials into their receive slots), 1 pull (owners read the partials with SM
// loads), 0 push (the dgrad epilogue stores each partial into its owner's receive slot)
static int rs_mode() {
  const char* e = getenv("CP_RS_MODE");
  if (e && strcmp(e, "pull") == 0) return 1;
  if (e && strcmp(e, "push") == 0) return 0;
  return 2;
}

int conv_part_forward(cp_layer L, const float* x, const float* w, const float* b, float* y, uint8_t* saved,
                      void* ws, void* stream, void* comm_stream) {
  if (!L || !x || !w || !y || !ws) CP_FAIL(CP_ERR_ARG, "conv_part_forward: null pointer");
  if (L->d.bias && !b) CP_FAIL(CP_ERR_ARG, "conv_part_forward: bias enabled but b is null");
  if (L->d.pool && !saved) CP_FAIL(CP_ERR_ARG, "conv_part_forward: pooling needs saved");
  cudaStream_t s = (cudaStream_t)stream, cs = comm_stream ? (cudaStream_t)comm_stream : s;
  L->dy_ready = 0;
  float* yb = y + L->out.start[L->d.rank];
  const bool tf32 = L->d.math == CP_MATH_TF32;
  const float* xin = x;
  // image layer on the tensor cores: the dedicated kernel builds its im2col rows in shared memory
  const bool c1 = L->images && tf32 && c1_fwd_supported(*L) && !gather_push_in_epilogue();
  L->xcol_key = nullptr;
  if (L->images && !c1) {
    float* xcol = (float*)WS(ws, L->off_xcol);
    CP_TRY(launch_im2col(*L, x, xcol, tf32, s));
    L->xcol_key = x;
    xin = xcol;
  }
  // Channel AllGather over NVLink peer memory (B200 path), fused into the consumer
  // GEMM.  Producer side: when y_gathered is a symmetric buffer (cp_symmetric_alloc), a device-side
  // barrier first makes sure no peer still reads its copy (e.g. the next layer's async wgrad of the
  // previous step), then the GEMM writes this rank's block locally.  Consumer side: when x is a
  // symmetric gathered buffer, the forward kernel's otherwise idle warp 3 pushes this rank's block
  // into every peer's copy (full-line NVLink stores, a release-add per chunk on the peer's arrival
  // counter) while the MMA warps consume the own block first and each peer block once its counter
  // is complete - the gather overlaps the GEMM; no AllGather kernel, no NCCL call.  Consumers outside
  // the tensor-core forward use copy-engine copies + flags (comm_ce_distribute / cp_symmetric_wait).
  // CP_GATHER_PUSH=epilogue instead pushes from the producer's epilogue (A/B comparison).
  void* peers[CP_MAX_RANKS];
  uint32_t* pflags[CP_MAX_RANKS];
  float* peer_blocks[CP_MAX_RANKS];
  uint32_t* signal[CP_MAX_RANKS];
  int npeers = 0;
  const int me = L->d.rank;
  const bool epi_push = gather_push_in_epilogue();
  const bool gathered_out = L->comm && L->d.world > 1 && !L->d.local_output;
  const bool sym_out = gathered_out && comm_symmetric_peers(L->comm, y, peers, pflags);
  const bool push_in_epilogue = sym_out && tf32 && epi_push;
  if (sym_out) {
    for (int r = 0; r < L->d.world; ++r)
      if (r != me) {
        signal[npeers] = pflags[r];
        peer_blocks[npeers++] = (float*)peers[r] + L->out.start[me];
      }
    comm_symmetric_set_own(L->comm, y, L->out.start[me], L->out.start[me + 1] - L->out.start[me]);
  }
  void* ipeers[CP_MAX_RANKS];
  uint32_t* iflags[CP_MAX_RANKS];
  const bool sym_in = !L->images && L->comm && L->d.world > 1 && comm_symmetric_peers(L->comm, x, ipeers, iflags);
  const uint32_t* arrive = sym_in ? iflags[me] : nullptr;
  if (sym_in) {   // the producer's deferred barrier: no peer still reads its copy of the previous step
    cudaEvent_t pe = comm_symmetric_take_pending(L->comm, x);
    if (pe) CP_CUDA(cudaStreamWaitEvent(s, pe, 0));
  }
  const bool has_gemm = L->Kr > 0 || L->Kc > 0;
  GatherPush gp{};
  bool kernel_push = false, ce_forked = false;
  if (sym_in && !epi_push) {
    const int64_t n = L->in.start[me + 1] - L->in.start[me];
    if (tf32 && has_gemm && gather_on_copy_engines() && cs != s && !comm_is_loopback(L->comm)) {
      // copy-engine gather (default): the copy engines distribute this rank's block (need order, one
      // flag per peer after its copy) on the comm stream while the GEMM runs and waits for its
      // arrivals; no SM does transfer work.  Nothing queued ahead of the copies on the comm stream
      // waits for a peer (the producer barrier of this layer's own output is enqueued after them)
      if (!L->ev_gfork) {
        CP_CUDA(cudaEventCreateWithFlags(&L->ev_gfork, cudaEventDisableTiming));
        CP_CUDA(cudaEventCreateWithFlags(&L->ev_gjoin, cudaEventDisableTiming));
      }
      CP_CUDA(cudaEventRecord(L->ev_gfork, s));
      CP_CUDA(cudaStreamWaitEvent(cs, L->ev_gfork, 0));
      // CP_GATHER_CE_STREAMS=2: each peer's copy in two halves on two copy engines
      const bool split = tc_env_int("CP_GATHER_CE_STREAMS", 1) >= 2;
      if (split && !L->cs2) {
        CP_CUDA(cudaStreamCreateWithFlags(&L->cs2, cudaStreamNonBlocking));
        for (int k = 0; k < CP_MAX_RANKS; ++k) CP_CUDA(cudaEventCreateWithFlags(&L->ev_split[k], cudaEventDisableTiming));
      }
      if (split) CP_CUDA(cudaStreamWaitEvent(L->cs2, L->ev_gfork, 0));
      CP_TRY(tc_time_mark(*L, 3, 0, cs));   // gather window: first copy issued -> last flag written
      CP_TRY(comm_ce_distribute(L->comm, x, cs, true, split ? L->cs2 : nullptr, L->ev_split));
      CP_TRY(tc_time_mark(*L, 3, 1, cs));
      if (L->timing) L->ce_gather_timed = 1;
      CP_CUDA(cudaEventRecord(L->ev_gjoin, cs));
      ce_forked = true;
    } else if (tf32 && has_gemm) {
      kernel_push = true;
      gp.src = x + L->in.start[me];
      gp.n4 = n / 4;
      gp.chunks = kGatherChunks;
      gp.claim = iflags[me] + kClaimWord;
      if (L->timing) {   // push window: first chunk claimed -> last chunk's arrival released
        gp.stamp = (unsigned long long*)WS(ws, L->off_stamp);
        L->ws_last = ws;
        CP_CUDA(cudaMemsetAsync(gp.stamp, 0xff, 8, s));
        CP_CUDA(cudaMemsetAsync(gp.stamp + 1, 0, 8, s));
      }
      // NVLink multicast (CP_MULTICAST=1): one multimem store per 16 B reaches every rank's copy
      // through the NVSwitch (and rewrites the own block with itself); the arrival counter [me] is
      // raised on every rank by one multimem reduction per chunk
      char* mc = (char*)comm_symmetric_mc(L->comm, x);
      if (mc) {
        gp.mc = 1;
        gp.dst[gp.n] = (float*)mc + L->in.start[me];
        gp.cnt[gp.n++] = (uint32_t*)(mc + ((char*)iflags[me] - (char*)x)) + me;
      }
      // peer q walks its input blocks from its own upwards, so it needs this rank's block after
      // (me - q) mod P blocks: push to the soonest consumer first
      for (int d = 1; d < L->d.world && !mc; ++d) {
        const int q = (me - d + L->d.world) % L->d.world;
        gp.dst[gp.n] = (float*)ipeers[q] + L->in.start[me];
        gp.cnt[gp.n++] = iflags[q] + me;
      }
    } else {
      // (a TF32 rank without kernels here signals the chunk count its peers' GEMMs wait for)
      CP_TRY(comm_ce_distribute(L->comm, x, s, tf32));
    }
  }
  // Producer-side barrier of a gathered output (after the input-side distribution above: the comm
  // stream's copy-engine gather must not queue behind a cross-rank barrier while this rank's GEMM
  // holds every SM spinning on its peers' copies)
  if (sym_out) {
    if (!epi_push && cs != s && !comm_is_loopback(L->comm)) {
      // Nothing but this rank writes its own copy's own block, so only the consumer's distribution
      // (the push into the peers' copies, or their copy-engine copies) must wait for the barrier: it
      // runs on the comm stream, overlapped with this layer's GEMM, and the consumer's forward waits
      // for it (comm_symmetric_take_pending) - rank skew and the barrier latency hide behind conv1.
      if (!L->ev_bar) {
        CP_CUDA(cudaEventCreateWithFlags(&L->ev_bar_fork, cudaEventDisableTiming));
        CP_CUDA(cudaEventCreateWithFlags(&L->ev_bar, cudaEventDisableTiming));
      }
      CP_CUDA(cudaEventRecord(L->ev_bar_fork, s));
      CP_CUDA(cudaStreamWaitEvent(cs, L->ev_bar_fork, 0));
      CP_TRY(comm_barrier(L->comm, cs));
      CP_CUDA(cudaEventRecord(L->ev_bar, cs));
      comm_symmetric_set_pending(L->comm, y, L->ev_bar);
    } else {
      CP_TRY(comm_barrier(L->comm, s));
    }
  }
  if (sym_in && !(tf32 && has_gemm)) CP_TRY(launch_wait_flags(arrive, L->d.world, me, s, tf32 && !epi_push));
  if (has_gemm) {
    if (c1) {
      CP_TRY(c1_fwd(*L, x, w, b, yb, saved, s));
    } else if (tf32) {
      CP_TRY(tc_fwd(*L, xin, w, b, yb, saved, ws, s, push_in_epilogue ? peer_blocks : nullptr,
                    push_in_epilogue ? npeers : 0, arrive, kernel_push ? &gp : nullptr));
    } else if (L->d.math == CP_MATH_BF16) {
      // report-only bf16 mode: the GEMM reads bf16 copies of its input and weights (fp32 outputs);
      // the gathered input is complete here (copy-engine distribution + flags above)
      const int64_t nx = L->images ? (int64_t)L->Ho * L->Wo * L->Bp * L->Kcol : L->in.start[L->in.n];
      float* x16 = (float*)WS(ws, L->off_x16);
      float* w16 = (float*)WS(ws, L->off_w16);
      CP_TRY(launch_to_bf16(xin, x16, nx, s));
      CP_TRY(launch_to_bf16(w, w16, (int64_t)L->Kr * L->Ktot, s));
      CP_TRY(tc_fwd(*L, x16, w16, b, yb, saved, ws, s, nullptr, 0, nullptr, nullptr));
    } else {
      float* z = (float*)WS(ws, L->off_z);
      CP_TRY(launch_fwd_simt(*L, x, xin, w, b, z, s));
      CP_TRY(launch_relu_pool(*L, z, yb, saved, false, s));
    }
  }
  // reset the arrival counters and the push claim counter (the whole 256 B flag line)
  if (sym_in) CP_CUDA(cudaMemsetAsync((void*)arrive, 0, 256, s));
  if (ce_forked) CP_CUDA(cudaStreamWaitEvent(s, L->ev_gjoin, 0));   // own outgoing copies done
  if (push_in_epilogue) {
    CP_TRY(launch_signal_peers(signal, npeers, me, s));
  } else if (gathered_out && !sym_out) {
    CP_TRY(fork_comm(*L, s, cs));
    CP_TRY(comm_allgather_blocks(L->comm, y, L->out, cs));
    CP_TRY(join_comm(*L, s, cs));
  }
  return CP_OK;
}

// fused reduce-scatter variant: pull (default; owners read the partials) or push (CP_RS_MODE=push: the
// dgrad epilogue stores each partial into its owner's receive slot)
int conv_part_backward_data(cp_layer L, const float* dy_g, const uint8_t* saved, const float* y_g, const float* w,
                            float* dx, int32_t dx_mode, void* ws, void* stream, void* comm_stream) {
  if (!L || !dy_g || !y_g || !w || !dx || !ws) CP_FAIL(CP_ERR_ARG, "conv_part_backward_data: null pointer");
  if (L->d.pool && !saved) CP_FAIL(CP_ERR_ARG, "conv_part_backward_data: pooling needs saved");
  const bool async = (dx_mode & CP_DX_ASYNC) != 0;
  const bool ordered = (dx_mode & CP_DX_ORDERED) != 0;
  dx_mode &= ~(CP_DX_ASYNC | CP_DX_ORDERED);
  if (dx_mode < CP_DX_ALLREDUCE || dx_mode > CP_DX_LOCAL) CP_FAIL(CP_ERR_ARG, "bad dx_mode");
  if (L->images && dx_mode == CP_DX_REDUCE_SCATTER)
    CP_FAIL(CP_ERR_UNSUPPORTED, "reduce-scatter of dX needs a gather-layout input (images use all-reduce)");
  cudaStream_t s = (cudaStream_t)stream, cs = comm_stream ? (cudaStream_t)comm_stream : s;
  CP_TRY(ensure_dy(*L, dy_g, saved, y_g, ws, s));
  const float* dY = (const float*)WS(ws, L->off_dy);
  // Fused reduce-scatter (B200 path): dx symmetric with receive slots behind the
  // gather layout; the dgrad epilogue stores block q's partial into rank q's slot [this rank].
  void* peers[CP_MAX_RANKS];
  uint32_t* pflags[CP_MAX_RANKS];
  // GEMM operands: fp32 (tf32 mode) or the bf16 copies (bf16 mode; weights re-rounded here)
  const bool bf16 = L->d.math == CP_MATH_BF16;
  const float* dYg = bf16 ? (const float*)WS(ws, L->off_dy16) : dY;
  const float* wg = w;
  if (bf16) {
    CP_TRY(launch_to_bf16(w, WS(ws, L->off_w16), (int64_t)L->Kr * L->Ktot, s));
    wg = (const float*)WS(ws, L->off_w16);
  }
  const bool fused = L->d.math != CP_MATH_FP32_SIMT && !L->images && L->comm && L->d.world > 1 &&
                     dx_mode == CP_DX_REDUCE_SCATTER && comm_symmetric_peers(L->comm, dx, peers, pflags);
  // Pull variants (CP_RS_MODE=pull / ce): the dgrad writes every partial block into this rank's OWN copy
  // (plain local epilogue), raises "partials ready" at every peer, and each owner's comm-stream tail
  // fetches its block's partials from all copies over NVLink - SM loads (pull) or copy-engine copies
  // into its receive slots (ce) - and sums them in rank order; the transfer overlaps the next GEMM
  // (wgrad) instead of slowing the dgrad epilogue with peer stores.
  const int rsm = fused ? rs_mode() : 0;
  if (rsm != 0) {
    const int me = L->d.rank, world = L->d.world;
    uint32_t* signal[CP_MAX_RANKS];
    int ns = 0;
    for (int q = 0; q < world; ++q)
      if (q != me) signal[ns++] = pflags[q];
    if (!ordered) CP_TRY(comm_barrier(L->comm, s));   // no owner still reads last call's partials
    if (L->Kr > 0 && L->Kc > 0) {
      CP_TRY(tc_dgrad(*L, dYg, wg, dx, ws, s));
    } else {   // no own kernels: zero partials (the owners still read them)
      CP_TRY(launch_fill(dx, 0.f, L->in.start[L->in.n], s));
    }
    CP_TRY(launch_signal_peers(signal, ns, me, s));
    CP_CUDA(cudaEventRecord(L->ev_compute, s));
    uint32_t* own_flags = pflags[me];
    const int64_t off = L->in.start[me], n_own = L->in.start[me + 1] - L->in.start[me];
    int64_t mb = 0;
    for (int r = 0; r < L->in.n; ++r) mb = std::max(mb, L->in.start[r + 1] - L->in.start[r]);
    float* slots = dx + L->in.start[L->in.n];   // receive slots behind the gather layout (ce mode)
    const float* src[CP_MAX_RANKS];
    const float* remote[CP_MAX_RANKS];
    for (int r = 0; r < world; ++r) {
      remote[r] = (const float*)peers[r] + off;
      src[r] = (rsm == 2 && r != me) ? slots + (int64_t)r * mb : remote[r];
    }
    float* own = dx + off;
    cp_layer_s* Lp = L;
    std::vector<const float*> srcv(src, src + world), remv(remote, remote + world);
    auto tail = [=](const std::vector<cudaEvent_t>& computed) -> int {
      for (cudaEvent_t e : computed) CP_CUDA(cudaStreamWaitEvent(cs, e, 0));
      CP_TRY(launch_wait_flags(own_flags, world, me, cs));
      if (rsm == 2) {   // copy engines: every peer's partial of the own block into its local receive slot
        CP_TRY(tc_time_mark(*Lp, 4, 0, cs));   // transfer window: all partials ready -> copies done
        // CP_RS_CE_STREAMS=2: each copy in two halves, the second on another copy engine (stream cs2)
        const bool split = tc_env_int("CP_RS_CE_STREAMS", 1) >= 2;
        if (split && !Lp->cs2) {
          CP_CUDA(cudaStreamCreateWithFlags(&Lp->cs2, cudaStreamNonBlocking));
          for (int k = 0; k < CP_MAX_RANKS; ++k)
            CP_CUDA(cudaEventCreateWithFlags(&Lp->ev_split[k], cudaEventDisableTiming));
        }
        const int64_t h = split ? (n_own / 2 + 3) / 4 * 4 : n_own;
        if (split) {
          CP_CUDA(cudaEventRecord(Lp->ev_split[0], cs));
          CP_CUDA(cudaStreamWaitEvent(Lp->cs2, Lp->ev_split[0], 0));
        }
        for (int r = 0; r < world; ++r)
          if (r != me && n_own) {
            CP_CUDA(cudaMemcpyAsync((void*)srcv[r], remv[r], (size_t)h * 4, cudaMemcpyDeviceToDevice, cs));
            if (split && n_own > h)
              CP_CUDA(cudaMemcpyAsync((void*)(srcv[r] + h), remv[r] + h, (size_t)(n_own - h) * 4,
                                      cudaMemcpyDeviceToDevice, Lp->cs2));
          }
        if (split) {
          CP_CUDA(cudaEventRecord(Lp->ev_split[1], Lp->cs2));
          CP_CUDA(cudaStreamWaitEvent(cs, Lp->ev_split[1], 0));
        }
        CP_TRY(tc_time_mark(*Lp, 4, 1, cs));
        if (Lp->timing) Lp->rs_timed = 1;
      }
      CP_TRY(launch_sum_peer_blocks(srcv.data(), world, own, n_own, cs));
      CP_CUDA(cudaMemsetAsync(own_flags, 0, CP_MAX_RANKS * sizeof(uint32_t), cs));
      CP_CUDA(cudaEventRecord(Lp->ev_comm, cs));
      if (!(async && cs != s)) CP_CUDA(cudaStreamWaitEvent(s, Lp->ev_comm, 0));
      return CP_OK;
    };
    if (comm_is_loopback(L->comm)) return comm_loopback_defer(L->comm, L->ev_compute, tail);
    return tail(std::vector<cudaEvent_t>{L->ev_compute});
  }
  if (fused) {
    int64_t mb = 0;
    for (int r = 0; r < L->in.n; ++r) mb = std::max(mb, L->in.start[r + 1] - L->in.start[r]);
    const int64_t slots0 = L->in.start[L->in.n];   // receive slots follow the gather layout
    const int me = L->d.rank;
    float* dst[CP_MAX_RANKS];
    uint32_t* signal[CP_MAX_RANKS];
    int ns = 0;
    // CP_RS_LOCAL_DIAG=1 (timing diagnostic, WRONG results): every partial into the own copy's slots
    static const int rs_local_diag = tc_env_int("CP_RS_LOCAL_DIAG", 0);
    for (int q = 0; q < L->in.n; ++q) {
      dst[q] = (float*)peers[rs_local_diag ? me : q] + slots0 + (int64_t)(rs_local_diag ? q : me) * mb;
      if (q != me) signal[ns++] = pflags[q];
    }
    if (!ordered) CP_TRY(comm_barrier(L->comm, s));   // no rank still sums last call's slots
    if (L->Kr > 0 && L->Kc > 0) {
      CP_TRY(tc_dgrad(*L, dYg, wg, dx, ws, s, dst));
    } else {   // no own kernels: a zero partial for every block (peers still expect the signal)
      for (int q = 0; q < L->in.n; ++q) CP_TRY(launch_fill(dst[q], 0.f, L->in.start[q + 1] - L->in.start[q], s));
    }
    CP_TRY(launch_signal_peers(signal, ns, me, s));
    CP_CUDA(cudaEventRecord(L->ev_compute, s));
    // comm-stream tail: wait for every peer's slot, sum the slots in rank order into the own block
    uint32_t* own_flags = pflags[me];
    const int world = L->d.world;
    const int64_t n_own = L->in.start[me + 1] - L->in.start[me];
    float* slots = dx + slots0;
    float* own = dx + L->in.start[me];
    cp_layer_s* Lp = L;
    auto tail = [=](const std::vector<cudaEvent_t>& computed) -> int {
      for (cudaEvent_t e : computed) CP_CUDA(cudaStreamWaitEvent(cs, e, 0));
      CP_TRY(launch_wait_flags(own_flags, world, me, cs));
      CP_TRY(launch_sum_slots(slots, mb, world, own, n_own, cs));
      CP_CUDA(cudaMemsetAsync(own_flags, 0, CP_MAX_RANKS * sizeof(uint32_t), cs));
      CP_CUDA(cudaEventRecord(Lp->ev_comm, cs));
      if (!(async && cs != s)) CP_CUDA(cudaStreamWaitEvent(s, Lp->ev_comm, 0));
      return CP_OK;
    };
    // loopback (simulated ranks on one GPU): tails run once every rank issued its dgrad
    if (comm_is_loopback(L->comm)) return comm_loopback_defer(L->comm, L->ev_compute, tail);
    return tail(std::vector<cudaEvent_t>{L->ev_compute});
  }
  if (L->d.math != CP_MATH_FP32_SIMT && !L->images) {
    CP_TRY(tc_dgrad(*L, dYg, wg, dx, ws, s));
  } else {
    CP_TRY(launch_dgrad_simt(*L, dY, w, dx, s));
  }
  if (L->comm && L->d.world > 1 && dx_mode != CP_DX_LOCAL) {
    CP_TRY(fork_comm(*L, s, cs));
    if (L->images) {
      Blocks flat{};
      flat.n = 1;
      flat.start[0] = 0;
      flat.start[1] = (int64_t)L->B * L->C * L->H * L->W;
      CP_TRY(comm_sum_blocks(L->comm, dx, flat, CP_DX_ALLREDUCE, cs));
    } else {
      CP_TRY(comm_sum_blocks(L->comm, dx, L->in, dx_mode, cs));
    }
    if (async && cs != s) {
      CP_CUDA(cudaEventRecord(L->ev_comm, cs));
    } else {
      CP_TRY(join_comm(*L, s, cs));
    }
  }
  return CP_OK;
}

// backward-filter with an optional SGD update of the own slice (w, b non-null): fused into the kernels that
// produce the final dW / db (wgrad epilogue, its tail / split reduce, the bias reduce, the conv1 reduce);
// the modes without a fused variant run the separate update after the pass
static int backward_filter(cp_layer L, const float* dy_g, const uint8_t* saved, const float* y_g, const float* x,
                           float* dw, float* db, float* w, float* b, float lr, void* ws, cudaStream_t s) {
  if (L->Kr == 0) return CP_OK;
  if (L->images && L->d.math == CP_MATH_TF32 && c1_wgrad_supported(*L)) {
    // image layer: unpool + ReLU' + wgrad + db fused (no dY, no im2col rows in HBM)
    const int64_t o = L->out.start[L->d.rank];
    return c1_wgrad(*L, x, dy_g + o, saved, y_g + o, dw, db, (float*)WS(ws, L->off_c1w), s, w, b, lr);
  }
  CP_TRY(ensure_dy(*L, dy_g, saved, y_g, ws, s));
  if (db) CP_TRY(launch_bias_grad(*L, db, (const float*)WS(ws, L->off_dbpart), s, b, lr));
  const float* dY = (const float*)WS(ws, L->off_dy);
  const float* xcol = L->images ? (const float*)WS(ws, L->off_xcol) : nullptr;
  if (L->images && L->xcol_key != x) {   // the forward built its rows on chip: im2col for wgrad here
    CP_TRY(launch_im2col(*L, x, (float*)WS(ws, L->off_xcol), L->d.math == CP_MATH_TF32, s));
    L->xcol_key = x;
  }
  if (L->d.math == CP_MATH_TF32) {
    CP_TRY(tc_wgrad(*L, dY, L->images ? xcol : x, dw, ws, s, w, lr));
  } else if (L->d.math == CP_MATH_BF16) {   // bf16 copies of dY (ensure_dy) and of the input (forward)
    CP_TRY(tc_wgrad(*L, (const float*)WS(ws, L->off_dy16), (const float*)WS(ws, L->off_x16), dw, ws, s, w, lr));
  } else {
    CP_TRY(launch_wgrad_simt(*L, dY, x, xcol, dw, s));
    if (w) CP_TRY(cp_sgd(w, dw, (int64_t)L->Kr * L->Ktot, lr, s));
  }
  return CP_OK;
}

int conv_part_backward_filter(cp_layer L, const float* dy_g, const uint8_t* saved, const float* y_g, const float* x,
                              float* dw, float* db, void* ws, void* stream) {
  if (!L || !dy_g || !y_g || !x || !dw || !ws) CP_FAIL(CP_ERR_ARG, "conv_part_backward_filter: null pointer");
  if (L->d.pool && !saved) CP_FAIL(CP_ERR_ARG, "conv_part_backward_filter: pooling needs saved");
  return backward_filter(L, dy_g, saved, y_g, x, dw, db, nullptr, nullptr, 0.f, ws, (cudaStream_t)stream);
}

int conv_part_backward_filter_sgd(cp_layer L, const float* dy_g, const uint8_t* saved, const float* y_g,
                                  const float* x, float* dw, float* db, float* w, float* b, float lr, void* ws,
                                  void* stream) {
  if (!L || !dy_g || !y_g || !x || !dw || !ws || !w) CP_FAIL(CP_ERR_ARG, "conv_part_backward_filter_sgd: null pointer");
  if (L->d.pool && !saved) CP_FAIL(CP_ERR_ARG, "conv_part_backward_filter_sgd: pooling needs saved");
  if ((b != nullptr) != (db != nullptr))
    CP_FAIL(CP_ERR_ARG, "conv_part_backward_filter_sgd: b and db must be given together");
  if (w == dw || (b && b == db)) CP_FAIL(CP_ERR_ARG, "conv_part_backward_filter_sgd: w/b must not alias dw/db");
  return backward_filter(L, dy_g, saved, y_g, x, dw, db, w, b, lr, ws, (cudaStream_t)stream);
}

int conv_part_timing(cp_layer L, int32_t enable) {
  if (!L) CP_FAIL(CP_ERR_ARG, "conv_part_timing: null layer");
  if (enable && !L->timing) {
    for (int p = 0; p < 5; ++p)
      for (int e = 0; e < 2; ++e)
        if (!L->ev_t[p][e]) CP_CUDA(cudaEventCreate(&L->ev_t[p][e]));
    L->ce_gather_timed = L->rs_timed = 0;
  }
  L->timing = enable ? 1 : 0;
  return CP_OK;
}

int conv_part_kernel_time(cp_layer L, int32_t pass, float* ms) {
  if (!L || !ms || pass < 0 || pass > 4) CP_FAIL(CP_ERR_ARG, "conv_part_kernel_time: bad arguments");
  if (!L->timing) CP_FAIL(CP_ERR_STATE, "conv_part_kernel_time: timing not enabled");
  if (pass == 4) {   // reduce-scatter transfer window (copy-engine fetch of the partials, comm stream)
    if (!L->rs_timed) CP_FAIL(CP_ERR_STATE, "conv_part_kernel_time: no copy-engine reduce-scatter recorded");
    CP_CUDA(cudaEventElapsedTime(ms, L->ev_t[4][0], L->ev_t[4][1]));
    return CP_OK;
  }
  if (pass == 3 && L->ce_gather_timed) {   // copy-engine gather window (comm stream events)
    CP_CUDA(cudaEventElapsedTime(ms, L->ev_t[3][0], L->ev_t[3][1]));
    return CP_OK;
  }
  if (pass == 3) {   // fused gather push window (globaltimer stamps in the workspace; blocking read)
    if (!L->ws_last) CP_FAIL(CP_ERR_STATE, "conv_part_kernel_time: no forward with a fused gather push yet");
    unsigned long long t[2];
    CP_CUDA(cudaMemcpy(t, (char*)L->ws_last + L->off_stamp, sizeof(t), cudaMemcpyDeviceToHost));
    if (t[0] == ~0ull || t[1] < t[0]) CP_FAIL(CP_ERR_STATE, "conv_part_kernel_time: no push recorded");
    *ms = (float)((double)(t[1] - t[0]) * 1e-6);
    return CP_OK;
  }
  CP_CUDA(cudaEventElapsedTime(ms, L->ev_t[pass][0], L->ev_t[pass][1]));
  return CP_OK;
}

int conv_part_wait(cp_layer L, void* stream) {
  if (!L) CP_FAIL(CP_ERR_ARG, "conv_part_wait: null layer");
  CP_CUDA(cudaStreamWaitEvent((cudaStream_t)stream, L->ev_comm, 0));
  return CP_OK;
}

int conv_part_sgd_step(cp_layer L, float* w, float* b, const float* dw, const float* db, float lr, void* stream) {
  if (!L || !w || !dw) CP_FAIL(CP_ERR_ARG, "conv_part_sgd_step: null pointer");
  CP_TRY(cp_sgd(w, dw, (int64_t)L->Kr * L->Ktot, lr, stream));
  if (b && db) CP_TRY(cp_sgd(b, db, L->Kr, lr, stream));
  return CP_OK;
}

int conv_part_probe_bytes(const cp_conv_desc* desc, size_t* bytes) {
  if (!desc || !bytes) CP_FAIL(CP_ERR_ARG, "conv_part_probe_bytes: null pointer");
  cp_conv_desc d = *desc;
  d.out_part = cp_partition{};
  d.out_part.n_ranks = 1;
  d.out_part.num_k = d.num_k;
  d.out_part.k_count[0] = d.num_k;
  d.out_part.k_width[0] = roundup(d.num_k, 8);
  d.rank = 0;
  d.world = 1;
  Layer L{};
  CP_TRY(derive(L, d));
  const size_t x = L.images ? (size_t)L.B * L.C * L.H * L.W * 4 : (size_t)L.in.start[L.in.n] * 4;
  *bytes = al256(x + 256) + al256((size_t)L.Kr * L.Ktot * 4 + 256) + al256((size_t)L.Kc * 4) +
           al256((size_t)L.out.start[1] * 4 + 256) + al256((size_t)L.Hp * L.Wp * L.Bp * L.Kc) + al256(L.ws_total);
  return CP_OK;
}

int conv_part_probe(const cp_conv_desc* desc, int32_t warmups, int32_t reps, void* scratch, size_t scratch_bytes,
                    void* stream, double* median_s) {
  if (!desc || !scratch || !median_s) CP_FAIL(CP_ERR_ARG, "conv_part_probe: null pointer");
  if (reps < 1 || warmups < 0) CP_FAIL(CP_ERR_ARG, "conv_part_probe: reps >= 1, warmups >= 0");
  size_t need = 0;
  CP_TRY(conv_part_probe_bytes(desc, &need));
  if (scratch_bytes < need) CP_FAIL(CP_ERR_ARG, "conv_part_probe: scratch too small, need " + std::to_string(need));
  cp_conv_desc d = *desc;
  d.out_part = cp_partition{};
  d.out_part.n_ranks = 1;
  d.out_part.num_k = d.num_k;
  d.out_part.k_count[0] = d.num_k;
  d.out_part.k_width[0] = roundup(d.num_k, 8);
  d.rank = 0;
  d.world = 1;
  cp_layer L = nullptr;
  CP_TRY(conv_part_create(&d, nullptr, &L));
  cudaStream_t s = (cudaStream_t)stream;
  char* p = (char*)scratch;
  const size_t xb = L->images ? (size_t)L->B * L->C * L->H * L->W * 4 : (size_t)L->in.start[L->in.n] * 4;
  float* x = (float*)p; p += al256(xb + 256);
  float* w = (float*)p; p += al256((size_t)L->Kr * L->Ktot * 4 + 256);
  float* b = (float*)p; p += al256((size_t)L->Kc * 4);
  float* y = (float*)p; p += al256((size_t)L->out.start[1] * 4 + 256);
  uint8_t* sv = (uint8_t*)p; p += al256((size_t)L->Hp * L->Wp * L->Bp * L->Kc);
  void* ws = p;
  // "The convolution is run using random values, since only the time spent performing
  // calculations is relevant".
  int rc = launch_random_fill(x, xb / 4, 1234u, 1.0f, s);
  if (rc == CP_OK) rc = launch_random_fill(w, (int64_t)L->Kr * L->Ktot, 5678u, 0.01f, s);
  if (rc == CP_OK) rc = launch_fill(b, 0.f, L->Kc, s);
  std::vector<double> t;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (rc == CP_OK && (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)) {
    set_error("conv_part_probe: event create failed");
    rc = CP_ERR_CUDA;
  }
  for (int i = 0; rc == CP_OK && i < warmups + reps; ++i) {
    cudaEventRecord(e0, s);
    rc = conv_part_forward(L, x, w, b, y, sv, ws, s, s);
    cudaEventRecord(e1, s);
    if (rc == CP_OK && cudaEventSynchronize(e1) != cudaSuccess) {
      set_error("conv_part_probe: kernel failure");
      rc = CP_ERR_CUDA;
    }
    float ms = 0;
    if (rc == CP_OK) cudaEventElapsedTime(&ms, e0, e1);
    if (i >= warmups) t.push_back(ms * 1e-3);
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  conv_part_destroy(L);
  if (rc != CP_OK) return rc;
  std::sort(t.begin(), t.end());
  *median_s = t[t.size() / 2];
  return CP_OK;
}

}  // extern "C"
