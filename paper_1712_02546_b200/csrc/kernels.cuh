// kernels.cuh — internal launchers (namespace cp).  All enqueue on `s` and count launches.
#pragma once
#include <functional>
#include <vector>

#include <cuda.h>

#include "common.cuh"

namespace cp {

constexpr int kGatherChunks = CP_GATHER_CHUNKS;   // pieces of a kernel-pushed gather block (= the receivers' target)

// ---- layout / elementwise (kernels_simt.cu)
int launch_im2col(const Layer& L, const float* x, float* xcol, bool round_tf32, cudaStream_t s);
int launch_relu_pool(const Layer& L, const float* z, float* y_block, uint8_t* saved, bool round_tf32,
                     cudaStream_t s);
// unpool + ReLU' of the own block; also writes the bias-gradient partials (bias_part, may be null)
constexpr int kBiasSplitMax = 256;
int launch_unpool(const Layer& L, const float* dy_block, const uint8_t* saved, const float* y_block,
                  float* dY, float* bias_part, bool round_tf32, cudaStream_t s);
// db from the partials launch_unpool wrote
int launch_bias_grad(const Layer& L, float* db, const float* part, cudaStream_t s, float* sgd_b = nullptr,
                     float lr = 0.f);

// ---- FP32 SIMT reference convolutions (kernels_simt.cu)
int launch_fwd_simt(const Layer& L, const float* x, const float* xcol, const float* w, const float* b,
                    float* z, cudaStream_t s);
int launch_dgrad_simt(const Layer& L, const float* dY, const float* w, float* dx, cudaStream_t s);
int launch_wgrad_simt(const Layer& L, const float* dY, const float* x, const float* xcol, float* dw,
                      cudaStream_t s);
int launch_fill(float* p, float v, int64_t n, cudaStream_t s);
// fp32 -> bf16 (round to nearest even) copy of n elements (CP_MATH_BF16 operand copies)
int launch_to_bf16(const float* src, void* dst, int64_t n, cudaStream_t s);
int launch_random_fill(float* p, int64_t n, uint32_t seed, float scale, cudaStream_t s);
// cross-GPU arrival flags (fused AllGather): set slot `slot` of every peer's flag array / wait for
// every slot of the own array except `self` (for consumers outside the tensor-core forward)
int launch_signal_peers(uint32_t* const* peer_flags, int n, int slot, cudaStream_t s);
int launch_wait_flags(const uint32_t* flags, int n, int self, cudaStream_t s, bool chunks = false);

// ---- tcgen05 / TMA tensor-core convolutions (kernels_tc.cu)
size_t tc_workspace_bytes(const Layer& L);
// create-time validation of the tensor-core plans (every launch-time rejection, checked up front)
int tc_validate(const Layer& L);
// fused all-gather -> GEMM (forward over a symmetric gathered input): the kernel's warp 3 pushes
// this rank's input block (src, n4 float4) into each peer's copy dst[k] in `chunks` pieces, one
// release-add on the peer's arrival counter cnt[k] per piece; the GEMM waits for `chunks` arrivals
// from every peer before consuming that peer's block.
struct GatherPush {
  const float* src;
  float* dst[CP_MAX_RANKS];
  uint32_t* cnt[CP_MAX_RANKS];
  uint32_t* claim;   // chunk claim counter, zero at launch (own flag line word kClaimWord)
  unsigned long long* stamp = nullptr;  // timing: [0] min start, [1] max end (globaltimer ns) of the push
  int n, chunks;
  long long n4;
  int mc = 0;   // 1: dst[0] / cnt[0] are multicast addresses (one store reaches every rank)
};
constexpr int kClaimWord = 32;   // flag-line word of a symmetric gathered input: the push claim counter
int tc_fwd(Layer& L, const float* xin, const float* w, const float* b, float* y_block, uint8_t* saved,
           void* ws, cudaStream_t s, float* const* peer_blocks = nullptr, int npeers = 0,
           const uint32_t* arrive = nullptr, const GatherPush* gp = nullptr);
// dst_blocks (fused reduce-scatter): per input block, where this rank's partial of that block goes
int tc_dgrad(Layer& L, const float* dY, const float* w, float* dx, void* ws, cudaStream_t s,
             float* const* dst_blocks = nullptr);
// dx_own = sum over q (ascending) of the P receive slots (fused reduce-scatter epilogue)
// pull reduce-scatter: out = sum over r ascending of src[r] (n floats, 16-byte aligned blocks)
int launch_sum_peer_blocks(const float* const* src, int n_src, float* out, int64_t n, cudaStream_t s);
int launch_sum_slots(const float* slots, int64_t slot_stride, int n_slots, float* out, int64_t n, cudaStream_t s);
// sgd_w: fused SGD update of the own weights wherever the final dW is produced (w -= sgd_lr * dW)
int tc_wgrad(Layer& L, const float* dY, const float* xin, float* dw, void* ws, cudaStream_t s, float* sgd_w = nullptr,
             float sgd_lr = 0.f);
void tc_release(Layer& L);
// helpers of kernels_tc.cu shared with kernels_conv1.cu
int tc_make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                const uint32_t* box, bool mn_major, int es);
int tc_num_sms();
int tc_make_map_plain(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                      const uint32_t* box);
int tc_env_int(const char* name, int dflt);
// dedicated image-layer (conv1) forward: transposed tcgen05 GEMM with the im2col rows built in shared
// memory from the NCHW images and the 2x2 pool in registers (kernels_conv1.cu); false = use tc_fwd
bool c1_fwd_supported(const Layer& L);
int c1_fwd(Layer& L, const float* x, const float* w, const float* b, float* y_block, uint8_t* saved, cudaStream_t s);
// fused image-layer backward-filter: unpool + ReLU' + wgrad + db in one split-K tcgen05 kernel + a
// deterministic reduce (kernels_conv1.cu); da/codes/y are the own pooled block; part = workspace
bool c1_wgrad_supported(const Layer& L);
size_t c1_wgrad_workspace(const Layer& L);
int c1_wgrad(Layer& L, const float* x, const float* da, const uint8_t* codes, const float* y, float* dw, float* db,
             float* part, cudaStream_t s, float* sgd_w = nullptr, float* sgd_b = nullptr, float lr = 0.f);
// timing events around a pass's GEMM launch (no-ops unless L.timing): external records, so they
// also time when the launch is captured into a CUDA graph
int tc_time_mark(Layer& L, int pass, int end, cudaStream_t s);

// ---- NCCL collectives (comm.cu)
int comm_check_plan(cp_comm c, const Layer& L);
int comm_allgather_blocks(cp_comm c, float* buf, const Blocks& g, cudaStream_t s);
// symmetric (peer-mapped) buffer lookup: peers[r] = rank r's copy; flags[r] = rank r's arrival-flag
// array (CP_MAX_RANKS u32, indexed by sender rank).  False if `local` is not a symmetric buffer.
bool comm_symmetric_peers(cp_comm c, const void* local, void** peers, uint32_t** flags = nullptr);
// deferred producer barrier of a symmetric gathered buffer: recorded by the producer's forward on the
// comm stream, waited for (once) by the consumer's forward before it distributes its block
void comm_symmetric_set_pending(cp_comm c, const void* local, cudaEvent_t ev);
cudaEvent_t comm_symmetric_take_pending(cp_comm c, const void* local);
// NVLink multicast address of a symmetric buffer (CP_MULTICAST=1), else nullptr
void* comm_symmetric_mc(cp_comm c, const void* local);
bool multicast_requested();
// producer records its block of a symmetric gathered buffer (for copy-engine distribution)
void comm_symmetric_set_own(cp_comm c, const void* local, int64_t off, int64_t elems);
int comm_ce_distribute(cp_comm c, const void* local, cudaStream_t s, bool chunks = false, cudaStream_t s2 = nullptr,
                       const cudaEvent_t* evs = nullptr);
// CP_GATHER_PUSH=epilogue: the producer's GEMM epilogue pushes (A/B experiment), else the consumer
bool gather_push_in_epilogue();
// cross-rank barrier on s (device-side epoch flags once symmetric memory exists, else NCCL)
int comm_barrier(cp_comm c, cudaStream_t s);
// raise slot `slot` of each flag array with copy-engine writes (no SM), ordered after prior copies on s
// (value 1, or kGatherChunks when `chunks`: stands in for a kernel push of zero bytes)
int comm_signal_ce(cp_comm c, uint32_t* const* flags, int n, int slot, cudaStream_t s, bool chunks = false);
int comm_sum_blocks(cp_comm c, float* buf, const Blocks& g, int dx_mode, cudaStream_t s);
// loopback communicator (P simulated ranks on one GPU, cp_comm_create_loopback)
bool comm_is_loopback(cp_comm c);
// hold `tail` (the comm-stream part of a fused reduce-scatter) until every simulated rank issued its
// compute (`done` recorded after it), then run all tails in rank order with every rank's `done`
int comm_loopback_defer(cp_comm c, cudaEvent_t done, std::function<int(const std::vector<cudaEvent_t>&)> tail);

}  // namespace cp
