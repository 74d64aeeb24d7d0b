// common.cuh — internal helpers of libconvpart (B200, sm_100a).
// Nothing here is shared with the oracle (oracle/ is a separate C program).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <string>

#include "../../include/convpart.h"

namespace cp {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
std::atomic<int64_t>& launch_counter();

#define CP_FAIL(code, msg)         \
  do {                             \
    ::cp::set_error(msg);          \
    return (code);                 \
  } while (0)

#define CP_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e__ = (call);                                                              \
    if (e__ != cudaSuccess) {                                                              \
      ::cp::set_error(std::string(#call) + ": " + cudaGetErrorString(e__));                \
      return CP_ERR_CUDA;                                                                  \
    }                                                                                      \
  } while (0)

// after a kernel launch: count it and surface launch errors
#define CP_LAUNCHED()                                                                      \
  do {                                                                                     \
    ::cp::launch_counter().fetch_add(1, std::memory_order_relaxed);                        \
    cudaError_t e__ = cudaGetLastError();                                                  \
    if (e__ != cudaSuccess) {                                                              \
      ::cp::set_error(std::string("kernel launch (") + __FILE__ + ":" +                   \
                      std::to_string(__LINE__) + "): " + cudaGetErrorString(e__));         \
      return CP_ERR_CUDA;                                                                  \
    }                                                                                      \
  } while (0)

#define CP_TRY(expr)                 \
  do {                               \
    int rc__ = (expr);               \
    if (rc__ != CP_OK) return rc__;  \
  } while (0)

static inline int roundup(int a, int b) { return (a + b - 1) / b * b; }
static inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------- gather geometry
// A tensor in the rank-blocked gather layout: blocks [H][W][Bp][kw[r]] in rank order.
struct Blocks {
  int n;                     // number of rank blocks
  int H, W, Bp;              // spatial extent of every block, padded batch
  int kb[CP_MAX_RANKS];      // first logical channel of block r
  int kc[CP_MAX_RANKS];      // real channels in block r
  int kw[CP_MAX_RANKS];      // slots in block r (multiple of 8)
  int coff[CP_MAX_RANKS];    // slot offset of block r in the concatenated slot space
  int64_t start[CP_MAX_RANKS + 1];  // element offset of block r (start[n] = total)
  int Cg;                    // total slots = sum kw
};

// experiment hook: extra floats between consecutive rank blocks (L2 set-aliasing study)
static inline int64_t block_pad() {
  static const int64_t v = [] {
    const char* e = getenv("CP_BLOCK_PAD");
    return e ? (int64_t)atoll(e) / 32 * 32 : (int64_t)0;
  }();
  return v;
}

static inline Blocks make_blocks(const cp_partition& p, int H, int W, int Bp) {
  Blocks g{};
  g.n = p.n_ranks;
  g.H = H;
  g.W = W;
  g.Bp = Bp;
  int64_t s = 0;
  int c = 0;
  for (int r = 0; r < p.n_ranks; ++r) {
    g.kb[r] = p.k_begin[r];
    g.kc[r] = p.k_count[r];
    g.kw[r] = p.k_width[r];
    g.coff[r] = c;
    g.start[r] = s;
    c += p.k_width[r];
    s += (int64_t)H * W * Bp * p.k_width[r];
    if (r + 1 < p.n_ranks) s += block_pad();
  }
  g.start[p.n_ranks] = s;
  g.Cg = c;
  return g;
}

// block owning concatenated slot c' (device side; n <= 16, linear scan)
__host__ __device__ inline int block_of_slot(const Blocks& g, int cslot) {
  int r = 0;
  while (r + 1 < g.n && cslot >= g.coff[r + 1]) ++r;
  return r;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ---------------------------------------------------------------- cross-GPU arrival flags
// A producer rank sets its slot in every consumer's flag array (st.release.sys after its peer stores);
// the consumer spins with ld.acquire.sys.  The spin is bounded (~2^35 cycles, >15 s): a missing
// signal traps (a reported launch failure) instead of hanging the GPU.
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// softmax cross-entropy over B rows of O <= kHeadMaxO logits by one thread block:
// loss = mean_b (logsumexp(l_b) - l_b[y_b]), dl = (softmax - onehot) / B; the loss sum is a
// fixed-order tree (warp shuffles, then the warps in order) - identical wherever it runs.
// wsum: shared scratch of blockDim/32 floats.
constexpr int kHeadMaxO = 16;
__device__ __forceinline__ void softmax_xent_block(const float* logits, const int* y, int B, int O, float* loss,
                                                   float* dl, float* wsum) {
  float part = 0.f;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const float* lp = logits + (int64_t)b * O;   // the row's logits in registers (one pass)
    float l[kHeadMaxO];
#pragma unroll
    for (int o = 0; o < kHeadMaxO; ++o) l[o] = o < O ? lp[o] : -INFINITY;
    const int lab = y[b];
    float m = l[0];
#pragma unroll
    for (int o = 1; o < kHeadMaxO; ++o) m = fmaxf(m, l[o]);
    float se = 0.f;
#pragma unroll
    for (int o = 0; o < kHeadMaxO; ++o)
      if (o < O) se += expf(l[o] - m);
    const float lse = m + logf(se);
    if (lab < 0 || lab >= O) {
      part += __int_as_float(0x7fc00000);  // NaN loss flags an out-of-range label
      continue;
    }
    float ll = 0.f;
#pragma unroll
    for (int o = 0; o < kHeadMaxO; ++o)
      if (o == lab) ll = l[o];
    part += lse - ll;
#pragma unroll
    for (int o = 0; o < kHeadMaxO; ++o)
      if (o < O) dl[(int64_t)b * O + o] = (expf(l[o] - lse) - (o == lab ? 1.f : 0.f)) / (float)B;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += wsum[w];
    *loss = t / (float)B;
  }
}

// wait until *p >= target (arrival counters / flags)
__device__ __forceinline__ void wait_flag_sys(const uint32_t* p, uint32_t target = 1) {
  const long long t0 = clock64();
  while ((int)(ld_acquire_sys(p) - target) < 0) {
    asm volatile("nanosleep.u32 100;");
    if (clock64() - t0 > (1ll << 35)) __trap();
  }
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void red_add_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---------------------------------------------------------------- layer state
struct Layer {
  cp_conv_desc d;
  cp_comm comm;
  // derived geometry
  int B, Bp;
  int C, H, W, R, S;      // input
  int Ho, Wo, Hp, Wp;     // conv output and pooled output
  int K, Kr, Kc, k0;      // all kernels, own count, own width, own first kernel
  int images;             // input kind
  int Kcol;               // im2col width (images)
  int Ktot;               // weight row length: Kcol or R*S*Cg
  Blocks in;              // input gather geometry (gather input)
  Blocks out;             // output gather geometry (pooled grid)
  // workspace carve-up (bytes)
  size_t ws_xcol, ws_z, ws_dy, ws_split, ws_dbpart, ws_total;
  size_t off_xcol, off_z, off_dy, off_split, off_dbpart;
  size_t off_x16, off_w16, off_dy16;   // bf16 operand copies (CP_MATH_BF16 only)
  size_t off_stamp;                    // 2 x u64 globaltimer stamps of the fused gather push (timing only)
  size_t off_c1w;                      // fused image-layer wgrad: per-CTA partial dW / db
  void* ws_last;                       // workspace of the last forward that recorded push stamps
  const void* xcol_key;                // images whose im2col rows the workspace holds (null: none)
  int dy_ready;           // epilogue-backward already computed for this step
  const void* dy_key[3];
  cudaEvent_t ev_compute, ev_comm;
  cudaEvent_t ev_bar_fork = nullptr, ev_bar = nullptr;   // deferred gather barrier (comm stream)
  cudaEvent_t ev_gfork = nullptr, ev_gjoin = nullptr;     // copy-engine gather on the comm stream
  cudaStream_t cs2 = nullptr;                              // second copy stream (split gather copies)
  cudaEvent_t ev_split[CP_MAX_RANKS] = {};
  // optional per-pass GEMM timing (conv_part_timing): events around the tensor-core kernel launch
  int timing;
  cudaEvent_t ev_t[5][2];   // timing: GEMM of pass 0/1/2, 3 copy-engine gather, 4 reduce-scatter transfer
  int ce_gather_timed = 0, rs_timed = 0;   // a window of kind 3 / 4 was recorded since timing was enabled

  // TMA descriptor cache lives in the TC module (opaque)
  void* tc_cache;
};

}  // namespace cp
