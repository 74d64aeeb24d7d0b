// kernels_simt.cu — FP32 SIMT reference convolutions (CP_MATH_FP32_SIMT), layout kernels
// (im2col, pack/unpack), the fused ReLU+max-pool epilogue used after SIMT convolutions,
// the epilogue backward (unpool + ReLU'), bias gradient, replicated head (FC, softmax
// cross-entropy) and SGD.  All reductions have a fixed order (deterministic, bitwise
// identical on every rank).
//
// Method cites: conv = valid cross-correlation, stride 1; ReLU + 2x2/2
// max-pool with first-max ties; FC + softmax loss (P:L275-276,
// S:L98-115); SGD.
#include <algorithm>

#include "kernels.cuh"

namespace cp {

static inline dim3 grid1d(int64_t n, int t) { return dim3((unsigned)((n + t - 1) / t)); }

// ============================================================== generic SIMT implicit GEMM
// C[m][n] = sum_k A(m,k) * B(k,n), fp32, k ascending per output (fixed order).
// 64x64 tile, 16-deep k slab, 256 threads, 4x4 outputs per thread.
template <bool A_KIN, bool B_KIN, class AL, class BL, class EP>
__global__ void __launch_bounds__(256) simt_gemm_kernel(int M, int N, int K, AL al, BL bl, EP ep) {
  __shared__ float As[16][68];
  __shared__ float Bs[16][68];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.x * 64, n0 = blockIdx.y * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += 16) {
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int i = tid + it * 256;
      const int kk = A_KIN ? (i & 15) : (i >> 6);
      const int mm = A_KIN ? (i >> 4) : (i & 63);
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? al(m, k) : 0.f;
    }
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int i = tid + it * 256;
      const int kk = B_KIN ? (i & 15) : (i >> 6);
      const int nn = B_KIN ? (i >> 4) : (i & 63);
      const int n = n0 + nn, k = k0 + kk;
      Bs[kk][nn] = (n < N && k < K) ? bl(k, n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) ep(m, n, acc[i][j]);
    }
}

template <bool A_KIN, bool B_KIN, class AL, class BL, class EP>
static int run_gemm(int M, int N, int K, AL al, BL bl, EP ep, cudaStream_t s) {
  if (M <= 0 || N <= 0) return CP_OK;
  dim3 grid(cdiv(M, 64), cdiv(N, 64));
  simt_gemm_kernel<A_KIN, B_KIN><<<grid, 256, 0, s>>>(M, N, K, al, bl, ep);
  CP_LAUNCHED();
  return CP_OK;
}

// value of a gather-layout input at spatial (h, w), image b, concatenated slot cs
__device__ __forceinline__ float gather_at(const float* __restrict__ x, const Blocks& g, int h, int w,
                                           int b, int cs) {
  const int rb = block_of_slot(g, cs);
  const int slot = cs - g.coff[rb];
  return x[g.start[rb] + ((int64_t)(h * g.W + w) * g.Bp + b) * g.kw[rb] + slot];
}

// ---------------------------------------------------------------- forward functors
struct FwdAGather {
  const float* x; Blocks g; int Wo, Bp, S, Cg;
  __device__ float operator()(int m, int k) const {
    const int b = m % Bp, pq = m / Bp, q = pq % Wo, p = pq / Wo;
    const int tap = k / Cg, cs = k - tap * Cg, r = tap / S, s = tap - r * S;
    return gather_at(x, g, p + r, q + s, b, cs);
  }
};
struct FwdAXcol {
  const float* xcol; int Kcol;
  __device__ float operator()(int m, int k) const { return xcol[(int64_t)m * Kcol + k]; }
};
struct FwdB {
  const float* w; int Kr, Ktot;
  __device__ float operator()(int k, int n) const { return n < Kr ? w[(int64_t)n * Ktot + k] : 0.f; }
};
struct FwdEp {
  float* z; const float* bias; int Kr, Kc;
  __device__ void operator()(int m, int n, float acc) const {
    z[(int64_t)m * Kc + n] = acc + ((bias && n < Kr) ? bias[n] : 0.f);
  }
};

int launch_fwd_simt(const Layer& L, const float* x, const float* xcol, const float* w, const float* b,
                    float* z, cudaStream_t s) {
  const int M = L.Ho * L.Wo * L.Bp, N = L.Kc, K = L.Ktot;
  FwdB bl{w, L.Kr, L.Ktot};
  FwdEp ep{z, L.d.bias ? b : nullptr, L.Kr, L.Kc};
  if (L.images) return run_gemm<true, true>(M, N, K, FwdAXcol{xcol, L.Kcol}, bl, ep, s);
  return run_gemm<true, true>(M, N, K, FwdAGather{x, L.in, L.Wo, L.Bp, L.S, L.in.Cg}, bl, ep, s);
}

// ---------------------------------------------------------------- dgrad functors
struct DgA {
  const float* dY; int Win, Ho, Wo, Bp, S, Kc;
  __device__ float operator()(int m, int k) const {
    const int b = m % Bp, hw = m / Bp, x = hw % Win, h = hw / Win;
    const int tap = k / Kc, kk = k - tap * Kc, r = tap / S, s = tap - r * S;
    const int p = h - r, q = x - s;
    if (p < 0 || p >= Ho || q < 0 || q >= Wo) return 0.f;
    return dY[((int64_t)(p * Wo + q) * Bp + b) * Kc + kk];
  }
};
struct DgB {
  const float* w; int Kr, Kc, Ktot, Cg;
  __device__ float operator()(int k, int n) const {
    const int tap = k / Kc, kk = k - tap * Kc;
    return kk < Kr ? w[(int64_t)kk * Ktot + tap * Cg + n] : 0.f;
  }
};
struct DgEp {
  float* dx; Blocks g;
  __device__ void operator()(int m, int n, float acc) const {
    const int rb = block_of_slot(g, n);
    dx[g.start[rb] + (int64_t)m * g.kw[rb] + (n - g.coff[rb])] = acc;
  }
};

// conv1 dgrad onto NCHW images (a14: API completeness, not on the training path)
__global__ void dgrad_images_kernel(const float* __restrict__ dY, const float* __restrict__ w, float* dx,
                                    int B, int C, int H, int W, int R, int S, int Ho, int Wo, int Bp,
                                    int Kr, int Kc, int Kcol) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)B * C * H * W) return;
  const int x = e % W, h = (e / W) % H, c = (e / ((int64_t)W * H)) % C, b = e / ((int64_t)W * H * C);
  float acc = 0.f;
  for (int kk = 0; kk < Kr; ++kk)
    for (int r = 0; r < R; ++r) {
      const int p = h - r;
      if (p < 0 || p >= Ho) continue;
      for (int s = 0; s < S; ++s) {
        const int q = x - s;
        if (q < 0 || q >= Wo) continue;
        acc = fmaf(dY[((int64_t)(p * Wo + q) * Bp + b) * Kc + kk], w[(int64_t)kk * Kcol + (r * S + s) * C + c], acc);
      }
    }
  dx[e] = acc;
}

int launch_dgrad_simt(const Layer& L, const float* dY, const float* w, float* dx, cudaStream_t s) {
  if (L.images) {
    const int64_t n = (int64_t)L.B * L.C * L.H * L.W;
    dgrad_images_kernel<<<grid1d(n, 256), 256, 0, s>>>(dY, w, dx, L.B, L.C, L.H, L.W, L.R, L.S, L.Ho, L.Wo,
                                                       L.Bp, L.Kr, L.Kc, L.Kcol);
    CP_LAUNCHED();
    return CP_OK;
  }
  const int M = L.H * L.W * L.Bp, N = L.in.Cg, K = L.R * L.S * L.Kc;
  return run_gemm<true, false>(M, N, K, DgA{dY, L.W, L.Ho, L.Wo, L.Bp, L.S, L.Kc},
                               DgB{w, L.Kr, L.Kc, L.Ktot, L.in.Cg}, DgEp{dx, L.in}, s);
}

// ---------------------------------------------------------------- wgrad functors
struct WgA {
  const float* dY; int Kc;
  __device__ float operator()(int m, int k) const { return dY[(int64_t)k * Kc + m]; }
};
struct WgBGather {
  const float* x; Blocks g; int Wo, Bp, S, Cg;
  __device__ float operator()(int k, int n) const {
    const int b = k % Bp, pq = k / Bp, q = pq % Wo, p = pq / Wo;
    const int tap = n / Cg, cs = n - tap * Cg, r = tap / S, s = tap - r * S;
    return gather_at(x, g, p + r, q + s, b, cs);
  }
};
struct WgBXcol {
  const float* xcol; int Kcol;
  __device__ float operator()(int k, int n) const { return xcol[(int64_t)k * Kcol + n]; }
};
struct WgEp {
  float* dw; int Kr, Ktot;
  __device__ void operator()(int m, int n, float acc) const {
    if (m < Kr) dw[(int64_t)m * Ktot + n] = acc;
  }
};

int launch_wgrad_simt(const Layer& L, const float* dY, const float* x, const float* xcol, float* dw,
                      cudaStream_t s) {
  const int M = L.Kr, N = L.Ktot, K = L.Ho * L.Wo * L.Bp;
  if (L.images)
    return run_gemm<false, false>(M, N, K, WgA{dY, L.Kc}, WgBXcol{xcol, L.Kcol}, WgEp{dw, L.Kr, L.Ktot}, s);
  return run_gemm<false, false>(M, N, K, WgA{dY, L.Kc}, WgBGather{x, L.in, L.Wo, L.Bp, L.S, L.in.Cg},
                                WgEp{dw, L.Kr, L.Ktot}, s);
}

// ============================================================== layout / elementwise
// im2col of the images for conv1: rows (p,q,b) of the output grid, columns (r,s,c) padded to Kcol.
// One thread per 4 consecutive columns (float4 store); reads are tiny and L2/L1-resident.
__global__ void im2col_kernel(const float* __restrict__ x, float* __restrict__ xcol, int B, int C, int H,
                              int W, int R, int S, int Wo, int Bp, int Kcol, int64_t total4, int round) {
  const int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e4 >= total4) return;
  const int kc4 = Kcol >> 2;
  const int col0 = (int)(e4 % kc4) * 4;
  const int m = (int)(e4 / kc4);
  const int b = m % Bp, pq = m / Bp, q = pq % Wo, p = pq / Wo;
  float v[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int col = col0 + t;
    float u = 0.f;
    if (b < B && col < R * S * C) {
      const int c = col % C, tap = col / C, r = tap / S, s = tap - r * S;
      u = __ldg(x + (((int64_t)b * C + c) * H + p + r) * W + q + s);
    }
    v[t] = round ? tf32_rna(u) : u;
  }
  reinterpret_cast<float4*>(xcol)[e4] = make_float4(v[0], v[1], v[2], v[3]);
}

int launch_im2col(const Layer& L, const float* x, float* xcol, bool round_tf32, cudaStream_t s) {
  const int64_t total4 = (int64_t)L.Ho * L.Wo * L.Bp * (L.Kcol / 4);
  im2col_kernel<<<grid1d(total4, 256), 256, 0, s>>>(x, xcol, L.B, L.C, L.H, L.W, L.R, L.S, L.Wo, L.Bp, L.Kcol,
                                                    total4, round_tf32 ? 1 : 0);
  CP_LAUNCHED();
  return CP_OK;
}

// Z own block [Ho][Wo][Bp][Kc] -> y own block [Hp][Wp][Bp][Kc] + argmax codes.
__global__ void relu_pool_kernel(const float* __restrict__ z, float* __restrict__ y, uint8_t* __restrict__ am,
                                 int Wo, int Wp, int Bp, int B, int Kr, int Kc, int64_t total, int relu,
                                 int pool, int round) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int slot = e % Kc;
  const int64_t rest = e / Kc;
  const int b = rest % Bp;
  const int64_t ij = rest / Bp;
  if (b >= B || slot >= Kr) {
    y[e] = 0.f;
    if (pool) am[e] = 0;
    return;
  }
  if (!pool) {
    float v = z[e];
    if (relu && !(v > 0.f)) v = 0.f;
    y[e] = round ? tf32_rna(v) : v;
    return;
  }
  const int j = ij % Wp, i = ij / Wp;
  float best = 0.f;
  int code = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int h = 2 * i + (t >> 1), w = 2 * j + (t & 1);
    float v = z[((int64_t)(h * Wo + w) * Bp + b) * Kc + slot];
    if (relu && !(v > 0.f)) v = 0.f;
    if (t == 0 || v > best) {
      best = v;
      code = t;
    }
  }
  y[e] = round ? tf32_rna(best) : best;
  am[e] = (uint8_t)code;
}

int launch_relu_pool(const Layer& L, const float* z, float* y_block, uint8_t* saved, bool round_tf32,
                     cudaStream_t s) {
  const int64_t total = (int64_t)L.Hp * L.Wp * L.Bp * L.Kc;
  relu_pool_kernel<<<grid1d(total, 256), 256, 0, s>>>(z, y_block, saved, L.Wo, L.Wp, L.Bp, L.B, L.Kr, L.Kc,
                                                      total, L.d.relu, L.d.pool, round_tf32 ? 1 : 0);
  CP_LAUNCHED();
  return CP_OK;
}

// Epilogue backward: dY[h][w][b][slot] = dy_pooled routed to the argmax position, times ReLU'
// (ReLU'(0)=0, reading R7).  One thread per (pooled position, image, 4 slots): it reads
// dy/y/codes once (float4 + 4 bytes) and writes the four window positions (4 x float4), so every
// pre-pool element is written exactly once with coalesced 16-byte stores.
__global__ void unpool_kernel(const float* __restrict__ dyp, const uint8_t* __restrict__ am,
                              const float* __restrict__ y, float* __restrict__ dY, int Wo, int Wp, int Bp,
                              int Kc, int64_t total4, int relu, int pool, int round) {
  const int64_t e4 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e4 >= total4) return;
  const int kc4 = Kc >> 2;
  const int slot = (int)(e4 % kc4) * 4;
  const int64_t rest = e4 / kc4;  // pooled row index (i*Wp + j)*Bp + b
  const int b = (int)(rest % Bp);
  const int ij = (int)(rest / Bp);
  const int64_t pe = rest * Kc + slot;
  const float4 g = *reinterpret_cast<const float4*>(dyp + pe);
  const float4 yy = *reinterpret_cast<const float4*>(y + pe);
  float gv[4] = {g.x, g.y, g.z, g.w};
  const float yv[4] = {yy.x, yy.y, yy.z, yy.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    if (relu && !(yv[t] > 0.f)) gv[t] = 0.f;
    if (round) gv[t] = tf32_rna(gv[t]);
  }
  if (!pool) {
    *reinterpret_cast<float4*>(dY + pe) = make_float4(gv[0], gv[1], gv[2], gv[3]);
    return;
  }
  const uint32_t codes = *reinterpret_cast<const uint32_t*>(am + pe);
  const int j = ij % Wp, i = ij / Wp;
#pragma unroll
  for (int pos = 0; pos < 4; ++pos) {
    const int h = 2 * i + (pos >> 1), w = 2 * j + (pos & 1);
    float o[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) o[t] = ((codes >> (8 * t)) & 0xFFu) == (uint32_t)pos ? gv[t] : 0.f;
    *reinterpret_cast<float4*>(dY + ((int64_t)(h * Wo + w) * Bp + b) * Kc + slot) = make_float4(o[0], o[1], o[2], o[3]);
  }
}

int launch_unpool(const Layer& L, const float* dy_block, const uint8_t* saved, const float* y_block, float* dY,
                  bool round_tf32, cudaStream_t s) {
  const int64_t total4 = (int64_t)L.Hp * L.Wp * L.Bp * (L.Kc / 4);
  if (total4 == 0) return CP_OK;
  unpool_kernel<<<grid1d(total4, 256), 256, 0, s>>>(dy_block, saved, y_block, dY, L.Wo, L.Wp, L.Bp, L.Kc, total4,
                                                    L.d.relu, L.d.pool, round_tf32 ? 1 : 0);
  CP_LAUNCHED();
  return CP_OK;
}

// db[slot] = sum over pooled rows of dy * [y > 0]: every pooled gradient reaches exactly one
// pre-pool position unless masked, so this equals sum of dY.  Two fixed-order phases.
constexpr int kBiasSplit = 64;
__global__ void bias_grad_partial(const float* __restrict__ dy, const float* __restrict__ y, float* part,
                                  int64_t rows, int Kc, int relu) {
  __shared__ float sm[8][33];
  const int slot = blockIdx.x * 32 + threadIdx.x;
  const int64_t per = (rows + kBiasSplit - 1) / kBiasSplit;
  const int64_t r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float acc = 0.f;
  if (slot < Kc)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) {
      const int64_t e = r * Kc + slot;
      const float g = dy[e];
      acc += (!relu || y[e] > 0.f) ? g : 0.f;
    }
  sm[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && slot < Kc) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += sm[i][threadIdx.x];
    part[(int64_t)blockIdx.y * Kc + slot] = t;
  }
}
__global__ void bias_grad_final(const float* __restrict__ part, float* db, int Kr, int Kc) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= Kr) return;
  float t = 0.f;
  for (int i = 0; i < kBiasSplit; ++i) t += part[(int64_t)i * Kc + slot];
  db[slot] = t;
}

int launch_bias_grad(const Layer& L, const float* dy_block, const float* y_block, float* db, float* part,
                     cudaStream_t s) {
  const int64_t rows = (int64_t)L.Hp * L.Wp * L.Bp;
  bias_grad_partial<<<dim3(cdiv(L.Kc, 32), kBiasSplit), dim3(32, 8), 0, s>>>(dy_block, y_block, part, rows,
                                                                             L.Kc, L.d.relu);
  CP_LAUNCHED();
  bias_grad_final<<<cdiv(L.Kr > 0 ? L.Kr : 1, 128), 128, 0, s>>>(part, db, L.Kr, L.Kc);
  CP_LAUNCHED();
  return CP_OK;
}

__global__ void fill_kernel(float* p, float v, int64_t n) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n) p[e] = v;
}
int launch_fill(float* p, float v, int64_t n, cudaStream_t s) {
  if (n <= 0) return CP_OK;
  fill_kernel<<<grid1d(n, 256), 256, 0, s>>>(p, v, n);
  CP_LAUNCHED();
  return CP_OK;
}

__global__ void random_fill_kernel(float* p, int64_t n, uint32_t seed, float scale) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  uint32_t h = (uint32_t)e * 2654435761u ^ seed;
  h ^= h >> 16; h *= 0x7feb352du; h ^= h >> 15; h *= 0x846ca68bu; h ^= h >> 16;
  p[e] = scale * ((float)(h >> 8) * (1.0f / 16777216.0f) * 2.f - 1.f);
}
int launch_random_fill(float* p, int64_t n, uint32_t seed, float scale, cudaStream_t s) {
  if (n <= 0) return CP_OK;
  random_fill_kernel<<<grid1d(n, 256), 256, 0, s>>>(p, n, seed, scale);
  CP_LAUNCHED();
  return CP_OK;
}

}  // namespace cp

// ============================================================== C-ABI boundary helpers
using namespace cp;

namespace {
__device__ __forceinline__ int block_of_elem(const Blocks& g, int64_t e) {
  int r = 0;
  while (r + 1 < g.n && e >= g.start[r + 1]) ++r;
  return r;
}

__global__ void pack_nchw_kernel(const float* __restrict__ x, float* __restrict__ out, Blocks g, int B, int C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= g.start[g.n]) return;
  const int r = block_of_elem(g, e);
  const int64_t l = e - g.start[r];
  const int slot = l % g.kw[r];
  const int64_t rest = l / g.kw[r];
  const int b = rest % g.Bp;
  const int64_t hw = rest / g.Bp;
  const int w = hw % g.W, h = hw / g.W;
  float v = 0.f;
  if (b < B && slot < g.kc[r]) v = x[(((int64_t)b * C + g.kb[r] + slot) * g.H + h) * g.W + w];
  out[e] = v;
}

__global__ void unpack_nchw_kernel(const float* __restrict__ gsrc, float* __restrict__ out, Blocks g, int B,
                                   int C) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)B * C * g.H * g.W) return;
  const int w = e % g.W, h = (e / g.W) % g.H;
  const int c = (e / ((int64_t)g.W * g.H)) % C, b = e / ((int64_t)g.W * g.H * C);
  int r = 0;
  while (r + 1 < g.n && c >= g.kb[r + 1]) ++r;
  // skip zero-count ranks that share a begin index
  while (r < g.n && c >= g.kb[r] + g.kc[r]) ++r;
  out[e] = gsrc[g.start[r] + ((int64_t)(h * g.W + w) * g.Bp + b) * g.kw[r] + (c - g.kb[r])];
}

__global__ void unpack_saved_kernel(const uint8_t* __restrict__ sv, uint8_t* __restrict__ out, int B, int Hp,
                                    int Wp, int Bp, int Kr, int Kc) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)B * Kr * Hp * Wp) return;
  const int j = e % Wp, i = (e / Wp) % Hp, kk = (e / ((int64_t)Wp * Hp)) % Kr, b = e / ((int64_t)Wp * Hp * Kr);
  out[e] = sv[((int64_t)(i * Wp + j) * Bp + b) * Kc + kk];
}

__global__ void pack_w_gather_kernel(const float* __restrict__ w, float* __restrict__ out, Blocks gin, int k0,
                                     int Kr, int C, int RS, int64_t total) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int Cg = gin.Cg;
  const int cs = e % Cg;
  const int tap = (e / Cg) % RS;
  const int kk = e / ((int64_t)Cg * RS);
  const int rb = block_of_slot(gin, cs);
  const int slot = cs - gin.coff[rb];
  float v = 0.f;
  if (slot < gin.kc[rb]) v = w[((int64_t)(k0 + kk) * C + gin.kb[rb] + slot) * RS + tap];
  out[e] = v;
  (void)Kr;
}

__global__ void unpack_w_gather_kernel(const float* __restrict__ wg, float* __restrict__ out, Blocks gin, int Kr,
                                       int C, int RS, int64_t total) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;  // total = Kr*C*RS, out KCRS rows
  const int tap = e % RS;
  const int c = (e / RS) % C;
  const int kk = e / ((int64_t)RS * C);
  int r = 0;
  while (r + 1 < gin.n && c >= gin.kb[r + 1]) ++r;
  while (r < gin.n && c >= gin.kb[r] + gin.kc[r]) ++r;
  out[e] = wg[((int64_t)kk * RS + tap) * gin.Cg + gin.coff[r] + (c - gin.kb[r])];
  (void)Kr;
}

__global__ void pack_w_images_kernel(const float* __restrict__ w, float* __restrict__ out, int k0, int C, int R,
                                     int S, int Kcol, int64_t total) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int col = e % Kcol;
  const int kk = e / Kcol;
  float v = 0.f;
  if (col < R * S * C) {
    const int c = col % C, tap = col / C;
    v = w[((int64_t)(k0 + kk) * C + c) * R * S + tap];
  }
  out[e] = v;
}

__global__ void unpack_w_images_kernel(const float* __restrict__ wg, float* __restrict__ out, int C, int R,
                                       int S, int Kcol, int64_t total) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int tap = e % (R * S);
  const int c = (e / (R * S)) % C;
  const int kk = e / ((int64_t)R * S * C);
  out[e] = wg[(int64_t)kk * Kcol + tap * C + c];
}

// ---------------------------------------------------------------- replicated head
// FC features in gather order: block r, position pos = h*Wp+w, slot; f' = Hp*Wp*coff[r] + pos*kw[r] + slot.
constexpr int kMaxO = 16;

// FC forward over the gather layout.  CTA = (rank block r, position pos, 128-slot chunk): the
// weight slice W[o][f(r,pos,chunk)] is staged in shared memory; thread (image b, slot half)
// streams 64 contiguous slots of x with float4 loads and accumulates all O logits.  The two
// halves combine by one shuffle; fc_fwd_reduce then adds the units in unit order (fixed order,
// bitwise identical on every rank).
constexpr int kFcChunk = 128;
__host__ __device__ inline int fc_nsc(const Blocks& g) {
  int m = 0;
  for (int r = 0; r < g.n; ++r) m = g.kw[r] > m ? g.kw[r] : m;
  return (m + kFcChunk - 1) / kFcChunk;
}

__global__ void __launch_bounds__(256) fc_fwd_partial(const float* __restrict__ x, const float* __restrict__ wg,
                                                      float* __restrict__ part, Blocks g, int B, int O, int PW,
                                                      int nsc) {
  __shared__ float4 ws[kMaxO][kFcChunk / 4];
  const int u = blockIdx.x;
  const int sc = u % nsc, rp = u / nsc;
  const int r = rp / PW, pos = rp % PW;
  const int kw = g.kw[r];
  const int s0 = sc * kFcChunk;
  const int64_t F = (int64_t)PW * g.Cg;
  const int64_t foff = (int64_t)PW * g.coff[r] + (int64_t)pos * kw + s0;
  for (int i = threadIdx.x; i < kMaxO * (kFcChunk / 4); i += blockDim.x) {
    const int o = i / (kFcChunk / 4), q4 = (i % (kFcChunk / 4)) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (o < O && s0 + q4 < kw) v = __ldg(reinterpret_cast<const float4*>(wg + o * F + foff + q4));
    ws[o][i % (kFcChunk / 4)] = v;
  }
  __syncthreads();
  const int b = blockIdx.y * 128 + (threadIdx.x >> 1), half = threadIdx.x & 1;
  float acc[kMaxO];
#pragma unroll
  for (int o = 0; o < kMaxO; ++o) acc[o] = 0.f;
  if (b < B) {
    const float* xr = x + g.start[r] + ((int64_t)pos * g.Bp + b) * kw + s0;
    const int n4 = min(kFcChunk, kw - s0) / 4;
#pragma unroll 4
    for (int q = half * (kFcChunk / 8); q < (half + 1) * (kFcChunk / 8); ++q) {
      if (q >= n4) break;
      const float4 xv = __ldg(reinterpret_cast<const float4*>(xr) + q);
#pragma unroll
      for (int o = 0; o < kMaxO; ++o) {
        if (o < O) {
          const float4 w = ws[o][q];
          acc[o] = fmaf(xv.x, w.x, fmaf(xv.y, w.y, fmaf(xv.z, w.z, fmaf(xv.w, w.w, acc[o]))));
        }
      }
    }
  }
#pragma unroll
  for (int o = 0; o < kMaxO; ++o) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], 1);
  if (half == 0 && b < g.Bp)
    for (int o = 0; o < O; ++o) part[((int64_t)u * g.Bp + b) * O + o] = acc[o];
}

// logits[b][o] = bias[o] + sum_u part[u][b][o]: one warp per (b, o); lanes take units in strides
// of 32 (ascending), then a fixed xor-shuffle tree — a fixed order, identical on every rank.
__global__ void fc_fwd_reduce(const float* __restrict__ part, const float* __restrict__ bfc, float* logits,
                              int U, int Bp, int B, int O) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (e >= B * O) return;
  const int b = e / O, o = e % O;
  float t = 0.f;
  for (int u = lane; u < U; u += 32) t += part[((int64_t)u * Bp + b) * O + o];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
  if (lane == 0) logits[e] = t + (bfc ? bfc[o] : 0.f);
}

__global__ void softmax_xent_kernel(const float* __restrict__ logits, const int* __restrict__ y, int B, int O,
                                    float* loss, float* dl) {
  extern __shared__ float terms[];
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const float* l = logits + (int64_t)b * O;
    float m = l[0];
    for (int o = 1; o < O; ++o) m = fmaxf(m, l[o]);
    float se = 0.f;
    for (int o = 0; o < O; ++o) se += expf(l[o] - m);
    const float lse = m + logf(se);
    const int lab = y[b];
    if (lab < 0 || lab >= O) {
      terms[b] = __int_as_float(0x7fc00000);  // NaN loss flags an out-of-range label
      continue;
    }
    terms[b] = lse - l[lab];
    for (int o = 0; o < O; ++o) dl[(int64_t)b * O + o] = (expf(l[o] - lse) - (o == lab ? 1.f : 0.f)) / (float)B;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int b = 0; b < B; ++b) t += terms[b];
    *loss = t / (float)B;
  }
}

// dA2 in gather layout: dx[(r,pos,b,slot)] = sum_o dlogits[b][o] * W[o][f(r,pos,slot)], zero for b >= B.
// Grid (r*PW + pos, ceil(Bp*kw/4 / 256)); one thread per 4 slots (float4).
__global__ void fc_bwd_dx(const float* __restrict__ dl, const float* __restrict__ wg, float* __restrict__ dx,
                          Blocks g, int B, int O, int PW) {
  const int rp = blockIdx.x;
  const int r = rp / PW, pos = rp % PW;
  const int kw = g.kw[r];
  const int kw4 = kw >> 2;
  const int e4 = blockIdx.y * blockDim.x + threadIdx.x;
  if (e4 >= g.Bp * kw4) return;
  const int b = e4 / kw4, slot = (e4 % kw4) * 4;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (b < B) {
    const int64_t F = (int64_t)PW * g.Cg;
    const int64_t f = (int64_t)PW * g.coff[r] + (int64_t)pos * kw + slot;
    for (int o = 0; o < O; ++o) {
      const float d = __ldg(dl + b * O + o);
      const float4 w = __ldg(reinterpret_cast<const float4*>(wg + o * F + f));
      acc.x = fmaf(d, w.x, acc.x); acc.y = fmaf(d, w.y, acc.y);
      acc.z = fmaf(d, w.z, acc.z); acc.w = fmaf(d, w.w, acc.w);
    }
  }
  *reinterpret_cast<float4*>(dx + g.start[r] + ((int64_t)pos * g.Bp + b) * kw + slot) = acc;
}

// dW_fc[o][f] = sum_b dlogits[b][o] * x(b, f): thread (4 features, batch quarter); the four
// quarters are added in order in shared memory (fixed order).
__global__ void __launch_bounds__(128) fc_bwd_dw(const float* __restrict__ dl, const float* __restrict__ x,
                                                 float* __restrict__ dwg, Blocks g, int B, int O, int PW) {
  __shared__ float4 red[3][32][kMaxO];
  const int64_t F = (int64_t)PW * g.Cg;
  const int64_t f = ((int64_t)blockIdx.x * 32 + threadIdx.x) * 4;
  const int qb = threadIdx.y;
  float acc[kMaxO][4];
#pragma unroll
  for (int o = 0; o < kMaxO; ++o)
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[o][t] = 0.f;
  if (f < F) {
    int r = 0;
    while (r + 1 < g.n && f >= (int64_t)PW * g.coff[r + 1]) ++r;
    const int64_t l = f - (int64_t)PW * g.coff[r];
    const int kw = g.kw[r];
    const int pos = (int)(l / kw), slot = (int)(l % kw);
    const float* xp = x + g.start[r] + (int64_t)pos * g.Bp * kw + slot;
    const int bq = (B + 3) / 4;
    const int b0 = qb * bq, b1 = min(B, b0 + bq);
    for (int b = b0; b < b1; ++b) {
      const float4 xv = __ldg(reinterpret_cast<const float4*>(xp + (int64_t)b * kw));
#pragma unroll
      for (int o = 0; o < kMaxO; ++o) {
        if (o < O) {
          const float d = __ldg(dl + b * O + o);
          acc[o][0] = fmaf(d, xv.x, acc[o][0]); acc[o][1] = fmaf(d, xv.y, acc[o][1]);
          acc[o][2] = fmaf(d, xv.z, acc[o][2]); acc[o][3] = fmaf(d, xv.w, acc[o][3]);
        }
      }
    }
  }
  if (qb > 0) {
#pragma unroll
    for (int o = 0; o < kMaxO; ++o) red[qb - 1][threadIdx.x][o] = make_float4(acc[o][0], acc[o][1], acc[o][2], acc[o][3]);
  }
  __syncthreads();
  if (qb == 0 && f < F) {
#pragma unroll
    for (int o = 0; o < kMaxO; ++o) {
      if (o >= O) continue;
      float4 t = make_float4(acc[o][0], acc[o][1], acc[o][2], acc[o][3]);
#pragma unroll
      for (int q = 1; q < 4; ++q) {
        const float4 u = red[q - 1][threadIdx.x][o];
        t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
      }
      *reinterpret_cast<float4*>(dwg + o * F + f) = t;
    }
  }
}

__global__ void fc_bwd_db(const float* __restrict__ dl, float* dbfc, int B, int O) {
  const int o = threadIdx.x;
  if (o >= O) return;
  float t = 0.f;
  for (int b = 0; b < B; ++b) t += dl[(int64_t)b * O + o];
  dbfc[o] = t;
}

__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t n, float lr) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n && ((reinterpret_cast<uintptr_t>(p + i) | reinterpret_cast<uintptr_t>(g + i)) & 15) == 0) {
    float4 a = *reinterpret_cast<float4*>(p + i);
    const float4 b = *reinterpret_cast<const float4*>(g + i);
    a.x -= lr * b.x; a.y -= lr * b.y; a.z -= lr * b.z; a.w -= lr * b.w;
    *reinterpret_cast<float4*>(p + i) = a;
  } else {
    for (int64_t j = i; j < n && j < i + 4; ++j) p[j] -= lr * g[j];
  }
}

__global__ void pack_fc_kernel(const float* __restrict__ w, float* __restrict__ out, Blocks g, int O, int C,
                               int64_t total) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int64_t PW = (int64_t)g.H * g.W;
  const int64_t FF = PW * g.Cg;
  const int o = e / FF;
  const int64_t f = e % FF;
  int r = 0;
  while (r + 1 < g.n && f >= PW * g.coff[r + 1]) ++r;
  const int64_t l = f - PW * g.coff[r];
  const int pos = l / g.kw[r], slot = l % g.kw[r];
  float v = 0.f;
  if (slot < g.kc[r]) v = w[((int64_t)o * C + g.kb[r] + slot) * PW + pos];
  out[e] = v;
  (void)O;
}

__global__ void unpack_fc_kernel(const float* __restrict__ wg, float* __restrict__ out, Blocks g, int C,
                                 int64_t total) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int64_t PW = (int64_t)g.H * g.W;
  const int pos = e % PW;
  const int c = (e / PW) % C;
  const int o = e / (PW * C);
  int r = 0;
  while (r + 1 < g.n && c >= g.kb[r + 1]) ++r;
  while (r < g.n && c >= g.kb[r] + g.kc[r]) ++r;
  out[e] = wg[(int64_t)o * PW * g.Cg + PW * g.coff[r] + (int64_t)pos * g.kw[r] + (c - g.kb[r])];
}

int check_part(const cp_partition* p) {
  if (!p) CP_FAIL(CP_ERR_ARG, "null partition");
  if (p->n_ranks < 1 || p->n_ranks > CP_MAX_RANKS) CP_FAIL(CP_ERR_CONFIG, "partition: n_ranks out of range");
  int b = 0;
  for (int r = 0; r < p->n_ranks; ++r) {
    if (p->k_begin[r] != b || p->k_count[r] < 0 || p->k_width[r] < p->k_count[r] || p->k_width[r] % 8)
      CP_FAIL(CP_ERR_CONFIG, "partition: ranges not contiguous or widths not multiples of 8 >= count");
    b += p->k_count[r];
  }
  if (b != p->num_k) CP_FAIL(CP_ERR_CONFIG, "partition: counts do not sum to num_k");
  return CP_OK;
}
}  // namespace

extern "C" {

int cp_pack_nchw(const float* x, int32_t B, int32_t C, int32_t H, int32_t W, const cp_partition* part, float* out,
                 void* stream) {
  CP_TRY(check_part(part));
  if (!x || !out) CP_FAIL(CP_ERR_ARG, "cp_pack_nchw: null pointer");
  if (part->num_k != C) CP_FAIL(CP_ERR_SHAPE, "cp_pack_nchw: C=" + std::to_string(C) + " vs partition num_k=" +
                                              std::to_string(part->num_k));
  Blocks g = make_blocks(*part, H, W, roundup(B, 32));
  pack_nchw_kernel<<<grid1d(g.start[g.n], 256), 256, 0, (cudaStream_t)stream>>>(x, out, g, B, C);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_unpack_nchw(const float* gsrc, int32_t B, int32_t C, int32_t H, int32_t W, const cp_partition* part,
                   float* out, void* stream) {
  CP_TRY(check_part(part));
  if (!gsrc || !out) CP_FAIL(CP_ERR_ARG, "cp_unpack_nchw: null pointer");
  if (part->num_k != C) CP_FAIL(CP_ERR_SHAPE, "cp_unpack_nchw: C vs partition num_k mismatch");
  Blocks g = make_blocks(*part, H, W, roundup(B, 32));
  unpack_nchw_kernel<<<grid1d((int64_t)B * C * H * W, 256), 256, 0, (cudaStream_t)stream>>>(gsrc, out, g, B, C);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_unpack_saved(const uint8_t* saved, int32_t B, int32_t Hp, int32_t Wp, const cp_partition* part,
                    int32_t rank, uint8_t* out, void* stream) {
  CP_TRY(check_part(part));
  if (!saved || !out) CP_FAIL(CP_ERR_ARG, "cp_unpack_saved: null pointer");
  if (rank < 0 || rank >= part->n_ranks) CP_FAIL(CP_ERR_ARG, "cp_unpack_saved: rank out of range");
  const int Kr = part->k_count[rank], Kc = part->k_width[rank];
  const int64_t n = (int64_t)B * Kr * Hp * Wp;
  if (n == 0) return CP_OK;
  unpack_saved_kernel<<<grid1d(n, 256), 256, 0, (cudaStream_t)stream>>>(saved, out, B, Hp, Wp, roundup(B, 32), Kr,
                                                                        Kc);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_pack_conv_weights(const cp_conv_desc* d, const float* w, float* out, void* stream) {
  if (!d || !w || !out) CP_FAIL(CP_ERR_ARG, "cp_pack_conv_weights: null pointer");
  CP_TRY(check_part(&d->out_part));
  const int k0 = d->out_part.k_begin[d->rank], Kr = d->out_part.k_count[d->rank];
  const int RS = d->k_h * d->k_w;
  cudaStream_t s = (cudaStream_t)stream;
  if (d->input_kind == CP_INPUT_IMAGES) {
    const int Kcol = roundup(RS * d->in_c, 8);
    const int64_t total = (int64_t)Kr * Kcol;
    if (total == 0) return CP_OK;
    pack_w_images_kernel<<<grid1d(total, 256), 256, 0, s>>>(w, out, k0, d->in_c, d->k_h, d->k_w, Kcol, total);
  } else {
    CP_TRY(check_part(&d->in_part));
    Blocks gin = make_blocks(d->in_part, 1, 1, 32);
    const int64_t total = (int64_t)Kr * RS * gin.Cg;
    if (total == 0) return CP_OK;
    pack_w_gather_kernel<<<grid1d(total, 256), 256, 0, s>>>(w, out, gin, k0, Kr, d->in_c, RS, total);
  }
  CP_LAUNCHED();
  return CP_OK;
}

int cp_unpack_conv_weights(const cp_conv_desc* d, const float* wg, float* out, void* stream) {
  if (!d || !wg || !out) CP_FAIL(CP_ERR_ARG, "cp_unpack_conv_weights: null pointer");
  CP_TRY(check_part(&d->out_part));
  const int Kr = d->out_part.k_count[d->rank];
  const int RS = d->k_h * d->k_w;
  const int64_t total = (int64_t)Kr * d->in_c * RS;
  if (total == 0) return CP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (d->input_kind == CP_INPUT_IMAGES) {
    unpack_w_images_kernel<<<grid1d(total, 256), 256, 0, s>>>(wg, out, d->in_c, d->k_h, d->k_w,
                                                              roundup(RS * d->in_c, 8), total);
  } else {
    CP_TRY(check_part(&d->in_part));
    Blocks gin = make_blocks(d->in_part, 1, 1, 32);
    unpack_w_gather_kernel<<<grid1d(total, 256), 256, 0, s>>>(wg, out, gin, Kr, d->in_c, RS, total);
  }
  CP_LAUNCHED();
  return CP_OK;
}

int cp_head_workspace_bytes(int32_t B, int32_t Hp, int32_t Wp, const cp_partition* part, int32_t O,
                            size_t* bytes) {
  CP_TRY(check_part(part));
  if (!bytes) CP_FAIL(CP_ERR_ARG, "null bytes");
  Blocks g = make_blocks(*part, Hp, Wp, roundup(B, 32));
  *bytes = (size_t)g.n * Hp * Wp * fc_nsc(g) * g.Bp * O * sizeof(float) + 256;
  return CP_OK;
}

int cp_pack_fc_weights(const float* wfc, int32_t O, int32_t Hp, int32_t Wp, const cp_partition* part, float* out,
                       void* stream) {
  CP_TRY(check_part(part));
  if (!wfc || !out) CP_FAIL(CP_ERR_ARG, "cp_pack_fc_weights: null pointer");
  // the FC weight rows [O][K*Hp*Wp] (NCHW flatten) are "images" of shape (O, K, Hp, Wp)
  // packed per row into gather feature order: reuse the activation pack with B=O, Bp irrelevant.
  Blocks g = make_blocks(*part, Hp, Wp, 32);
  const int64_t total = (int64_t)O * Hp * Wp * g.Cg;
  pack_fc_kernel<<<grid1d(total, 256), 256, 0, (cudaStream_t)stream>>>(wfc, out, g, O, part->num_k, total);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_unpack_fc_weights(const float* wg, int32_t O, int32_t Hp, int32_t Wp, const cp_partition* part, float* out,
                         void* stream) {
  CP_TRY(check_part(part));
  if (!wg || !out) CP_FAIL(CP_ERR_ARG, "cp_unpack_fc_weights: null pointer");
  Blocks g = make_blocks(*part, Hp, Wp, 32);
  const int64_t PW = (int64_t)Hp * Wp;
  const int64_t total = (int64_t)O * part->num_k * PW;
  unpack_fc_kernel<<<grid1d(total, 256), 256, 0, (cudaStream_t)stream>>>(wg, out, g, part->num_k, total);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_fc_forward(const float* x, int32_t B, int32_t Hp, int32_t Wp, const cp_partition* part, const float* wg,
                  const float* bfc, int32_t O, float* logits, void* ws, void* stream) {
  CP_TRY(check_part(part));
  if (!x || !wg || !logits || !ws) CP_FAIL(CP_ERR_ARG, "cp_fc_forward: null pointer");
  if (O < 1 || O > kMaxO) CP_FAIL(CP_ERR_UNSUPPORTED, "cp_fc_forward: O must be in [1,16]");
  Blocks g = make_blocks(*part, Hp, Wp, roundup(B, 32));
  const int PW = Hp * Wp, nsc = fc_nsc(g), U = g.n * PW * nsc;
  float* part_buf = (float*)ws;
  cudaStream_t s = (cudaStream_t)stream;
  fc_fwd_partial<<<dim3(U, (g.Bp + 127) / 128), 256, 0, s>>>(x, wg, part_buf, g, B, O, PW, nsc);
  CP_LAUNCHED();
  fc_fwd_reduce<<<cdiv((int64_t)B * O * 32, 256), 256, 0, s>>>(part_buf, bfc, logits, U, g.Bp, B, O);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_softmax_xent(const float* logits, const int32_t* labels, int32_t B, int32_t O, float* loss, float* dl,
                    void* stream) {
  if (!logits || !labels || !loss || !dl) CP_FAIL(CP_ERR_ARG, "cp_softmax_xent: null pointer");
  if (B < 1 || B > 8192 || O < 1) CP_FAIL(CP_ERR_SHAPE, "cp_softmax_xent: B must be in [1,8192]");
  softmax_xent_kernel<<<1, 256, B * sizeof(float), (cudaStream_t)stream>>>(logits, labels, B, O, loss, dl);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_fc_backward(const float* dl, const float* x, int32_t B, int32_t Hp, int32_t Wp, const cp_partition* part,
                   const float* wg, int32_t O, float* dx, float* dwg, float* dbfc, void* ws, void* stream) {
  CP_TRY(check_part(part));
  if (!dl || !x || !wg) CP_FAIL(CP_ERR_ARG, "cp_fc_backward: null pointer");
  if (O < 1 || O > kMaxO) CP_FAIL(CP_ERR_UNSUPPORTED, "cp_fc_backward: O must be in [1,16]");
  Blocks g = make_blocks(*part, Hp, Wp, roundup(B, 32));
  const int PW = Hp * Wp;
  cudaStream_t s = (cudaStream_t)stream;
  if (dx) {
    int maxkw = 0;
    for (int r = 0; r < g.n; ++r) maxkw = std::max(maxkw, g.kw[r]);
    fc_bwd_dx<<<dim3(g.n * PW, cdiv((int64_t)g.Bp * (maxkw / 4), 256)), 256, 0, s>>>(dl, wg, dx, g, B, O, PW);
    CP_LAUNCHED();
  }
  if (dwg) {
    fc_bwd_dw<<<grid1d((int64_t)PW * g.Cg / 4, 32), dim3(32, 4), 0, s>>>(dl, x, dwg, g, B, O, PW);
    CP_LAUNCHED();
  }
  if (dbfc) {
    fc_bwd_db<<<1, 32, 0, s>>>(dl, dbfc, B, O);
    CP_LAUNCHED();
  }
  (void)ws;
  return CP_OK;
}

int cp_sgd(float* p, const float* g, int64_t n, float lr, void* stream) {
  if (n == 0) return CP_OK;
  if (!p || !g || n < 0) CP_FAIL(CP_ERR_ARG, "cp_sgd: bad arguments");
  sgd_kernel<<<grid1d((n + 3) / 4, 256), 256, 0, (cudaStream_t)stream>>>(p, g, n, lr);
  CP_LAUNCHED();
  return CP_OK;
}

}  // extern "C"
