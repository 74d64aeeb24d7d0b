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

#include <cuda_bf16.h>

#include "kernels.cuh"

namespace cp {

static inline dim3 grid1d(int64_t n, int t) { return dim3((unsigned)((n + t - 1) / t)); }
static int num_sms_simt() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

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
// One block per (output row p, nimg images).  Load phase: input rows p..p+R-1 of every channel are
// R*W contiguous floats per (image, channel) - copied into shared memory coalesced (TF32-rounded
// when the consumer is the tensor-core path).  Write phase: every output pixel q of the row, the
// nimg x Kcol floats of xcol at ((p*Wo + q)*Bp + b0)*Kcol are contiguous - float4 stores, values
// picked from shared memory through a column -> offset table.  The output stays in L2.
constexpr int kIm2colMaxK = 256;
constexpr int kIm2colMaxBC = 1024;   // (image, channel) pairs per block
__global__ void __launch_bounds__(256) im2col_kernel(const float* __restrict__ x, float* __restrict__ xcol, int B,
                                                     int C, int H, int W, int R, int S, int Wo, int Bp, int Kcol,
                                                     int nimg, int round) {
  extern __shared__ float xs[];                 // [nimg][C][R][W]
  __shared__ int tab[kIm2colMaxK];              // column -> offset within one image's rows, -1 = padding
  const int p = blockIdx.x, b0 = blockIdx.y * nimg;
  const int RW = R * W, CRW = C * RW, RSC = R * S * C;
  const int nt = blockDim.x * blockDim.y, tid = threadIdx.y * blockDim.x + threadIdx.x;
  for (int col = tid; col < Kcol; col += nt) {
    int o = -1;
    if (col < RSC) {
      const int c = col % C, tap = col / C, r = tap / S, sx = tap - r * S;
      o = c * RW + r * W + sx;
    }
    tab[col] = o;
  }
  // load: (image, channel) pairs outer, the pair's R*W contiguous floats inner; row bases from a
  // table, 8 independent loads in flight per thread (latency, not bandwidth, bounds this phase)
  __shared__ long long base[kIm2colMaxBC];
  const int nbc = nimg * C;
  for (int bc = tid; bc < nbc; bc += nt) {
    const int bl = bc / C, c = bc - bl * C, b = b0 + bl;
    base[bc] = b < B ? (((long long)b * C + c) * H + p) * W : -1;
  }
  __syncthreads();
  if (RW <= nt) {
    const int k = tid;
    if (k < RW)
      for (int bc0 = 0; bc0 < nbc; bc0 += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int bc = bc0 + u;
          v[u] = (bc < nbc && base[bc] >= 0) ? __ldg(x + base[bc] + k) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (bc0 + u < nbc) xs[(bc0 + u) * RW + k] = round ? tf32_rna(v[u]) : v[u];
      }
  } else {
    for (int bc = 0; bc < nbc; ++bc)
      for (int k = tid; k < RW; k += nt) {
        const float u = base[bc] >= 0 ? __ldg(x + base[bc] + k) : 0.f;
        xs[bc * RW + k] = round ? tf32_rna(u) : u;
      }
  }
  __syncthreads();
  // write: thread x = fixed float4 column group of the pixel's nimg x Kcol floats (table lookups
  // hoisted), thread y strides the output pixels q
  const int e = threadIdx.x;                    // blockDim.x = nimg * Kcol / 4
  const int bl = (4 * e) / Kcol, col0 = 4 * e - bl * Kcol;
  int off[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) off[t] = tab[col0 + t];
  const float* src = xs + bl * CRW;
  float4* dst = reinterpret_cast<float4*>(xcol + ((int64_t)p * Wo * Bp + b0) * Kcol) + e;
  const int64_t qstride4 = (int64_t)Bp * Kcol / 4;
  for (int q = threadIdx.y; q < Wo; q += blockDim.y) {
    float v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) v[t] = off[t] >= 0 ? src[off[t] + q] : 0.f;
    dst[q * qstride4] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

int launch_im2col(const Layer& L, const float* x, float* xcol, bool round_tf32, cudaStream_t s) {
  const size_t per_img = (size_t)L.C * L.R * L.W * 4;
  // nimg images per block: the pixel row of nimg x Kcol floats is one float4 per thread (<= 256)
  int nimg = 8;
  while (nimg > 1 && ((size_t)nimg * per_img > 48 * 1024 || nimg * L.Kcol / 4 > 256)) nimg >>= 1;
  if (L.Kcol > kIm2colMaxK || (size_t)nimg * per_img > 48 * 1024 || nimg * L.Kcol / 4 > 256 || nimg * L.C > kIm2colMaxBC ||
      (int64_t)L.B * L.C * L.H * L.W >= (1ll << 31))
    CP_FAIL(CP_ERR_UNSUPPORTED, "im2col: image layer too large (Kcol > 256 or C*R*W*4 > 48 KB)");
  const int bx = nimg * L.Kcol / 4, by = std::max(1, 256 / bx);
  dim3 grid((unsigned)L.Ho, (unsigned)(L.Bp / nimg));
  im2col_kernel<<<grid, dim3(bx, by), nimg * per_img, s>>>(x, xcol, L.B, L.C, L.H, L.W, L.R, L.S, L.Wo, L.Bp,
                                                           L.Kcol, nimg, round_tf32 ? 1 : 0);
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
// Epilogue backward of the own block: dY (pre-pool grid) = the pooled gradient routed to
// the argmax position of its window, masked by ReLU' (y > 0), zero elsewhere; TF32-rounded for the
// tensor-core passes.  Fused: the bias gradient db[slot] = sum over pooled rows of dy * [y > 0]
// (every unmasked pooled gradient reaches exactly one pre-pool position, so this is sum dY).
// Block (32 float4 columns, 8 rows) on a contiguous row range; per-block column sums combine the
// 8 row lanes in fixed order -> part[split][slot]; bias_grad_final adds the splits in order.
__global__ void __launch_bounds__(256) unpool_kernel(const float* __restrict__ dyp, const uint8_t* __restrict__ am,
                                                     const float* __restrict__ y, float* __restrict__ dY,
                                                     float* __restrict__ part, int Wo, int Wp, int Bp, int Kc,
                                                     int rows, int per, int relu, int pool, int round) {
  __shared__ float4 red[8][32];
  const int kc4 = Kc >> 2;
  const int c4 = blockIdx.x * 32 + threadIdx.x;
  const int r0 = blockIdx.y * per, r1 = min(rows, r0 + per);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (c4 < kc4) {
    const int slot = c4 * 4;
    for (int rest = r0 + threadIdx.y; rest < r1; rest += 8) {   // pooled row (i*Wp + j)*Bp + b
      const int64_t pe = (int64_t)rest * Kc + slot;
      const float4 g = *reinterpret_cast<const float4*>(dyp + pe);
      const float4 yy = *reinterpret_cast<const float4*>(y + pe);
      float gv[4] = {g.x, g.y, g.z, g.w};
      const float yv[4] = {yy.x, yy.y, yy.z, yy.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (relu && !(yv[t] > 0.f)) gv[t] = 0.f;
      acc.x += gv[0]; acc.y += gv[1]; acc.z += gv[2]; acc.w += gv[3];
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (round) gv[t] = tf32_rna(gv[t]);
      if (!pool) {
        *reinterpret_cast<float4*>(dY + pe) = make_float4(gv[0], gv[1], gv[2], gv[3]);
        continue;
      }
      const uint32_t codes = *reinterpret_cast<const uint32_t*>(am + pe);
      const int b = rest % Bp, ij = rest / Bp;
      const int j = ij % Wp, i = ij / Wp;
#pragma unroll
      for (int pos = 0; pos < 4; ++pos) {
        const int h = 2 * i + (pos >> 1), w = 2 * j + (pos & 1);
        float o[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) o[t] = ((codes >> (8 * t)) & 0xFFu) == (uint32_t)pos ? gv[t] : 0.f;
        *reinterpret_cast<float4*>(dY + ((int64_t)(h * Wo + w) * Bp + b) * Kc + slot) =
            make_float4(o[0], o[1], o[2], o[3]);
      }
    }
  }
  if (!part) return;
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c4 < kc4) {
    float4 t = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      const float4 u = red[k][threadIdx.x];
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    reinterpret_cast<float4*>(part + (int64_t)blockIdx.y * Kc)[c4] = t;
  }
}

// number of row splits of the unpool grid (also the number of bias partials)
static int unpool_splits(const Layer& L) {
  const int rows = L.Hp * L.Wp * L.Bp;
  const int cb = cdiv(L.Kc / 4, 32);
  int ns = cdiv(4 * 148, cb);
  ns = std::min(ns, kBiasSplitMax);
  ns = std::min(ns, std::max(1, rows / 8));
  return std::max(ns, 1);
}

int launch_unpool(const Layer& L, const float* dy_block, const uint8_t* saved, const float* y_block, float* dY,
                  float* bias_part, bool round_tf32, cudaStream_t s) {
  if (L.Kc == 0) return CP_OK;
  const int rows = L.Hp * L.Wp * L.Bp;
  const int ns = unpool_splits(L);
  const int per = cdiv(rows, ns);
  unpool_kernel<<<dim3(cdiv(L.Kc / 4, 32), ns), dim3(32, 8), 0, s>>>(
      dy_block, saved, y_block, dY, bias_part, L.Wo, L.Wp, L.Bp, L.Kc, rows, per, L.d.relu, L.d.pool,
      round_tf32 ? 1 : 0);
  CP_LAUNCHED();
  return CP_OK;
}

// db[slot] = sum of the unpool kernel's bias partials, splits added in ascending order:
// block (32 slots, 8 split lanes), lanes combined in fixed order.
__global__ void __launch_bounds__(256) bias_grad_final(const float* __restrict__ part, float* db, int ns, int Kr,
                                                       int Kc, float* sgd_b, float lr) {
  __shared__ float red[8][33];
  const int slot = blockIdx.x * 32 + threadIdx.x;
  const int per = (ns + 7) / 8;
  const int s0 = threadIdx.y * per, s1 = min(ns, s0 + per);
  float t = 0.f;
  if (slot < Kr) {
    // loads batched (all of a lane's when <= 32: 7 / 25 splits per lane at P=1 / 4; else 8 at a time),
    // added in the same ascending order
    int i = s0;
    if (s1 - s0 <= 32) {
      float v[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) v[u] = s0 + u < s1 ? part[(int64_t)(s0 + u) * Kc + slot] : 0.f;
#pragma unroll
      for (int u = 0; u < 32; ++u)
        if (s0 + u < s1) t += v[u];
      i = s1;
    }
    for (; i + 8 <= s1; i += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = part[(int64_t)(i + u) * Kc + slot];
#pragma unroll
      for (int u = 0; u < 8; ++u) t += v[u];
    }
    for (; i < s1; ++i) t += part[(int64_t)i * Kc + slot];
  }
  red[threadIdx.y][threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.y == 0 && slot < Kr) {
    float u = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < 8; ++k) u += red[k][threadIdx.x];
    db[slot] = u;
    if (sgd_b) sgd_b[slot] = fmaf(-lr, u, sgd_b[slot]);   // fused SGD of the own biases
  }
}

int launch_bias_grad(const Layer& L, float* db, const float* part, cudaStream_t s, float* sgd_b, float lr) {
  if (L.Kr == 0) return CP_OK;
  bias_grad_final<<<cdiv(L.Kr, 32), dim3(32, 8), 0, s>>>(part, db, unpool_splits(L), L.Kr, L.Kc, sgd_b, lr);
  CP_LAUNCHED();
  return CP_OK;
}

__global__ void to_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst, int64_t n) {
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += (int64_t)gridDim.x * blockDim.x * 4) {
    if (i + 3 < n) {
      const float4 v = *reinterpret_cast<const float4*>(src + i);
      __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
      reinterpret_cast<__nv_bfloat162*>(dst + i)[0] = lo;
      reinterpret_cast<__nv_bfloat162*>(dst + i)[1] = hi;
    } else {
      for (int64_t j = i; j < n; ++j) dst[j] = __float2bfloat16_rn(src[j]);
    }
  }
}
int launch_to_bf16(const float* src, void* dst, int64_t n, cudaStream_t s) {
  if (n <= 0) return CP_OK;
  const int blocks = (int)std::min<int64_t>((n / 4 + 255) / 256 + 1, 148 * 16);
  to_bf16_kernel<<<blocks, 256, 0, s>>>(src, reinterpret_cast<__nv_bfloat16*>(dst), n);
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

// fused reduce-scatter epilogue: out[e] = sum_{q ascending} slots[q*slot_stride + e] (float4)
__global__ void sum_slots_kernel(const float* __restrict__ slots, int64_t slot_stride, int n_slots,
                                 float* __restrict__ out, int64_t n4) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  float4 acc = reinterpret_cast<const float4*>(slots)[i];
  for (int q = 1; q < n_slots; ++q) {
    const float4 v = reinterpret_cast<const float4*>(slots + q * slot_stride)[i];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  reinterpret_cast<float4*>(out)[i] = acc;
}
int launch_sum_slots(const float* slots, int64_t slot_stride, int n_slots, float* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return CP_OK;
  if ((n | slot_stride) & 3) CP_FAIL(CP_ERR_UNSUPPORTED, "sum_slots: sizes not multiples of 4");
  sum_slots_kernel<<<grid1d(n / 4, 256), 256, 0, s>>>(slots, slot_stride, n_slots, out, n / 4);
  CP_LAUNCHED();
  return CP_OK;
}

// pull reduce-scatter: out[e] = sum_{r ascending} src[r][e] (float4; src[r] = rank r's partial of the
// own block, read from its copy over NVLink).  Every rank's load of an element is issued before the sum
// (NVLink read latency); in place when out == src[self] (the same thread reads, then writes).
struct SrcPtrs {
  const float* p[CP_MAX_RANKS];
};
__global__ void __launch_bounds__(256) sum_peer_blocks_kernel(SrcPtrs src, int n_src, float* out, int64_t n4) {
  // one float4 per thread over a full grid: beside the concurrent wgrad the sum needs many resident
  // warps to finish in time (a 32-block grid-stride version left 53-59 us of dX wait at N=2)
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= n4) return;
  float4 v[CP_MAX_RANKS];
#pragma unroll
  for (int r = 0; r < CP_MAX_RANKS; ++r)
    if (r < n_src) v[r] = reinterpret_cast<const float4*>(src.p[r])[i];
  float4 a = v[0];
#pragma unroll
  for (int r = 1; r < CP_MAX_RANKS; ++r)
    if (r < n_src) {
      a.x += v[r].x; a.y += v[r].y; a.z += v[r].z; a.w += v[r].w;
    }
  reinterpret_cast<float4*>(out)[i] = a;
}
int launch_sum_peer_blocks(const float* const* src, int n_src, float* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return CP_OK;
  if (n & 3) CP_FAIL(CP_ERR_UNSUPPORTED, "sum_peer_blocks: size not a multiple of 4");
  SrcPtrs sp{};
  for (int r = 0; r < n_src; ++r) {
    if (reinterpret_cast<uintptr_t>(src[r]) & 15) CP_FAIL(CP_ERR_UNSUPPORTED, "sum_peer_blocks: unaligned block");
    sp.p[r] = src[r];
  }
  sum_peer_blocks_kernel<<<(unsigned)((n / 4 + 255) / 256), 256, 0, s>>>(sp, n_src, out, n / 4);
  CP_LAUNCHED();
  return CP_OK;
}

struct FlagPtrs {
  uint32_t* f[CP_MAX_RANKS];
};
// Runs after the storing kernel (stream order); thread k releases peer k's flag (a system-scope release
// orders everything before it, the previous kernel's stores included) - the releases run in parallel
// instead of one system fence after another.
__global__ void signal_peers_kernel(FlagPtrs fp, int n, int slot) {
  if ((int)threadIdx.x < n) st_release_sys(fp.f[threadIdx.x] + slot, 1u);
}
__global__ void wait_flags_kernel(const uint32_t* flags, int n, int self, uint32_t target) {
  for (int r = 0; r < n; ++r)
    if (r != self) wait_flag_sys(flags + r, target);
}

int launch_signal_peers(uint32_t* const* peer_flags, int n, int slot, cudaStream_t s) {
  if (n <= 0) return CP_OK;
  FlagPtrs fp{};
  for (int k = 0; k < n; ++k) fp.f[k] = peer_flags[k];
  signal_peers_kernel<<<1, 32, 0, s>>>(fp, n, slot);
  CP_LAUNCHED();
  return CP_OK;
}

int launch_wait_flags(const uint32_t* flags, int n, int self, cudaStream_t s, bool chunks) {
  if (n <= 1) return CP_OK;
  wait_flags_kernel<<<1, 1, 0, s>>>(flags, n, self, chunks ? (uint32_t)kGatherChunks : 1u);
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
constexpr int kMaxO = kHeadMaxO;

// FC forward over the gather layout (logits = W x + b).  CTA = (rank block r, position pos,
// 64-slot chunk) x 128-image chunk: the x tile [128 images][64 slots] and the weight slice
// W[o][f(r,pos,chunk)] are staged in shared memory with coalesced float4 loads; thread (image b,
// half) accumulates all O logits over 32 of the slots, the halves combine by one shuffle, and
// fc_fwd_reduce adds the units in unit order (fixed order, bitwise identical on every rank).
constexpr int kFcChunk = 64;
constexpr int kFcLd = 72;     // x tile row stride (floats): conflict-free float4 reads by (b, half)
__host__ __device__ inline int fc_nsc(const Blocks& g) {
  int m = 0;
  for (int r = 0; r < g.n; ++r) m = g.kw[r] > m ? g.kw[r] : m;
  return (m + kFcChunk - 1) / kFcChunk;
}

template <int OO>   // compile-time class bound (10 for CIFAR's 10 classes, else kMaxO)
__global__ void __launch_bounds__(256) fc_fwd_partial(const float* __restrict__ x, const float* __restrict__ wg,
                                                      float* __restrict__ part, Blocks g, int B, int O, int PW,
                                                      int nsc) {
  __shared__ __align__(16) float xs[128 * kFcLd];
  __shared__ float4 ws[kMaxO][kFcChunk / 4];
  const int u = blockIdx.x;
  const int sc = u % nsc, rp = u / nsc;
  const int r = rp / PW, pos = rp % PW;
  const int kw = g.kw[r];
  const int s0 = sc * kFcChunk;
  const int b0 = blockIdx.y * 128;
  const int64_t F = (int64_t)PW * g.Cg;
  const int64_t foff = (int64_t)PW * g.coff[r] + (int64_t)pos * kw + s0;
  for (int i = threadIdx.x; i < kMaxO * (kFcChunk / 4); i += blockDim.x) {
    const int o = i / (kFcChunk / 4), q4 = (i % (kFcChunk / 4)) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (o < O && s0 + q4 < kw) v = __ldg(reinterpret_cast<const float4*>(wg + o * F + foff + q4));
    ws[o][i % (kFcChunk / 4)] = v;
  }
  const float* xb = x + g.start[r] + (int64_t)pos * g.Bp * kw + s0;
  {  // 128 x 16 float4: 8 independent loads in flight per thread (blockDim 256)
    float4 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = threadIdx.x + k * 256, row = i >> 4, q = i & 15, b = b0 + row;
      v[k] = (b < B && s0 + 4 * q < kw) ? __ldg(reinterpret_cast<const float4*>(xb + (int64_t)b * kw) + q)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = threadIdx.x + k * 256;
      *reinterpret_cast<float4*>(xs + (i >> 4) * kFcLd + 4 * (i & 15)) = v[k];
    }
  }
  __syncthreads();
  const int bl = threadIdx.x >> 1, half = threadIdx.x & 1;
  float acc[OO];
#pragma unroll
  for (int o = 0; o < OO; ++o) acc[o] = 0.f;
#pragma unroll
  for (int k = 0; k < kFcChunk / 8; ++k) {
    const int q = 2 * k + half;
    const float4 xv = *reinterpret_cast<const float4*>(xs + bl * kFcLd + 4 * q);
#pragma unroll
    for (int o = 0; o < OO; ++o) {
      if (o < O) {
        const float4 w = ws[o][q];
        acc[o] = fmaf(xv.x, w.x, fmaf(xv.y, w.y, fmaf(xv.z, w.z, fmaf(xv.w, w.w, acc[o]))));
      }
    }
  }
#pragma unroll
  for (int o = 0; o < OO; ++o) acc[o] += __shfl_xor_sync(0xffffffffu, acc[o], 1);
  const int b = b0 + bl;
  if (half == 0 && b < g.Bp)
    for (int o = 0; o < O; ++o) part[((int64_t)u * g.Bp + b) * O + o] = acc[o];
}

// logits[b][o] = bias[o] + sum_u part[u][b][o].  Block (32 consecutive (b,o) elements, 32 unit
// lanes): lane y adds units y*per.. in ascending order (coalesced rows of part), the 32 lane sums
// combine in fixed order - identical on every rank.
__global__ void __launch_bounds__(1024) fc_fwd_reduce(const float* __restrict__ part, const float* __restrict__ bfc,
                                                      float* logits, int U, int Bp, int B, int O) {
  __shared__ float red[32][33];
  const int e = blockIdx.x * 32 + threadIdx.x;
  const int per = (U + 31) / 32;
  const int u0 = threadIdx.y * per, u1 = min(U, u0 + per);
  float t = 0.f;
  if (e < B * O) {
    int u = u0;   // loads batched (all of them when <= 24 per lane: 600 units at P=1), added in ascending unit order
    if (u1 - u0 <= 24) {
      float v[24];
#pragma unroll
      for (int q = 0; q < 24; ++q) v[q] = u0 + q < u1 ? part[(int64_t)(u0 + q) * Bp * O + e] : 0.f;
#pragma unroll
      for (int q = 0; q < 24; ++q)
        if (u0 + q < u1) t += v[q];
      u = u1;
    }
    for (; u + 8 <= u1; u += 8) {
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = part[(int64_t)(u + q) * Bp * O + e];
#pragma unroll
      for (int q = 0; q < 8; ++q) t += v[q];
    }
    for (; u < u1; ++u) t += part[(int64_t)u * Bp * O + e];
  }
  red[threadIdx.y][threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.y == 0 && e < B * O) {
    float v = red[0][threadIdx.x];
    for (int k = 1; k < 32; ++k) v += red[k][threadIdx.x];
    logits[e] = v + (bfc ? bfc[e % O] : 0.f);
  }
}

// softmax cross-entropy: loss = mean_b (logsumexp(l_b) - l_b[y_b]),
// dlogits = (softmax - onehot) / B.  One block; the loss sum is a fixed-order tree.
__global__ void __launch_bounds__(256) softmax_xent_kernel(const float* __restrict__ logits, const int* __restrict__ y,
                                                           int B, int O, float* loss, float* dl) {
  __shared__ float wsum[8];
  softmax_xent_block(logits, y, B, O, loss, dl, wsum);
}

// FC backward, one CTA column per gather-layout feature f = (rank block r, position pos, slot) (S:L98-115,
// chain rule through logits = W x + b):
//   dx[b][f] = sum_o dlogits[b][o] * W[o][f]      (stored in the gathered input's layout), and
//   dW[o][f] = sum_b dlogits[b][o] * x[b][f]      (fixed order: image groups ascending, within a group
//                                                  images ascending; identical on all ranks).
// CTA = 64 features x 8 image groups (512 threads): thread (f, g) handles images g, g+8, ... with 8 loads
// of x in flight (the load latency, not bandwidth, bounded the one-thread-per-feature version); its W
// column sits in registers, dlogits rows in shared memory (broadcast reads); the 8 groups' dW partials
// combine through shared memory.  CTA 0 also writes dbfc = sum_b dlogits.
// features x image groups per CTA: 8 groups (512 threads) when the grid fits on the SMs in one wave,
// else 4 (256 threads, twice as many resident CTAs: the paper net's 37,600 features at P=1 run in one
// wave, 28.7 -> 20.5 us; profiles/r02_head_variants.jsonl)
constexpr int kFcF = 64;
constexpr int kFcRows = 256;         // images per shared-memory dlogits chunk
template <int OO, int kFcG>
__global__ void __launch_bounds__(kFcF * kFcG) fc_bwd_cols(const float* __restrict__ dl, const float* __restrict__ x,
                                                          const float* __restrict__ wg, float* __restrict__ dx,
                                                          float* __restrict__ dwg, float* __restrict__ dbfc, Blocks g,
                                                          int B, int O, int PW, int64_t F) {
  __shared__ __align__(16) float dls[kFcRows][OO];
  __shared__ float red[kFcG][OO][kFcF];
  const int tx = threadIdx.x, ig = threadIdx.y, tid = ig * kFcF + tx;
  const int64_t f = (int64_t)blockIdx.x * kFcF + tx;
  if (dbfc && blockIdx.x == 0) {
    const int w = tid >> 5, lane = tid & 31;
    for (int o = w; o < O; o += kFcF * kFcG / 32) {
      float t = 0.f;
      for (int b = lane; b < B; b += 32) t += dl[(int64_t)b * O + o];
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) t += __shfl_xor_sync(0xffffffffu, t, d);
      if (lane == 0) dbfc[o] = t;
    }
  }
  // feature f -> (block r, position, slot)
  const bool valid = f < F;
  int r = 0;
  while (r + 1 < g.n && f >= (int64_t)PW * g.coff[r + 1]) ++r;
  const int64_t rem = valid ? f - (int64_t)PW * g.coff[r] : 0;
  const int kw = g.kw[r] > 0 ? g.kw[r] : 1;
  const int pos = (int)(rem / kw), slot = (int)(rem - (int64_t)pos * kw);
  const int64_t xo = g.start[r] + (int64_t)pos * g.Bp * kw + slot;
  float w[OO], acc[OO];
#pragma unroll
  for (int o = 0; o < OO; ++o) {
    w[o] = (valid && o < O) ? __ldg(wg + o * F + f) : 0.f;
    acc[o] = 0.f;
  }
  for (int b0 = 0; b0 < g.Bp; b0 += kFcRows) {
    const int nb = min(kFcRows, g.Bp - b0);
    __syncthreads();
    for (int i = tid; i < nb * OO; i += kFcF * kFcG) {
      const int row = i / OO, o = i - row * OO;
      dls[row][o] = (b0 + row < B && o < O) ? __ldg(dl + (int64_t)(b0 + row) * O + o) : 0.f;
    }
    __syncthreads();
    if (!valid) continue;
    for (int bb = ig; bb < nb; bb += 8 * kFcG) {
      float xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = bb + u * kFcG;
        xv[u] = b < nb ? __ldg(x + xo + (int64_t)(b0 + b) * kw) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int b = bb + u * kFcG;
        if (b >= nb) break;
        float dxv = 0.f;
#pragma unroll
        for (int o = 0; o < OO; ++o) {
          const float d = dls[b][o];
          dxv = fmaf(d, w[o], dxv);
          acc[o] = fmaf(d, xv[u], acc[o]);
        }
        if (dx) dx[xo + (int64_t)(b0 + b) * kw] = dxv;
      }
    }
  }
#pragma unroll
  for (int o = 0; o < OO; ++o) red[ig][o][tx] = acc[o];
  __syncthreads();
  if (ig == 0 && valid && dwg)
#pragma unroll
    for (int o = 0; o < OO; ++o) {
      if (o >= O) continue;
      float t = red[0][o][tx];
#pragma unroll
      for (int q = 1; q < kFcG; ++q) t += red[q][o][tx];
      dwg[o * F + f] = t;
    }
}

__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t n, float lr) {
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n && ((reinterpret_cast<uintptr_t>(p + i) | reinterpret_cast<uintptr_t>(g + i)) & 15) == 0) {
    float4 a = *reinterpret_cast<float4*>(p + i);
    const float4 b = *reinterpret_cast<const float4*>(g + i);
    a.x = fmaf(-lr, b.x, a.x); a.y = fmaf(-lr, b.y, a.y); a.z = fmaf(-lr, b.z, a.z); a.w = fmaf(-lr, b.w, a.w);
    *reinterpret_cast<float4*>(p + i) = a;
  } else {
    for (int64_t j = i; j < n && j < i + 4; ++j) p[j] = fmaf(-lr, g[j], p[j]);
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
  if (total == 0) return CP_OK;   // a rank without channels in the last layer (partitioned head)
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
  if (total == 0) return CP_OK;
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
  if (U > 0) {   // U == 0: no features on this rank (partitioned head) -> logits = bias (or 0)
    if (O <= 10) fc_fwd_partial<10><<<dim3(U, (g.Bp + 127) / 128), 256, 0, s>>>(x, wg, part_buf, g, B, O, PW, nsc);
    else fc_fwd_partial<kMaxO><<<dim3(U, (g.Bp + 127) / 128), 256, 0, s>>>(x, wg, part_buf, g, B, O, PW, nsc);
    CP_LAUNCHED();
  }
  fc_fwd_reduce<<<cdiv((int64_t)B * O, 32), dim3(32, 32), 0, s>>>(part_buf, bfc, logits, U, g.Bp, B, O);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_softmax_xent(const float* logits, const int32_t* labels, int32_t B, int32_t O, float* loss, float* dl,
                    void* stream) {
  if (!logits || !labels || !loss || !dl) CP_FAIL(CP_ERR_ARG, "cp_softmax_xent: null pointer");
  if (B < 1 || B > 8192 || O < 1) CP_FAIL(CP_ERR_SHAPE, "cp_softmax_xent: B must be in [1,8192]");
  softmax_xent_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(logits, labels, B, O, loss, dl);
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
  if (dx || dwg || dbfc) {
    const int64_t F = (int64_t)PW * g.Cg;   // (0 features on this rank: one CTA computes dbfc only)
    const unsigned nblk = (unsigned)std::max<int64_t>(1, (F + kFcF - 1) / kFcF);
    // 512-thread CTAs: 2 resident per SM (64 registers); 256-thread: 4
    const bool narrow = (int64_t)nblk > 2 * (int64_t)num_sms_simt();
    if (O <= 10 && narrow) fc_bwd_cols<10, 4><<<nblk, dim3(kFcF, 4), 0, s>>>(dl, x, wg, dx, dwg, dbfc, g, B, O, PW, F);
    else if (O <= 10) fc_bwd_cols<10, 8><<<nblk, dim3(kFcF, 8), 0, s>>>(dl, x, wg, dx, dwg, dbfc, g, B, O, PW, F);
    else if (narrow) fc_bwd_cols<kMaxO, 4><<<nblk, dim3(kFcF, 4), 0, s>>>(dl, x, wg, dx, dwg, dbfc, g, B, O, PW, F);
    else fc_bwd_cols<kMaxO, 8><<<nblk, dim3(kFcF, 8), 0, s>>>(dl, x, wg, dx, dwg, dbfc, g, B, O, PW, F);
    CP_LAUNCHED();
  }
  (void)ws;
  return CP_OK;
}

// ---------------------------------------------------------------- LRN + max-pool (NEXT row f2)
// Cross-channel local response normalisation ("Normalization layer"; form S:L89-97):
//   s_c = bias + alpha * sum_{|j-c|<=n/2, 0<=j<C} a_j^2,  n_c = a_c * s_c^(-beta)
// on the gathered pre-pool map (every rank holds all channels), followed by the 2x2 max-pool with
// first-max ties.  Logical channel c lives in rank block r at slot c - k_begin[r]: the
// per-launch channel table (shared memory) holds each channel's block offset and row stride, so
// the window crosses rank blocks transparently.
constexpr int kLrnMaxC = 2048;

// Forward: one CTA per pooled (i, j, b): the four pre-pool pixel rows of all C channels are loaded
// once into shared memory (per rank block, contiguous), then thread = channel computes the window
// sums, n = a s^-beta for the four window positions, the max with first-max ties, and writes the
// pooled value and code into the channel's rank block (padding slots / images are written as 0).
__global__ void __launch_bounds__(256) lrn_pool_fwd_kernel(const float* __restrict__ a, float* __restrict__ y,
                                                           uint8_t* __restrict__ codes, Blocks gi, Blocks go,
                                                           int C, int B, int W, int half, float alpha,
                                                           float beta, float bias, int round) {
  __shared__ float av[4][kLrnMaxC];
  const int Wp = go.W, Bp = go.Bp;
  const int b = blockIdx.x % Bp, ij = blockIdx.x / Bp, j = ij % Wp, i = ij / Wp;
  const int64_t prow = (int64_t)ij * Bp + b;                    // pooled pixel row
  const bool real = b < B;
  if (real)
    for (int q = 0; q < 4; ++q) {
      const int64_t row = ((int64_t)(2 * i + (q >> 1)) * W + 2 * j + (q & 1)) * Bp + b;
      for (int r = 0; r < gi.n; ++r)
        for (int cc = threadIdx.x; cc < gi.kc[r]; cc += blockDim.x)
          av[q][gi.kb[r] + cc] = a[gi.start[r] + row * gi.kw[r] + cc];
    }
  __syncthreads();
  for (int r = 0; r < go.n; ++r)
    for (int cc = threadIdx.x; cc < go.kw[r]; cc += blockDim.x) {
      float best = 0.f;
      uint32_t code = 0;
      if (real && cc < go.kc[r]) {
        const int c = go.kb[r] + cc;
        const int j0 = max(0, c - half), j1 = min(C - 1, c + half);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float acc = 0.f;
          for (int jj = j0; jj <= j1; ++jj) acc = fmaf(av[q][jj], av[q][jj], acc);
          const float n = av[q][c] * powf(fmaf(alpha, acc, bias), -beta);
          if (q == 0 || n > best) {
            best = n;
            code = q;
          }
        }
      }
      const int64_t o = go.start[r] + prow * go.kw[r] + cc;
      y[o] = round ? tf32_rna(best) : best;
      codes[o] = (uint8_t)code;
    }
}

// Backward for this rank's own channels, one CTA per pre-pool (h, w, b) row: a and the routed
// pooled gradient dn (dy where the pooling code selected this position, else 0) of all channels
// are staged in shared memory; the scales s_j are computed once for j in own range +- n/2:
//   da_c = dn_c s_c^(-beta) - 2 alpha beta a_c sum_{|j-c|<=n/2} dn_j a_j s_j^(-beta-1)
__global__ void __launch_bounds__(256) lrn_pool_bwd_kernel(const float* __restrict__ dy, const float* __restrict__ a,
                                                           const uint8_t* __restrict__ codes, float* __restrict__ da,
                                                           Blocks gi, Blocks go, int rank, int C, int B, int W,
                                                           int half, float alpha, float beta, float bias) {
  __shared__ float av[kLrnMaxC], dn[kLrnMaxC], tj[kLrnMaxC], pw[kLrnMaxC];
  const int Bp = gi.Bp;
  const int b = blockIdx.x % Bp, hw = blockIdx.x / Bp, w = hw % W, h = hw / W;
  const int64_t row = (int64_t)hw * Bp + b;
  const int kb = gi.kb[rank], kc = gi.kc[rank], kw = gi.kw[rank];
  float* out = da + gi.start[rank] + row * kw;
  if (b >= B) {
    for (int cc = threadIdx.x; cc < kw; cc += blockDim.x) out[cc] = 0.f;
    return;
  }
  const int64_t prow = ((int64_t)(h >> 1) * go.W + (w >> 1)) * Bp + b;
  const uint8_t pos = (uint8_t)(2 * (h & 1) + (w & 1));
  for (int r = 0; r < gi.n; ++r)
    for (int cc = threadIdx.x; cc < gi.kc[r]; cc += blockDim.x) {
      const int c = gi.kb[r] + cc;
      av[c] = a[gi.start[r] + row * gi.kw[r] + cc];
      const int64_t po = go.start[r] + prow * go.kw[r] + cc;
      dn[c] = codes[po] == pos ? dy[po] : 0.f;
    }
  __syncthreads();
  const int lo = max(0, kb - half), hi = min(C - 1, kb + kc - 1 + half);
  for (int jj = lo + threadIdx.x; jj <= hi; jj += blockDim.x) {
    float acc = 0.f;
    for (int i2 = max(0, jj - half); i2 <= min(C - 1, jj + half); ++i2) acc = fmaf(av[i2], av[i2], acc);
    const float sj = fmaf(alpha, acc, bias);
    const float p = powf(sj, -beta);
    pw[jj] = p;
    tj[jj] = dn[jj] * av[jj] * p / sj;
  }
  __syncthreads();
  for (int cc = threadIdx.x; cc < kw; cc += blockDim.x) {
    float v = 0.f;
    if (cc < kc) {
      const int c = kb + cc;
      float sum = 0.f;
      for (int jj = max(0, c - half); jj <= min(C - 1, c + half); ++jj) sum += tj[jj];
      v = dn[c] * pw[c] - 2.f * alpha * beta * av[c] * sum;
    }
    out[cc] = v;
  }
}

int launch_lrn_check(int C, int depth, float bias) {
  if (depth < 1 || depth % 2 == 0 || !(bias > 0.f)) CP_FAIL(CP_ERR_CONFIG, "LRN: depth must be odd >= 1 and bias > 0");
  if (C > kLrnMaxC) CP_FAIL(CP_ERR_UNSUPPORTED, "LRN: more than 2048 channels");
  return CP_OK;
}

// SGD over up to kSgdMax tensors in one launch: grid-stride over the concatenated
// float4 index space; the owning tensor is found by a scan of the (short) prefix table.
constexpr int kSgdMax = 16;
struct SgdList {
  float* p[kSgdMax];
  const float* g[kSgdMax];
  long long n[kSgdMax];
  long long off4[kSgdMax + 1];   // prefix of ceil(n/4)
  int count;
};
__global__ void sgd_multi_kernel(const __grid_constant__ SgdList L, float lr) {
  const long long total = L.off4[L.count];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    int t = 0;
    while (i >= L.off4[t + 1]) ++t;
    const long long e = (i - L.off4[t]) * 4;
    float* p = L.p[t];
    const float* g = L.g[t];
    if (e + 3 < L.n[t] && ((reinterpret_cast<uintptr_t>(p + e) | reinterpret_cast<uintptr_t>(g + e)) & 15) == 0) {
      float4 a = *reinterpret_cast<float4*>(p + e);
      const float4 b = *reinterpret_cast<const float4*>(g + e);
      a.x = fmaf(-lr, b.x, a.x); a.y = fmaf(-lr, b.y, a.y); a.z = fmaf(-lr, b.z, a.z); a.w = fmaf(-lr, b.w, a.w);
      *reinterpret_cast<float4*>(p + e) = a;
    } else {
      for (long long j = e; j < L.n[t] && j < e + 4; ++j) p[j] = fmaf(-lr, g[j], p[j]);
    }
  }
}

int cp_lrn_pool_forward(const float* a_g, int32_t B, int32_t H, int32_t W, const cp_partition* part, int32_t depth,
                        float alpha, float beta, float bias, int32_t round_tf32, float* y_g, uint8_t* codes_g,
                        void* stream) {
  CP_TRY(check_part(part));
  if (!a_g || !y_g || !codes_g) CP_FAIL(CP_ERR_ARG, "cp_lrn_pool_forward: null pointer");
  if (B < 1 || (H & 1) || (W & 1) || H < 2 || W < 2) CP_FAIL(CP_ERR_SHAPE, "cp_lrn_pool_forward: bad map shape");
  CP_TRY(launch_lrn_check(part->num_k, depth, bias));
  const int Bp = roundup(B, 32);
  const Blocks gi = make_blocks(*part, H, W, Bp), go = make_blocks(*part, H / 2, W / 2, Bp);
  lrn_pool_fwd_kernel<<<(H / 2) * (W / 2) * Bp, 256, 0, (cudaStream_t)stream>>>(
      a_g, y_g, codes_g, gi, go, part->num_k, B, W, depth / 2, alpha, beta, bias, round_tf32 ? 1 : 0);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_lrn_pool_backward(const float* dy_g, const float* a_g, const uint8_t* codes_g, int32_t B, int32_t H, int32_t W,
                         const cp_partition* part, int32_t rank, int32_t depth, float alpha, float beta, float bias,
                         float* da_g, void* stream) {
  CP_TRY(check_part(part));
  if (!dy_g || !a_g || !codes_g || !da_g) CP_FAIL(CP_ERR_ARG, "cp_lrn_pool_backward: null pointer");
  if (B < 1 || (H & 1) || (W & 1) || H < 2 || W < 2) CP_FAIL(CP_ERR_SHAPE, "cp_lrn_pool_backward: bad map shape");
  if (rank < 0 || rank >= part->n_ranks) CP_FAIL(CP_ERR_ARG, "cp_lrn_pool_backward: bad rank");
  CP_TRY(launch_lrn_check(part->num_k, depth, bias));
  const int Bp = roundup(B, 32);
  const Blocks gi = make_blocks(*part, H, W, Bp), go = make_blocks(*part, H / 2, W / 2, Bp);
  if (gi.kw[rank] == 0) return CP_OK;
  lrn_pool_bwd_kernel<<<H * W * Bp, 256, 0, (cudaStream_t)stream>>>(dy_g, a_g, codes_g, da_g, gi, go, rank,
                                                                  part->num_k, B, W, depth / 2, alpha, beta, bias);
  CP_LAUNCHED();
  return CP_OK;
}

int cp_sgd_multi(float* const* params, const float* const* grads, const int64_t* sizes, int32_t count, float lr,
                 void* stream) {
  if (count < 0 || (count > 0 && (!params || !grads || !sizes))) CP_FAIL(CP_ERR_ARG, "cp_sgd_multi: bad arguments");
  for (int i0 = 0; i0 < count; i0 += kSgdMax) {
    SgdList L{};
    L.off4[0] = 0;
    for (int i = i0; i < count && L.count < kSgdMax; ++i) {
      if (sizes[i] < 0 || (sizes[i] > 0 && (!params[i] || !grads[i]))) CP_FAIL(CP_ERR_ARG, "cp_sgd_multi: bad tensor");
      const int k = L.count++;
      L.p[k] = params[i];
      L.g[k] = grads[i];
      L.n[k] = sizes[i];
      L.off4[k + 1] = L.off4[k] + (sizes[i] + 3) / 4;
    }
    const long long total = L.off4[L.count];
    if (total == 0) continue;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 8);
    sgd_multi_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(L, lr);
    CP_LAUNCHED();
  }
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
