/*
 * convnet_oracle.c — fp64 CPU oracle for kernel-partitioned conv-layer training
 * (arXiv 1712.02546).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or helper with the CUDA product path (paper_1712_02546_b200/).
 *
 * Every function is the plain definition written out as direct loops in a fixed
 * summation order (OpenMP only splits *independent output elements*, never a sum),
 * so results are bit-identical for any thread count.
 *
 * Citations: P:Lnn = PAPER.md line nn, S:Lnn = SPEC.md line nn (read-only reference).
 * Layout: NCHW / KCRS, row-major, fp64 ("Tensor4", "KernelBank").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG -1
#define ORC_ERR_SHAPE -2
#define ORC_ERR_CONFIG -3
#define ORC_ERR_DATA -4

#define IX4(a, b, c, d, B_, C_, D_) ((((int64_t)(a) * (B_) + (b)) * (C_) + (c)) * (D_) + (d))

/* --------------------------------------------------------------------------
 * Convolution forward — valid cross-correlation, stride 1 (reading 1-2
 * of DESIGN.md: padding/stride never stated by the paper, shape chain
 * 32->28->14->10->5 of S:L131 fixes "valid, stride 1").  Output map k depends
 * only on kernel k — the exactness basis of kernel partitioning
 * ("All slaves receive same inputs but different kernels").
 *   z[b,k,p,q] = bias[k] + sum_c sum_r sum_s x[b,c,p+r,q+s] * w[k,c,r,s]
 * bias may be NULL (SPEC-literal, no bias).
 * -------------------------------------------------------------------------- */
int orc_conv_fwd(const double* x, int B, int C, int H, int W,
                 const double* w, int K, int R, int S,
                 const double* bias, double* z) {
  if (!x || !w || !z) return ORC_ERR_ARG;
  if (B < 1 || C < 1 || K < 1 || R < 1 || S < 1 || H < R || W < S) return ORC_ERR_SHAPE;
  const int P = H - R + 1, Q = W - S + 1;
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < K; ++k)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) {
          double acc = 0.0;
          for (int c = 0; c < C; ++c)
            for (int r = 0; r < R; ++r)
              for (int s = 0; s < S; ++s)
                acc += x[IX4(b, c, p + r, q + s, C, H, W)] * w[IX4(k, c, r, s, C, R, S)];
          z[IX4(b, k, p, q, K, P, Q)] = (bias ? bias[k] : 0.0) + acc;
        }
  return ORC_OK;
}

/* One output element by brute force (sampled parity at full size, §8(c)).
 * Same summation order as orc_conv_fwd. */
int orc_conv_fwd_points(const double* x, int B, int C, int H, int W,
                        const double* w, int K, int R, int S, const double* bias,
                        const int64_t* idx /* n x 4: b,k,p,q */, int64_t n, double* out) {
  if (!x || !w || !idx || !out) return ORC_ERR_ARG;
  const int P = H - R + 1, Q = W - S + 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const int b = (int)idx[4 * i], k = (int)idx[4 * i + 1], p = (int)idx[4 * i + 2], q = (int)idx[4 * i + 3];
    if (b < 0 || b >= B || k < 0 || k >= K || p < 0 || p >= P || q < 0 || q >= Q) { out[i] = NAN; continue; }
    double acc = 0.0;
    for (int c = 0; c < C; ++c)
      for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s)
          acc += x[IX4(b, c, p + r, q + s, C, H, W)] * w[IX4(k, c, r, s, C, R, S)];
    out[i] = (bias ? bias[k] : 0.0) + acc;
  }
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Conv backward-data (dgrad): the analytic gradient of orc_conv_fwd w.r.t. x
 * (Abstract P:L17 "forward and backward propagation included").
 *   dx[b,c,h,w] = sum_k sum_{(r,s): 0<=h-r<P, 0<=w-s<Q} dy[b,k,h-r,w-s] * w[k,c,r,s]
 * k ascending outermost, then r, s.  k_begin/k_end restrict the sum to one
 * kernel slice (the per-rank partial dX of the partitioned method, north_star);
 * pass 0,K for the unsplit layer.  If accumulate != 0 the result is added to dx
 * (carried-accumulator mode: slice r continues slices < r, §8(c) item 10).
 * -------------------------------------------------------------------------- */
int orc_conv_dgrad(const double* dy, int B, int K, int P, int Q,
                   const double* w, int C, int R, int S,
                   int k_begin, int k_end, int accumulate, double* dx) {
  if (!dy || !w || !dx) return ORC_ERR_ARG;
  if (B < 1 || K < 1 || C < 1 || R < 1 || S < 1 || P < 1 || Q < 1) return ORC_ERR_SHAPE;
  if (k_begin < 0 || k_end > K || k_begin > k_end) return ORC_ERR_ARG;
  const int H = P + R - 1, W = Q + S - 1;
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int c = 0; c < C; ++c)
      for (int h = 0; h < H; ++h)
        for (int x_ = 0; x_ < W; ++x_) {
          double acc = accumulate ? dx[IX4(b, c, h, x_, C, H, W)] : 0.0;
          for (int k = k_begin; k < k_end; ++k)
            for (int r = 0; r < R; ++r) {
              const int p = h - r;
              if (p < 0 || p >= P) continue;
              for (int s = 0; s < S; ++s) {
                const int q = x_ - s;
                if (q < 0 || q >= Q) continue;
                acc += dy[IX4(b, k, p, q, K, P, Q)] * w[IX4(k, c, r, s, C, R, S)];
              }
            }
          dx[IX4(b, c, h, x_, C, H, W)] = acc;
        }
  return ORC_OK;
}

int orc_conv_dgrad_points(const double* dy, int B, int K, int P, int Q,
                          const double* w, int C, int R, int S,
                          const int64_t* idx /* n x 4: b,c,h,w */, int64_t n, double* out) {
  if (!dy || !w || !idx || !out) return ORC_ERR_ARG;
  const int H = P + R - 1, W = Q + S - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const int b = (int)idx[4 * i], c = (int)idx[4 * i + 1], h = (int)idx[4 * i + 2], x_ = (int)idx[4 * i + 3];
    if (b < 0 || b >= B || c < 0 || c >= C || h < 0 || h >= H || x_ < 0 || x_ >= W) { out[i] = NAN; continue; }
    double acc = 0.0;
    for (int k = 0; k < K; ++k)
      for (int r = 0; r < R; ++r) {
        const int p = h - r;
        if (p < 0 || p >= P) continue;
        for (int s = 0; s < S; ++s) {
          const int q = x_ - s;
          if (q < 0 || q >= Q) continue;
          acc += dy[IX4(b, k, p, q, K, P, Q)] * w[IX4(k, c, r, s, C, R, S)];
        }
      }
    out[i] = acc;
  }
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Conv backward-filter (wgrad): analytic gradient w.r.t. w.
 *   dw[k,c,r,s] = sum_b sum_p sum_q dy[b,k,p,q] * x[b,c,p+r,q+s]
 * Weight gradients of a kernel slice depend only on that slice's dy rows
 * (north_star: "Weight gradients stay local because each rank owns its kernels").
 * -------------------------------------------------------------------------- */
int orc_conv_wgrad(const double* dy, int B, int K, int P, int Q,
                   const double* x, int C, int R, int S, double* dw) {
  if (!dy || !x || !dw) return ORC_ERR_ARG;
  if (B < 1 || K < 1 || C < 1 || R < 1 || S < 1 || P < 1 || Q < 1) return ORC_ERR_SHAPE;
  const int H = P + R - 1, W = Q + S - 1;
#pragma omp parallel for collapse(2) schedule(static)
  for (int k = 0; k < K; ++k)
    for (int c = 0; c < C; ++c)
      for (int r = 0; r < R; ++r)
        for (int s = 0; s < S; ++s) {
          double acc = 0.0;
          for (int b = 0; b < B; ++b)
            for (int p = 0; p < P; ++p)
              for (int q = 0; q < Q; ++q)
                acc += dy[IX4(b, k, p, q, K, P, Q)] * x[IX4(b, c, p + r, q + s, C, H, W)];
          dw[IX4(k, c, r, s, C, R, S)] = acc;
        }
  return ORC_OK;
}

int orc_conv_wgrad_points(const double* dy, int B, int K, int P, int Q,
                          const double* x, int C, int R, int S,
                          const int64_t* idx /* n x 4: k,c,r,s */, int64_t n, double* out) {
  if (!dy || !x || !idx || !out) return ORC_ERR_ARG;
  const int H = P + R - 1, W = Q + S - 1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const int k = (int)idx[4 * i], c = (int)idx[4 * i + 1], r = (int)idx[4 * i + 2], s = (int)idx[4 * i + 3];
    if (k < 0 || k >= K || c < 0 || c >= C || r < 0 || r >= R || s < 0 || s >= S) { out[i] = NAN; continue; }
    double acc = 0.0;
    for (int b = 0; b < B; ++b)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q)
          acc += dy[IX4(b, k, p, q, K, P, Q)] * x[IX4(b, c, p + r, q + s, C, H, W)];
    out[i] = acc;
  }
  return ORC_OK;
}

/* Bias gradient: db[k] = sum_{b,p,q} dy[b,k,p,q] (reading 4: conv bias present). */
int orc_bias_grad(const double* dy, int B, int K, int P, int Q, double* db) {
  if (!dy || !db) return ORC_ERR_ARG;
#pragma omp parallel for schedule(static)
  for (int k = 0; k < K; ++k) {
    double acc = 0.0;
    for (int b = 0; b < B; ++b)
      for (int p = 0; p < P; ++p)
        for (int q = 0; q < Q; ++q) acc += dy[IX4(b, k, p, q, K, P, Q)];
    db[k] = acc;
  }
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * ReLU (reading 3: on) followed by 2x2 stride-2 max pooling (P:L71,
 * P:L271 "Pooling layer, with stride 2").  Ties break to the first
 * position in row-major order (0,0),(0,1),(1,0),(1,1) via a strict '>' scan
 * (S:L137).  argmax code = 2*di + dj.  relu=0 gives SPEC-literal pooling.
 * pool=0 writes a = relu(z) and argmax untouched (may be NULL).
 * -------------------------------------------------------------------------- */
int orc_relu_pool_fwd(const double* z, int B, int K, int H, int W, int relu, int pool,
                      double* a, uint8_t* argmax) {
  if (!z || !a) return ORC_ERR_ARG;
  if (!pool) {
    const int64_t n = (int64_t)B * K * H * W;
    for (int64_t i = 0; i < n; ++i) a[i] = (relu && !(z[i] > 0.0)) ? 0.0 : z[i];
    return ORC_OK;
  }
  if (!argmax) return ORC_ERR_ARG;
  if ((H % 2) || (W % 2)) return ORC_ERR_SHAPE; /* S:L75 non-divisible -> dimension error */
  const int Hp = H / 2, Wp = W / 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < Hp; ++i)
        for (int j = 0; j < Wp; ++j) {
          double best = 0.0;
          int code = 0;
          for (int t = 0; t < 4; ++t) {
            const int di = t >> 1, dj = t & 1;
            double v = z[IX4(b, k, 2 * i + di, 2 * j + dj, K, H, W)];
            if (relu && !(v > 0.0)) v = 0.0;
            if (t == 0 || v > best) { best = v; code = t; }
          }
          a[IX4(b, k, i, j, K, Hp, Wp)] = best;
          argmax[IX4(b, k, i, j, K, Hp, Wp)] = (uint8_t)code;
        }
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Backward of ReLU + max-pool: route da to the argmax position,
 * times the ReLU derivative there.  ReLU'(0) = 0 (reading 7).  The ReLU
 * decision uses the pooled output a (a>0 <=> z(argmax)>0), so a GPU's
 * argmax codes and outputs can be *replayed* (reading 15, decision replay).
 *   dy[b,k,2i+di,2j+dj] = da[b,k,i,j] * [code==2di+dj] * [a[b,k,i,j] > 0 or !relu]
 * pool=0: dy = da * [a > 0 or !relu] elementwise on the full grid (H=Hp, W=Wp).
 * -------------------------------------------------------------------------- */
int orc_unpool_relu_bwd(const double* da, const uint8_t* argmax, const double* a,
                        int B, int K, int Hp, int Wp, int relu, int pool, double* dy) {
  if (!da || !a || !dy) return ORC_ERR_ARG;
  if (!pool) {
    const int64_t n = (int64_t)B * K * Hp * Wp;
    for (int64_t i = 0; i < n; ++i) dy[i] = (!relu || a[i] > 0.0) ? da[i] : 0.0;
    return ORC_OK;
  }
  if (!argmax) return ORC_ERR_ARG;
  const int H = 2 * Hp, W = 2 * Wp;
  memset(dy, 0, sizeof(double) * (size_t)B * K * H * W);
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < Hp; ++i)
        for (int j = 0; j < Wp; ++j) {
          const int64_t o = IX4(b, k, i, j, K, Hp, Wp);
          const int code = argmax[o];
          if (code > 3) continue;
          if (relu && !(a[o] > 0.0)) continue;
          dy[IX4(b, k, 2 * i + (code >> 1), 2 * j + (code & 1), K, H, W)] = da[o];
        }
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Local response normalisation across channels — the paper's "Normalization layer"
 * (form unspecified there, SPEC S:L89-97 and design decision S:L135):
 *   s[b,c,h,w]   = bias + alpha * sum_{j=max(0,c-n/2)}^{min(C-1,c+n/2)} in[b,j,h,w]^2
 *   out[b,c,h,w] = in[b,c,h,w] * s^(-beta)            (n = depth, odd; window clipped)
 * Errors: depth even or < 1, bias <= 0 -> configuration error.
 * -------------------------------------------------------------------------- */
static double lrn_scale(const double* in, int b, int c, int h, int w, int C, int H, int W, int half,
                        double alpha, double bias) {
  double acc = 0.0;
  const int j0 = c - half < 0 ? 0 : c - half, j1 = c + half > C - 1 ? C - 1 : c + half;
  for (int j = j0; j <= j1; ++j) {
    const double v = in[IX4(b, j, h, w, C, H, W)];
    acc += v * v;
  }
  return bias + alpha * acc;
}

int orc_lrn_fwd(const double* in, int B, int C, int H, int W, int depth, double alpha, double beta,
                double bias, double* out) {
  if (!in || !out) return ORC_ERR_ARG;
  if (depth < 1 || depth % 2 == 0 || !(bias > 0.0)) return ORC_ERR_CONFIG;
  const int half = depth / 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int c = 0; c < C; ++c)
      for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
          const double s = lrn_scale(in, b, c, h, w, C, H, W, half, alpha, bias);
          out[IX4(b, c, h, w, C, H, W)] = in[IX4(b, c, h, w, C, H, W)] * pow(s, -beta);
        }
  return ORC_OK;
}

/* Backward by the chain rule written out ("backward matches finite differences"):
 *   din[c] = sum_{j : |j-c| <= n/2, 0<=j<C} dout[j] * d out[j] / d in[c]
 *   d out[j] / d in[c] = [j==c] s_j^(-beta) - 2 alpha beta in[j] in[c] s_j^(-beta-1)        */
int orc_lrn_bwd(const double* in, const double* dout, int B, int C, int H, int W, int depth, double alpha,
                double beta, double bias, double* din) {
  if (!in || !dout || !din) return ORC_ERR_ARG;
  if (depth < 1 || depth % 2 == 0 || !(bias > 0.0)) return ORC_ERR_CONFIG;
  const int half = depth / 2;
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int c = 0; c < C; ++c)
      for (int h = 0; h < H; ++h)
        for (int w = 0; w < W; ++w) {
          const double xc = in[IX4(b, c, h, w, C, H, W)];
          double acc = 0.0;
          const int j0 = c - half < 0 ? 0 : c - half, j1 = c + half > C - 1 ? C - 1 : c + half;
          for (int j = j0; j <= j1; ++j) {
            const double sj = lrn_scale(in, b, j, h, w, C, H, W, half, alpha, bias);
            double d = -2.0 * alpha * beta * in[IX4(b, j, h, w, C, H, W)] * xc * pow(sj, -beta - 1.0);
            if (j == c) d += pow(sj, -beta);
            acc += dout[IX4(b, j, h, w, C, H, W)] * d;
          }
          din[IX4(b, c, h, w, C, H, W)] = acc;
        }
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Fully connected: logits[b,o] = bfc[o] + sum_f wfc[o,f] a[b,f]
 * with f the NCHW flatten of the pooled map (§8(c) item 4).
 * -------------------------------------------------------------------------- */
int orc_fc_fwd(const double* a, int B, int F, const double* wfc, const double* bfc, int O,
               double* logits) {
  if (!a || !wfc || !logits) return ORC_ERR_ARG;
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < B; ++b)
    for (int o = 0; o < O; ++o) {
      double acc = 0.0;
      for (int f = 0; f < F; ++f) acc += wfc[(int64_t)o * F + f] * a[(int64_t)b * F + f];
      logits[(int64_t)b * O + o] = (bfc ? bfc[o] : 0.0) + acc;
    }
  return ORC_OK;
}

/* FC backward: da = dlogits . wfc ; dwfc = dlogits^T . a ; dbfc = sum_b dlogits. */
int orc_fc_bwd(const double* dlogits, const double* a, const double* wfc, int B, int F, int O,
               double* da, double* dwfc, double* dbfc) {
  if (!dlogits || !a || !wfc) return ORC_ERR_ARG;
  if (da) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
      for (int f = 0; f < F; ++f) {
        double acc = 0.0;
        for (int o = 0; o < O; ++o) acc += dlogits[(int64_t)b * O + o] * wfc[(int64_t)o * F + f];
        da[(int64_t)b * F + f] = acc;
      }
  }
  if (dwfc) {
#pragma omp parallel for collapse(2) schedule(static)
    for (int o = 0; o < O; ++o)
      for (int f = 0; f < F; ++f) {
        double acc = 0.0;
        for (int b = 0; b < B; ++b) acc += dlogits[(int64_t)b * O + o] * a[(int64_t)b * F + f];
        dwfc[(int64_t)o * F + f] = acc;
      }
  }
  if (dbfc) {
    for (int o = 0; o < O; ++o) {
      double acc = 0.0;
      for (int b = 0; b < B; ++b) acc += dlogits[(int64_t)b * O + o];
      dbfc[o] = acc;
    }
  }
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Softmax loss ("Loss layer, with softmax loss"): mean
 * cross-entropy over the batch, max-subtracted; dlogits = (softmax-onehot)/B.
 * -------------------------------------------------------------------------- */
int orc_softmax_xent(const double* logits, const int32_t* y, int B, int O,
                     double* loss, double* dlogits) {
  if (!logits || !y || !loss) return ORC_ERR_ARG;
  double total = 0.0;
  for (int b = 0; b < B; ++b) {
    if (y[b] < 0 || y[b] >= O) return ORC_ERR_DATA; /* S:L111 label out of range */
    const double* l = logits + (int64_t)b * O;
    double m = l[0];
    for (int o = 1; o < O; ++o) if (l[o] > m) m = l[o];
    double se = 0.0;
    for (int o = 0; o < O; ++o) se += exp(l[o] - m);
    const double lse = m + log(se);
    total += lse - l[y[b]];
    if (dlogits)
      for (int o = 0; o < O; ++o)
        dlogits[(int64_t)b * O + o] = (exp(l[o] - lse) - (o == y[b] ? 1.0 : 0.0)) / (double)B;
  }
  *loss = total / (double)B;
  return ORC_OK;
}

/* SGD: p <- p - lr*g, elementwise, no momentum (reading 9). */
int orc_sgd(double* p, const double* g, int64_t n, double lr) {
  if (!p || !g) return ORC_ERR_ARG;
  for (int64_t i = 0; i < n; ++i) p[i] = p[i] - lr * g[i];
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Eq. 1 workload weights:
 *   w_i = (max(t)/t_i) / sum_j (max(t)/t_j)
 * nonpositive time -> data error.
 * -------------------------------------------------------------------------- */
int orc_eq1_weights(const double* t, int n, double* w) {
  if (!t || !w || n < 1) return ORC_ERR_ARG;
  double tmax = t[0];
  for (int i = 0; i < n; ++i) {
    if (!(t[i] > 0.0)) return ORC_ERR_DATA;
    if (t[i] > tmax) tmax = t[i];
  }
  double den = 0.0;
  for (int j = 0; j < n; ++j) den += tmax / t[j];
  for (int i = 0; i < n; ++i) w[i] = (tmax / t[i]) / den;
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Partition plan (a1): Eq. 1 + largest-remainder (Hamilton) apportionment
 * (floor quotas, leftover units by descending fractional
 * remainder, ties to the lower device id), contiguous ranges in device order
 * (S:L205-213), block width = roundup(count, align).
 * Exact-integer reading (reading R11): throughputs are quantised
 *   q_i = llround(2^20 * max(t)/t_i)
 * and quotas compared as exact rationals num_i = numK*q_i over den = sum q.
 * The leftover is handed out by repeatedly picking the largest remaining
 * remainder (a selection loop, O(n^2), no sort).
 * -------------------------------------------------------------------------- */
int orc_plan(const double* t, int n, int num_k, int align,
             int32_t* k_begin, int32_t* k_count, int32_t* k_width) {
  if (!t || !k_begin || !k_count || !k_width) return ORC_ERR_ARG;
  if (n < 1 || num_k < 0 || align < 1) return ORC_ERR_ARG;
  double tmax = t[0];
  for (int i = 0; i < n; ++i) {
    if (!(t[i] > 0.0) || !isfinite(t[i])) return ORC_ERR_DATA;
    if (t[i] > tmax) tmax = t[i];
  }
  int64_t* q = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* rem = (int64_t*)malloc(sizeof(int64_t) * n);
  char* taken = (char*)calloc(n, 1);
  int64_t sq = 0;
  for (int i = 0; i < n; ++i) {
    q[i] = llround(1048576.0 * (tmax / t[i]));
    sq += q[i];
  }
  int64_t assigned = 0;
  for (int i = 0; i < n; ++i) {
    const int64_t num = (int64_t)num_k * q[i];
    k_count[i] = (int32_t)(num / sq);
    rem[i] = num % sq;
    assigned += k_count[i];
  }
  for (int64_t left = num_k - assigned; left > 0; --left) {
    int best = -1;
    for (int i = 0; i < n; ++i)
      if (!taken[i] && (best < 0 || rem[i] > rem[best])) best = i; /* '>' keeps lower id on ties */
    taken[best] = 1;
    k_count[best] += 1;
  }
  int32_t acc = 0;
  for (int i = 0; i < n; ++i) {
    k_begin[i] = acc;
    acc += k_count[i];
    k_width[i] = (int32_t)(((k_count[i] + align - 1) / align) * align);
  }
  free(q); free(rem); free(taken);
  return ORC_OK;
}

/* --------------------------------------------------------------------------
 * Physical index map of the gathered, rank-blocked layout (§8(c) item 9):
 * logical channel c lives in rank r = owner(c) at slot c - k_begin[r]; element
 * (b,c,h,w) of an NCHW tensor sits at
 *   block_start[r] + ((h*W + w)*Bp + b)*Kc_r + (c - k_begin[r]),
 *   block_start[r] = sum_{r'<r} H*W*Bp*Kc_{r'}
 * Padding slots (slot >= count, b >= B) are zero.  This is the "reshape and
 * rearrange" of P:L235 written out as one index formula.
 * -------------------------------------------------------------------------- */
int orc_pack_gather(const double* x_nchw, int B, int C, int H, int W, int Bp,
                    int n_ranks, const int32_t* k_begin, const int32_t* k_count,
                    const int32_t* k_width, double* out) {
  if (!x_nchw || !out || !k_begin || !k_count || !k_width) return ORC_ERR_ARG;
  if (Bp < B) return ORC_ERR_SHAPE;
  int64_t total = 0;
  for (int r = 0; r < n_ranks; ++r) total += (int64_t)H * W * Bp * k_width[r];
  memset(out, 0, sizeof(double) * (size_t)total);
  int64_t start = 0;
  for (int r = 0; r < n_ranks; ++r) {
    for (int slot = 0; slot < k_count[r]; ++slot) {
      const int c = k_begin[r] + slot;
      if (c >= C) return ORC_ERR_SHAPE;
      for (int b = 0; b < B; ++b)
        for (int h = 0; h < H; ++h)
          for (int w = 0; w < W; ++w)
            out[start + (((int64_t)h * W + w) * Bp + b) * k_width[r] + slot] =
                x_nchw[IX4(b, c, h, w, C, H, W)];
    }
    start += (int64_t)H * W * Bp * k_width[r];
  }
  return ORC_OK;
}
