// kernels_conv1.cu — the image-input conv layer (the paper net's conv1) as a dedicated tcgen05 kernel.
//
// FORWARD (own kernels, bias + ReLU + 2x2 max-pool):
//   Z[k][(b, dh, c)] = bias[k] + sum_{(r,s,ch)} W[k][(r,s,ch)] * X[b][ch][2i+dh+r][c+s]
// computed transposed: the own kernels are the MMA's M rows (TMEM lanes), the output pixels its N
// columns.  A column block ("B-set") is nb images x the two output rows 2i, 2i+1 of one pooled row x
// a segment of wseg output columns, so the four positions of every 2x2 pooling window sit in the SAME
// thread's registers (lane = kernel): the pool, its argmax code, bias and ReLU run in registers with no
// shared-memory exchange, and each pooled value is one lane of a coalesced 128 B store (32 consecutive
// kernels of one pixel and image in the gather layout).
//   * The B operand (im2col rows, K-major, 128B-swizzled) is built directly from the NCHW images in
//     shared memory by four builder warps - no im2col pass through HBM/L2 (the old path wrote 32 MB
//     and read it back).  A B-set is built once and reused by every 128-kernel M tile.
//   * The A operand (the own kernels' weights [Kr][Kcol], K-major) streams through a TMA ring.
//   * Two TMEM accumulators (2 x 256 columns): the epilogue of one M tile overlaps the MMAs of the next.
// Warp roles (896 threads): w0 TMA producer (weights), w1 MMA issuer (one thread), w2 TMEM allocator,
// w3 input-patch TMA, w4-w11 B builders, w12-w27 epilogue (four groups of four, one TMEM lane quadrant per
// warp: the epilogue is TMEM-read and ALU bound, ~20 instructions per pooled output, and needs the warps).
#include <algorithm>
#include <cstdio>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace cp {
using namespace tc;

namespace {

constexpr int C1_BM = 128;            // own kernels per M tile (TMEM lanes)
constexpr int C1_NMAX = 224;          // pixels per B-set (MMA N), <= 224 so a 32-column load stays in 256
constexpr int C1_THREADS = 896;
constexpr int C1_BUILD_WARP0 = 4, C1_BUILD_THREADS = 256, C1_EPI_WARP0 = 12, C1_EPI_WARPS = 16;   // 4 epi groups
constexpr int C1_EPI_GROUPS = C1_EPI_WARPS / 4;
constexpr int C1_MAXK = 256;          // Kcol limit (R*S*C padded to 8)
constexpr int C1_ABYTES = C1_BM * 128;   // one 32-wide K chunk of a 128-kernel A tile

struct C1Params {
  CUtensorMap wmap;      // own weights [Kr][Kcol] (K-major), box {32, 128}
  CUtensorMap xmap;      // images (W, H, C, B), box {pw, R+1, C, nb}: the input patch of one B-set
  const float* x;        // images NCHW [B][C][H][W]
  const float* bias;     // [Kr] or null
  float* out;            // own block of the gathered output [Hp][Wp][Bp][Kc]
  uint8_t* saved;        // argmax codes, same layout
  int B, Bp, C, H, W, Ho, Wo, Hp, Wp;
  int Kr, Kc, Kcol, nch; // K chunks of 32 (the last one may be shorter)
  int nb, wseg, nseg, ngrp;  // B-set = nb images x 2 rows x wseg columns; nseg segments, ngrp image groups
  int nsets, mtiles;
  int balance;           // 1: each CTA takes a contiguous range of the nsets x mtiles (set, M tile) units
  int nbuf, astages;     // B-set buffers (1 or 2) and A ring depth, sized to shared memory
  int bset_bytes;        // nch * bstride
  int bstride;           // bytes of one 32-wide K chunk of a B-set: N rows (max over sets, x8) * 128 B
  int pw, pimg, patch_bytes;  // patch row width (>= wseg + S - 1, x4), floats per image C*(R+1)*pw, bytes
  int relu, round;
  int off[C1_MAXK];      // im2col column kk = (r*S + s)*C + ch -> (ch*(R+1) + r)*pw + s in the patch, -1 = pad
#ifdef C1F_TRACE
  unsigned long long* trace;   // experiment builds: CTA 0's per-set %globaltimer stamps [5][8]
#endif
};
#ifdef C1F_TRACE
#define C1F_STAMP(kind, ls)                                                                  \
  do {                                                                                        \
    if (blockIdx.x == 0 && (ls) < 8) p.trace[(kind) * 8 + (ls)] = globaltimer_ns();            \
  } while (0)
#else
#define C1F_STAMP(kind, ls) do { } while (0)
#endif

struct SetGeo {
  int i, c0, ws, b0, n;  // pooled row, first output column, segment width, first image, MMA N (x8)
};
__device__ __forceinline__ SetGeo set_geo(const C1Params& p, int set) {
  SetGeo g;
  const int bg = set % p.ngrp;
  const int rest = set / p.ngrp;
  const int sg = rest % p.nseg;
  g.i = rest / p.nseg;
  g.c0 = sg * p.wseg;
  g.ws = min(p.wseg, p.Wo - g.c0);
  g.b0 = bg * p.nb;
  g.n = (p.nb * 2 * g.ws + 7) / 8 * 8;
  return g;
}

// This CTA's work: sets set0, set0 + step, ... (nset of them), M tiles [mt_first, mtiles) of the first
// and [0, mt_end) of the last.  balance: a contiguous range of the (set, M tile) units, split as evenly
// as the grid allows (448 sets x 4 M tiles on 148 SMs: 12-13 units per CTA instead of 3 or 4 whole
// sets); otherwise whole sets strided by the grid.  A set whose tiles two CTAs share is built by both.
struct C1Work {
  int set0, step, nset, mt_first, mt_end;
};
__device__ __forceinline__ C1Work c1_work(const C1Params& p) {
  C1Work w;
  if (p.balance) {
    const int U = p.nsets * p.mtiles;
    const int lo = (int)((long long)blockIdx.x * U / gridDim.x);
    const int hi = (int)((long long)(blockIdx.x + 1) * U / gridDim.x);
    const int last = (hi - 1) / p.mtiles;
    w.set0 = lo / p.mtiles;
    w.step = 1;
    w.nset = hi > lo ? last - w.set0 + 1 : 0;
    w.mt_first = lo - w.set0 * p.mtiles;
    w.mt_end = hi - last * p.mtiles;
  } else {
    w.set0 = blockIdx.x;
    w.step = gridDim.x;
    w.nset = (int)blockIdx.x < p.nsets ? (p.nsets - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    w.mt_first = 0;
    w.mt_end = p.mtiles;
  }
  return w;
}
__device__ __forceinline__ int c1_mt_begin(const C1Work& w, int ls) { return ls == 0 ? w.mt_first : 0; }
__device__ __forceinline__ int c1_mt_end(const C1Work& w, int ls, int mtiles) {
  return ls == w.nset - 1 ? w.mt_end : mtiles;
}

__device__ __forceinline__ void tmem_ld_x32_nowait(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_x16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// round to the nearest tf32, ties away from zero: identical to cvt.rna.tf32.f32 for every finite input (and
// infinities); two integer ops instead of cvt's multi-instruction expansion on the CUDA cores
__device__ __forceinline__ float tf32_round(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

template <bool RELU>
__global__ void __launch_bounds__(C1_THREADS, 1) conv1_fwd_kernel(const __grid_constant__ C1Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sB = smem;                                      // nbuf x bset_bytes
  uint8_t* sA = smem + p.nbuf * p.bset_bytes;              // astages x 16 KB
  float* sP = reinterpret_cast<float*>(sA + p.astages * C1_ABYTES);   // nbuf x input patch
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sP) + p.nbuf * p.patch_bytes);
  uint64_t* afull = bars;                 // [astages]
  uint64_t* aempty = bars + 8;            // [astages]
  uint64_t* bfull = bars + 16;            // [2]
  uint64_t* bempty = bars + 18;           // [2]
  uint64_t* tfull = bars + 20;            // [2]
  uint64_t* tempty = bars + 22;           // [2]
  uint64_t* pfull = bars + 24;            // [2] input patch landed (TMA)
  uint64_t* pempty = bars + 26;           // [2] patch consumed by the builders
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 28);
  int* off_s = reinterpret_cast<int*>(bars + 29);         // C1_MAXK

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int k = threadIdx.x; k < C1_MAXK; k += blockDim.x) off_s[k] = p.off[k];
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.astages; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bfull[b], 1);
      mbar_init(&bempty[b], 1);
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], C1_EPI_WARPS);
      mbar_init(&pfull[b], 1);
      mbar_init(&pempty[b], 1);
    }
    fence_barrier_init();
    tma_prefetch(&p.wmap);
    tma_prefetch(&p.xmap);
  }
  if (warp == 2) tmem_alloc<1>(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const C1Work wk = c1_work(p);

  if (warp == 0) {
    // ======================= A producer: the own kernels' weight chunks, one M tile after another
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int ls = 0; ls < wk.nset; ++ls)
        for (int mt = c1_mt_begin(wk, ls); mt < c1_mt_end(wk, ls, p.mtiles); ++mt)
          for (int c = 0; c < p.nch; ++c) {
            mbar_wait(&aempty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&afull[stage], C1_ABYTES);
            tma_load_2d(sA + stage * C1_ABYTES, &p.wmap, &afull[stage], c * 32, mt * C1_BM);
            if (++stage == p.astages) {
              stage = 0;
              phase ^= 1;
            }
          }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int u = 0;
      for (int ls = 0; ls < wk.nset; ++ls) {
        const SetGeo g = set_geo(p, wk.set0 + ls * wk.step);
        const int buf = p.nbuf == 2 ? (ls & 1) : 0;
        const uint32_t bph = p.nbuf == 2 ? ((ls >> 1) & 1) : (ls & 1);
        mbar_wait(&bfull[buf], bph);
        tc_fence_after();
        C1F_STAMP(3, ls);
        const uint32_t idesc = idesc_tf32(C1_BM, g.n, 0, 0);
        const uint32_t bbase = smem_u32(sB + buf * p.bset_bytes);
        for (int mt = c1_mt_begin(wk, ls); mt < c1_mt_end(wk, ls, p.mtiles); ++mt, ++u) {
          const int acc = u & 1;
          mbar_wait(&tempty[acc], ((u >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * 256;
          uint32_t accumulate = 0;
          for (int c = 0; c < p.nch; ++c) {
            mbar_wait(&afull[stage], phase);
            tc_fence_after();
            const uint64_t ad0 = sdesc_k(smem_u32(sA + stage * C1_ABYTES), 0);
            const uint64_t bd0 = sdesc_k(bbase + c * p.bstride, 0);
            const int ksteps = min(32, p.Kcol - c * 32) / 8;
            for (int k = 0; k < ksteps; ++k) {
              mma_tf32(d_tmem, ad0 + 2 * k, bd0 + 2 * k, idesc, accumulate);
              accumulate = 1;
            }
            mma_commit(&aempty[stage]);
            if (++stage == p.astages) {
              stage = 0;
              phase ^= 1;
            }
          }
          mma_commit(&tfull[acc]);
        }
        mma_commit(&bempty[buf]);   // every M tile of this set issued: the buffer frees when they complete
      }
    }
  } else if (warp == 3) {
    // ======================= patch producer: the B-set's input pixels (nb images x C x R+1 rows x pw
    // columns, zero outside the images) in one TMA box
    if (lane == 0) {
      for (int ls = 0; ls < wk.nset; ++ls) {
        const SetGeo g = set_geo(p, wk.set0 + ls * wk.step);
        const int buf = p.nbuf == 2 ? (ls & 1) : 0;
        const uint32_t bph = p.nbuf == 2 ? ((ls >> 1) & 1) : (ls & 1);
        mbar_wait(&pempty[buf], bph ^ 1);
        mbar_arrive_expect_tx(&pfull[buf], p.nb * p.pimg * 4);   // exact box bytes (the buffer is rounded up)
        tma_load_4d(reinterpret_cast<uint8_t*>(sP) + buf * p.patch_bytes, &p.xmap, &pfull[buf], g.c0, 2 * g.i, 0, g.b0);
        C1F_STAMP(0, ls);
      }
    }
  } else if (warp >= C1_BUILD_WARP0 && warp < C1_EPI_WARP0) {
    // ======================= B builders: im2col rows of the set, straight from the NCHW images into
    // the 128B-swizzled K-major layout (row n = pixel, 32 tf32 per 128 B row, 16 B chunk j of row n at
    // chunk position j ^ (n & 7))
    const int t = threadIdx.x - C1_BUILD_WARP0 * 32;   // 0..C1_BUILD_THREADS-1
    const int grp = t & 7;                              // 16 B chunk (4 K columns) of the row
    // this thread's patch offsets (K columns grp*4 .. +3 of every 32-wide chunk), in registers
    int offr[C1_MAXK / 32][4];
#pragma unroll
    for (int c = 0; c < C1_MAXK / 32; ++c)
#pragma unroll
      for (int q = 0; q < 4; ++q) offr[c][q] = c < p.nch ? off_s[c * 32 + grp * 4 + q] : -1;
    for (int ls = 0; ls < wk.nset; ++ls) {
      const SetGeo g = set_geo(p, wk.set0 + ls * wk.step);
      const int buf = p.nbuf == 2 ? (ls & 1) : 0;
      const uint32_t bph = p.nbuf == 2 ? ((ls >> 1) & 1) : (ls & 1);
      mbar_wait(&pfull[buf], bph);
      mbar_wait(&bempty[buf], bph ^ 1);
      if (t == 0) C1F_STAMP(1, ls);
#if defined(C1_EXP) && C1_EXP == 3
      if (true) {   // experiment: no B build (timing only)
        asm volatile("bar.sync 1, %0;" ::"n"(C1_BUILD_THREADS) : "memory");
        if (t == 0) {
          mbar_arrive(&bfull[buf]);
          mbar_arrive(&pempty[buf]);
        }
        continue;
      }
#endif
      uint8_t* base = sB + buf * p.bset_bytes;
      const float* patch = sP + buf * (p.patch_bytes / 4);
      const int rows_per_img = 2 * g.ws;
      const int nreal = p.nb * rows_per_img;
      constexpr int RSTEP = C1_BUILD_THREADS / 8;     // rows per builder pass (8 threads per 128 B row)
      int n = t >> 3, bl = n / rows_per_img, rem = n - bl * rows_per_img;   // (image, row, column) of row n,
      for (; n < g.n; n += RSTEP) {                                          // stepped (no division per row)
        const int dh = rem >= g.ws ? 1 : 0, cc = rem - dh * g.ws;
        const bool real = n < nreal;                   // padded images read zeros from the patch (OOB fill)
        const float* src = patch + bl * p.pimg + dh * p.pw + cc;
        uint8_t* drow = base + n * 128 + ((grp ^ (n & 7)) << 4);
#pragma unroll
        for (int c = 0; c < C1_MAXK / 32; ++c) {
          if (c >= p.nch) break;
          float v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int o = offr[c][q];
            const float x = (real && o >= 0) ? src[o] : 0.f;
            v[q] = tf32_round(x);
          }
          *reinterpret_cast<float4*>(drow + c * p.bstride) = make_float4(v[0], v[1], v[2], v[3]);
        }
        rem += RSTEP;
        while (rem >= rows_per_img) {
          rem -= rows_per_img;
          ++bl;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
      asm volatile("bar.sync 1, %0;" ::"n"(C1_BUILD_THREADS) : "memory");
      if (t == 0) {
        C1F_STAMP(2, ls);
        mbar_arrive(&bfull[buf]);
        mbar_arrive(&pempty[buf]);
      }
    }
  } else if (warp >= C1_EPI_WARP0) {
    // ======================= epilogue: lane = own kernel, columns = (image, row dh, column)
    const int quad = warp & 3, egrp = (warp - C1_EPI_WARP0) >> 2;
    const int k = quad * 32 + lane;                    // row of the M tile
    int u = 0;
    for (int ls = 0; ls < wk.nset; ++ls) {
      const SetGeo g = set_geo(p, wk.set0 + ls * wk.step);
      const int nblk = (g.ws + 15) / 16;               // 16-column blocks per row (8 pooling windows)
      const int mt_end = c1_mt_end(wk, ls, p.mtiles);
      for (int mt = c1_mt_begin(wk, ls); mt < mt_end; ++mt, ++u) {
        const int acc = u & 1;
        const int kk = mt * C1_BM + k;
        const float bs = (p.bias && kk < p.Kr) ? __ldg(p.bias + kk) : 0.f;
        mbar_wait(&tfull[acc], (u >> 1) & 1);
        tc_fence_after();
        const uint32_t tb = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * 256;
        const int st = p.Bp * p.Kc;                    // consecutive pooled columns are Bp*Kc apart
        for (int it = egrp; it < p.nb * nblk; it += C1_EPI_GROUPS) {
          const int bl = it / nblk, cb = it - bl * nblk;
          // the last block of a row ends at the row end (overlaps the previous one, no reads past N + 16)
          const int cs = (cb == nblk - 1) ? max(0, g.ws - 16) : cb * 16;
          const int col0 = bl * 2 * g.ws + cs;
          uint32_t r0[16], r1[16];
#if defined(C1_EXP) && C1_EXP == 2
          continue;   // experiment: no TMEM reads, no epilogue
#endif
          tmem_ld_x16_nowait(tb + col0, r0);
          tmem_ld_x16_nowait(tb + col0 + g.ws, r1);
          tmem_wait_ld();
#if defined(C1_EXP) && C1_EXP == 1
          if (r0[0] == 0x7fffffffu && r1[3] == 0x7fffffffu) p.out[0] = 1.f;   // experiment: loads only
          continue;
#endif
          const int bb = g.b0 + bl;
          if (kk >= p.Kc) continue;                    // rows past the own block (last M tile)
          const bool ok = bb < p.B && kk < p.Kr;       // padded image / padded kernel slot -> exact 0
          const int q_lo = (cb * 16 - cs) >> 1, q_hi = min(8, (g.ws - cs) >> 1);
          // window q of this block: output (i, (c0 + cs)/2 + q, bb, kk).  All 8 windows are computed
          // unconditionally (independent, interleavable), only the stores are predicated.
          const int64_t o0 = ((int64_t)(g.i * p.Wp + ((g.c0 + cs) >> 1)) * p.Bp + bb) * p.Kc + kk;
          float* op = p.out + o0;
          uint8_t* sp = p.saved + o0;
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const float z0 = __uint_as_float(r0[2 * q]) + bs, z1 = __uint_as_float(r0[2 * q + 1]) + bs;
            const float z2 = __uint_as_float(r1[2 * q]) + bs, z3 = __uint_as_float(r1[2 * q + 1]) + bs;
            // ReLU + 2x2 max-pool, first maximum in row-major order: scanning the raw values
            // with '>' from a floor of 0 selects exactly the first maximum of max(z, 0), code 0 when
            // every position is <= 0 (ReLU'(0) = 0 routes no gradient there; reading R7)
            float best = RELU ? 0.f : z0;
            uint32_t code = 0;
            if (RELU && z0 > best) best = z0;
            if (z1 > best) { best = z1; code = 1; }
            if (z2 > best) { best = z2; code = 2; }
            if (z3 > best) { best = z3; code = 3; }
#if defined(C1_EXP) && C1_EXP == 4
            if (__float_as_uint(best) == 0x7fffffffu && code == 7) op[0] = 0.f;   // experiment: no stores
            continue;
#endif
            if (q >= q_lo && q < q_hi) {
              op[q * st] = ok ? tf32_round(best) : 0.f;
              sp[q * st] = ok ? (uint8_t)code : (uint8_t)0;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[acc]);
#ifdef C1F_TRACE
        if (warp == C1_EPI_WARP0 && lane == 0 && mt == mt_end - 1) C1F_STAMP(4, ls);
#endif
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 512);
  }
}


// ---------------------------------------------------------------------------------------------------
// BACKWARD-FILTER of the image layer, fused with the epilogue backward:
//   dW[k][(r,s,ch)] = sum_{(p,q,b)} dY[(p,q),b,k] * X[b][ch][p+r][q+s],   db[k] = sum dY,
//   dY[(2i+dh, 2j+dw), b, k] = dA[(i,j),b,k] * [code(i,j,b,k) == 2dh+dw] * [y(i,j,b,k) > 0]
// without materialising dY (202 MB at the paper net) or the im2col rows.  GEMM D[col][k] over
// K = (window (i,j), image, window position): M = the im2col columns (<= 128 TMEM lanes), N = one
// 256-kernel tile of the own kernels per CTA, one 32-deep K chunk = one pooling window x 8 images x
// its 4 positions (kk = 4 * image + position).  Both operands are built in shared memory by 12 builder
// warps straight from dA / codes / y and the NCHW images (K-major, 128B-swizzled): per (kernel, image)
// the routed gradient of the four window positions is one float4 (only the argmax position is non-zero),
// per (column, image) the four positions' input pixels likewise.  The builders form 2-4 groups that
// fill different ring stages, so that many chunks' global loads are in flight at once.  Split-K: the
// CTAs are (N tile, K range) pairs over contiguous chunk ranges; per-CTA partial dW / db go to a
// workspace and conv1_wgrad_reduce adds them in K-range order (deterministic).
#ifndef C1W_AWARPS
#define C1W_AWARPS 12  // A builder warps: 4 -> 8 -> 12 (1024 threads): conv1 backward-filter 65.5 -> 63.5 -> 61.5 us at P=1
#endif
constexpr int W1_BWARP0 = 4, W1_BWARPS = 16;  // warps 4..19 build B (2 threads per kernel, 4 images each),
                                              // warps 4..7 also run the final epilogue
constexpr int W1_AWARP0 = 20, W1_AWARPS = C1W_AWARPS;  // warps 20.. build A
constexpr int W1_THREADS = 32 * (W1_AWARP0 + W1_AWARPS);
constexpr int W1_MAXKC = 512;

struct W1Params {
  CUtensorMap damap, ymap;   // dA / y own blocks as rows (i,j,b) x Kc, box {256, 8}
  CUtensorMap xmap;          // images (W, H, C, B), box {8, R+1, C, 8}: one window's input patch
  const uint8_t* codes;      // argmax codes [Hp][Wp][Bp][Kc] (rows of a chunk copied in bulk)
  float* part;               // [nkr][Kc][Kcol] partial dW of every K range
  float* dbpart;             // [nkr][2][Kc] partial db (image halves of a chunk)
  int B, Bp, C, H, W, Hp, Wp, Kc, Kcol, ncolr;   // ncolr = R*S*C real im2col columns
  int nchunks, ngrp8, ntile, nkr, tile_bytes, raw_off_y, raw_off_c, raw_off_x, raw_bytes;
  int tstages, rstages;      // built-tile ring (released by the MMAs) and raw-input ring (released by the builders)
  int tstage_bytes, rstage_bytes;
  int xpw, pimg;             // patch row width (>= S + 1, x4) and floats of one image's patch C * (R+1) * xpw
  int relu, round;
  int off[C1_MAXK];          // im2col column -> (ch*(R+1) + r)*8 + s inside an image's patch
#ifdef C1W_TRACE
  unsigned long long* trace;   // experiment builds: CTA 0's per-chunk %globaltimer stamps [4][64]
#endif
};
#ifdef C1W_TRACE
#define C1W_STAMP(kind, c)                                                                               \
  do {                                                                                                    \
    if (blockIdx.x == 0 && (c) - c_begin < 64) p.trace[(kind) * 64 + ((c) - c_begin)] = globaltimer_ns(); \
  } while (0)
#else
#define C1W_STAMP(kind, c) do { } while (0)
#endif

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(W1_THREADS, 1) conv1_wgrad_kernel(const __grid_constant__ W1Params p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  // tile stage t: [A tile 16 KB][B tile <= 256 x 128 B]; raw stage r: [dA 8 KB | y 8 KB | codes 8 x Kc B |
  // x patch].  Two rings: the raw inputs run several chunks ahead of the builders (their slots are released
  // as soon as the builders have read them), the built tiles are released by the MMAs.
  uint8_t* raws = smem + p.tstages * p.tstage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(raws + p.rstages * p.rstage_bytes);
  uint64_t* rfull = bars;         // [rstages] raw inputs landed (TMA / bulk)
  uint64_t* rempty = bars + 8;    // [rstages] raw inputs read by every builder warp
  uint64_t* full = bars + 16;     // [tstages] tiles built
  uint64_t* empty = bars + 24;    // [tstages] MMAs done
  uint64_t* tfull = bars + 32;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 33);
  int* off_s = reinterpret_cast<int*>(bars + 34);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = blockIdx.x % p.ntile, kr = blockIdx.x / p.ntile;
  const int k0 = nt * 256, nN = min(256, p.Kc - k0);
  for (int k = threadIdx.x; k < C1_MAXK; k += blockDim.x) off_s[k] = p.off[k];
  // A rows >= ncolr stay zero for the whole kernel (columns past R*S*C)
  for (int st = 0; st < p.tstages; ++st)
    for (int e = threadIdx.x; e < (128 - p.ncolr) * 32; e += blockDim.x)
      reinterpret_cast<float*>(smem + st * p.tstage_bytes)[p.ncolr * 32 + e] = 0.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0 && lane == 0) {
    for (int st = 0; st < p.rstages; ++st) {
      mbar_init(&rfull[st], 1);
      mbar_init(&rempty[st], W1_BWARPS + W1_AWARPS);
    }
    for (int st = 0; st < p.tstages; ++st) {
      mbar_init(&full[st], W1_BWARPS + W1_AWARPS);
      mbar_init(&empty[st], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
    tma_prefetch(&p.damap);
    tma_prefetch(&p.ymap);
    tma_prefetch(&p.xmap);
  }
  if (warp == 2) tmem_alloc<1>(tmem_slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // this CTA's contiguous chunk range
  const int per = p.nchunks / p.nkr, extra = p.nchunks % p.nkr;
  const int c_begin = kr * per + min(kr, extra);
  const int c_end = c_begin + per + (kr < extra ? 1 : 0);

  if (warp == 0) {
    // ======================= raw-input producer: per chunk (window (i,j), 8 images) the gradient and
    // output rows of this CTA's kernels (2-D TMA), the code rows (bulk copy) and the input patch (TMA)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t bytes = 2 * 8 * 256 * 4 + 8 * p.Kc + 8 * p.pimg * 4;
      for (int c = c_begin; c < c_end; ++c) {
        const int win = c / p.ngrp8, b0 = (c - win * p.ngrp8) * 8;
        const int i = win / p.Wp, j = win - i * p.Wp;
        const int row = win * p.Bp + b0;
        mbar_wait(&rempty[stage], phase ^ 1);
        uint8_t* rw = raws + stage * p.rstage_bytes;
        mbar_arrive_expect_tx(&rfull[stage], bytes);
        tma_load_2d(rw, &p.damap, &rfull[stage], k0, row);
        tma_load_2d(rw + p.raw_off_y, &p.ymap, &rfull[stage], k0, row);
        bulk_load(rw + p.raw_off_c, p.codes + (int64_t)row * p.Kc, 8 * p.Kc, &rfull[stage]);
        // (TMA: the innermost box coordinate must be 16-byte aligned -> start at the 4-float boundary at or
        // below column 2j; the builders add the shift (2j) & 3)
        tma_load_4d(rw + p.raw_off_x, &p.xmap, &rfull[stage], (2 * j) & ~3, 2 * i, 0, b0);
        C1W_STAMP(0, c);
        if (++stage == p.rstages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t idesc = idesc_tf32(128, nN, 0, 0);
      for (int c = c_begin; c < c_end; ++c) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        C1W_STAMP(1, c);
        const uint32_t a = smem_u32(smem + stage * p.tstage_bytes);
        const uint64_t ad = sdesc_k(a, 0), bd = sdesc_k(a + 128 * 128, 0);
#pragma unroll
        for (int k = 0; k < 4; ++k) mma_tf32(tmem_base, ad + 2 * k, bd + 2 * k, idesc, (c > c_begin || k > 0) ? 1u : 0u);
        mma_commit(&empty[stage]);
        if (++stage == p.tstages) {
          stage = 0;
          phase ^= 1;
        }
      }
      mma_commit(tfull);
    }
  } else if (warp >= W1_BWARP0 && warp < W1_BWARP0 + W1_BWARPS) {
    // ======================= B builders: thread = kernel kl of the tile; per chunk the 8 images' routed,
    // ReLU-masked gradients of the window's 4 positions (one float4 per image: only the argmax position
    // is non-zero), read from the staged rows
    const int tb = threadIdx.x - W1_BWARP0 * 32;       // 0..511
    const int kl = tb & 255, half = tb >> 8;            // kernel of the tile, images 4*half .. 4*half+3
    const bool active = kl < nN;
    float dbacc = 0.f;
    int rstage = 0, tstage = 0;
    uint32_t rphase = 0, tphase = 0;
    for (int c = c_begin; c < c_end; ++c) {
      mbar_wait(&rfull[rstage], rphase);
      if (threadIdx.x == W1_BWARP0 * 32) C1W_STAMP(2, c);
      mbar_wait(&empty[tstage], tphase ^ 1);          // the tile slot's previous MMAs are done
      if (threadIdx.x == W1_BWARP0 * 32) C1W_STAMP(3, c);
      const uint8_t* rw = raws + rstage * p.rstage_bytes;
      const float* rda = reinterpret_cast<const float*>(rw);
      const float* ry = reinterpret_cast<const float*>(rw + p.raw_off_y);
      const uint8_t* rc = rw + p.raw_off_c + k0;
      uint8_t* sb = smem + tstage * p.tstage_bytes + 128 * 128;
      if (active) {
        float g[4], yv[4];
        uint32_t cd[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int bb = half * 4 + q;
          g[q] = rda[bb * 256 + kl];
          yv[q] = ry[bb * 256 + kl];
          cd[q] = rc[bb * p.Kc + kl];
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int bb = half * 4 + q;
          const float gv = (p.relu && !(yv[q] > 0.f)) ? 0.f : g[q];
          dbacc += gv;
          // the four window positions of image bb: zero, then the routed value at the argmax position
          uint8_t* dst = sb + kl * 128 + ((bb ^ (kl & 7)) << 4);
          *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
          *reinterpret_cast<float*>(dst + 4 * cd[q]) = tf32_round(gv);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&full[tstage]);
        mbar_arrive(&rempty[rstage]);
      }
      if (++rstage == p.rstages) {
        rstage = 0;
        rphase ^= 1;
      }
      if (++tstage == p.tstages) {
        tstage = 0;
        tphase ^= 1;
      }
    }
    if (active) p.dbpart[((int64_t)kr * 2 + half) * p.Kc + k0 + kl] = dbacc;   // this K range's db (chunks ascending)
    if (warp < W1_BWARP0 + 4) {
      // ======================= epilogue (warps 4..7): partial dW^T from TMEM, lane = im2col column
      const int quad = warp & 3;
      const int col = quad * 32 + lane;
      mbar_wait(tfull, 0);
      tc_fence_after();
      const uint32_t tb = tmem_base + ((uint32_t)(quad * 32) << 16);
      if (quad * 32 < p.Kcol) {
        float* dst = p.part + ((int64_t)kr * p.Kc + k0) * p.Kcol + col;
        for (int c0 = 0; c0 < nN; c0 += 32) {
          uint32_t r[32];
          tmem_ld_x32_nowait(tb + c0, r);
          tmem_wait_ld();
          if (col < p.Kcol) {
            float* d = dst + (int64_t)c0 * p.Kcol;
#pragma unroll
            for (int q = 0; q < 32; ++q)
              if (c0 + q < nN) d[q * p.Kcol] = __uint_as_float(r[q]);
          }
        }
      }
    }
  } else if (warp >= W1_AWARP0) {
    // ======================= A builders: item = (im2col column, image): the window's 4 input pixels
    const int t = threadIdx.x - W1_AWARP0 * 32;        // 0 .. 32 * W1_AWARPS - 1
    int rstage = 0, tstage = 0;
    uint32_t rphase = 0, tphase = 0;
    int win = c_begin / p.ngrp8, bg = c_begin - win * p.ngrp8, jw = win % p.Wp;   // stepped per chunk
    for (int c = c_begin; c < c_end; ++c) {
      const int jsh = (2 * jw) & 3;                    // column shift of the aligned patch
      if (++bg == p.ngrp8) {
        bg = 0;
        if (++jw == p.Wp) jw = 0;
      }
      mbar_wait(&rfull[rstage], rphase);
      mbar_wait(&empty[tstage], tphase ^ 1);
      uint8_t* st = smem + tstage * p.tstage_bytes;
      const float* rx = reinterpret_cast<const float*>(raws + rstage * p.rstage_bytes + p.raw_off_x) + jsh;
      for (int it = t; it < p.ncolr * 8; it += 32 * W1_AWARPS) {
        const int col = it >> 3, bb = it & 7;
        const float* src = rx + bb * p.pimg + off_s[col];
        float4 v = make_float4(src[0], src[1], src[p.xpw], src[p.xpw + 1]);   // (dh,dw) = (0,0),(0,1),(1,0),(1,1)
        v = make_float4(tf32_round(v.x), tf32_round(v.y), tf32_round(v.z), tf32_round(v.w));
        *reinterpret_cast<float4*>(st + col * 128 + ((bb ^ (col & 7)) << 4)) = v;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&full[tstage]);
        mbar_arrive(&rempty[rstage]);
      }
      if (++rstage == p.rstages) {
        rstage = 0;
        rphase ^= 1;
      }
      if (++tstage == p.tstages) {
        tstage = 0;
        tphase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<1>(tmem_base, 256);
  }
}

// dW[k][col] = sum over the K ranges (ascending) of the partials; db[k] = sum over K ranges and builder
// groups.  Block = 32 outputs x 8 lanes: lane y sums K ranges y*per.. (all loads in flight when per <= 24,
// else batched 8 deep; the same ascending order either way), the 8 lane
// sums combine in fixed order (deterministic).
__global__ void __launch_bounds__(256) conv1_wgrad_reduce(const float* __restrict__ part, const float* __restrict__ dbpart,
                                                          float* __restrict__ dw, float* __restrict__ db, int nkr,
                                                          int Kr, int Kc, int Kcol, float* __restrict__ sgd_w,
                                                          float* __restrict__ sgd_b, float lr) {
  __shared__ float red[8][33];
  const int e = blockIdx.x * 32 + threadIdx.x;
  const int n = Kr * Kcol;
  const bool is_w = e < n, is_b = db && e >= n && e < n + Kr;
  const float* src;
  int64_t stride;
  int cnt;
  if (is_w) {
    const int k = e / Kcol, col = e - k * Kcol;
    src = part + (int64_t)k * Kcol + col;
    stride = (int64_t)Kc * Kcol;
    cnt = nkr;
  } else {
    src = dbpart + (is_b ? e - n : 0);
    stride = Kc;
    cnt = 2 * nkr;
  }
  const int per = (cnt + 7) / 8, g0 = threadIdx.y * per, g1 = min(cnt, g0 + per);
  float t = 0.f;
  if (is_w || is_b) {
    int g = g0;
    if (g1 - g0 <= 24) {   // dW: <= 148 K ranges -> <= 19 per lane, every load in flight at once
      float v[24];
#pragma unroll
      for (int u = 0; u < 24; ++u) v[u] = g0 + u < g1 ? src[(g0 + u) * stride] : 0.f;
#pragma unroll
      for (int u = 0; u < 24; ++u)
        if (g0 + u < g1) t += v[u];
      g = g1;
    }
    for (; g + 8 <= g1; g += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[(g + u) * stride];
#pragma unroll
      for (int u = 0; u < 8; ++u) t += v[u];
    }
    for (; g < g1; ++g) t += src[g * stride];
  }
  red[threadIdx.y][threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.y == 0 && (is_w || is_b)) {
    float u = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < 8; ++k) u += red[k][threadIdx.x];
    if (is_w) {
      dw[e] = u;
      if (sgd_w) sgd_w[e] = fmaf(-lr, u, sgd_w[e]);   // fused SGD (final dW)
    } else {
      db[e - n] = u;
      if (sgd_b) sgd_b[e - n] = fmaf(-lr, u, sgd_b[e - n]);
    }
  }
}

}  // namespace


// Plan of the dedicated image-layer forward, or false when the shape is outside its envelope.
static bool c1_plan(const Layer& L, C1Params& p, size_t* smem) {
  if (!L.images || !L.d.pool || L.d.math != CP_MATH_TF32 || L.Kc == 0) return false;
  if (L.Kcol > C1_MAXK || (L.Ho & 1) || (L.Wo & 1) || L.Kcol % 8 || L.W % 4) return false;
  p.B = L.B; p.Bp = L.Bp; p.C = L.C; p.H = L.H; p.W = L.W; p.Ho = L.Ho; p.Wo = L.Wo; p.Hp = L.Hp; p.Wp = L.Wp;
  p.Kr = L.Kr; p.Kc = L.Kc; p.Kcol = L.Kcol; p.nch = (L.Kcol + 31) / 32;
  // B-set: nb images (power of two dividing Bp) x 2 rows x wseg columns, nb * 2 * wseg <= 224
  p.wseg = std::min(L.Wo, C1_NMAX / 2) & ~1;
  p.nseg = (L.Wo + p.wseg - 1) / p.wseg;
  p.nb = 1;
  const int nb_cap = tc_env_int("CP_C1_NB", 1 << 20);   // images per B-set cap (A/B; default: as many as fit)
  while (p.nb * 2 <= L.Bp && L.Bp % (p.nb * 2) == 0 && p.nb * 2 * 2 * p.wseg <= C1_NMAX && p.nb * 2 <= nb_cap)
    p.nb *= 2;
  p.ngrp = L.Bp / p.nb;
  p.nsets = L.Hp * p.nseg * p.ngrp;
  p.mtiles = (L.Kc + C1_BM - 1) / C1_BM;
  p.balance = tc_env_int("CP_C1_BALANCE", p.mtiles > 1 ? 1 : 0);
  p.bstride = (p.nb * 2 * p.wseg + 7) / 8 * 8 * 128;   // the widest set's N rows
  p.bset_bytes = p.nch * p.bstride;
  p.pw = (p.wseg + L.S - 1 + 3) / 4 * 4;
  // patch rows (channel, tap row) start pw floats apart; an odd number of 16-byte groups spreads the
  // builders' 8 K-column lanes over 8 bank groups (pw = 32 put them all on one bank: 8-way conflicts,
  // the per-set build took ~3.7 us; profiles/r02_conv1_fwd_trace.txt)
  if (((p.pw / 4) & 1) == 0 && tc_env_int("CP_C1_PAD", 1)) p.pw += 4;
  p.pimg = L.C * (L.R + 1) * p.pw;
  p.patch_bytes = (p.nb * p.pimg * 4 + 127) / 128 * 128;
  if (p.pw > 256 || L.R + 1 > 256 || L.C > 256 || p.patch_bytes > 32 * 1024) return false;
  const size_t fixed = 1024 + 8 * 32 + 4 * C1_MAXK + 256;
  const size_t cap = 227 * 1024;
  p.nbuf = 0;
  for (int nbuf = 2; nbuf >= 1 && !p.nbuf; --nbuf)
    for (int st = std::min(8, std::max(2, tc_env_int("CP_C1_ASTAGES", 4))); st >= 2; --st)
      if (fixed + (size_t)nbuf * (p.bset_bytes + p.patch_bytes) + (size_t)st * C1_ABYTES <= cap) {
        p.nbuf = nbuf;
        p.astages = st;
        break;
      }
  if (!p.nbuf) return false;
  *smem = fixed + (size_t)p.nbuf * (p.bset_bytes + p.patch_bytes) + (size_t)p.astages * C1_ABYTES;
  for (int kk = 0; kk < C1_MAXK; ++kk) {
    int o = -1;
    if (kk < L.R * L.S * L.C) {
      const int ch = kk % L.C, tap = kk / L.C, r = tap / L.S, s = tap % L.S;
      o = (ch * (L.R + 1) + r) * p.pw + s;
    }
    p.off[kk] = o;
  }
  return true;
}

bool c1_fwd_supported(const Layer& L) {
  if (!tc_env_int("CP_C1_FWD", 1)) return false;
  C1Params p{};
  size_t smem = 0;
  return c1_plan(L, p, &smem);
}

int c1_fwd(Layer& L, const float* x, const float* w, const float* b, float* y_block, uint8_t* saved, cudaStream_t s) {
  C1Params p{};
  size_t smem = 0;
  if (!c1_plan(L, p, &smem)) CP_FAIL(CP_ERR_UNSUPPORTED, "conv1 forward kernel: shape outside its envelope");
  {
    const uint64_t dims[2] = {(uint64_t)L.Kcol, (uint64_t)std::max(L.Kr, 1)};
    const uint64_t str[1] = {(uint64_t)L.Kcol * 4};
    const uint32_t box[2] = {32, (uint32_t)C1_BM};
    CP_TRY(tc_make_map(&p.wmap, w, 2, dims, str, box, false, 4));
  }
  {
    const uint64_t dims[4] = {(uint64_t)L.W, (uint64_t)L.H, (uint64_t)L.C, (uint64_t)L.B};
    const uint64_t str[3] = {(uint64_t)L.W * 4, (uint64_t)L.H * L.W * 4, (uint64_t)L.C * L.H * L.W * 4};
    const uint32_t box[4] = {(uint32_t)p.pw, (uint32_t)(L.R + 1), (uint32_t)L.C, (uint32_t)p.nb};
    CP_TRY(tc_make_map_plain(&p.xmap, x, 4, dims, str, box));
  }
  p.x = x;
  p.bias = L.d.bias ? b : nullptr;
  p.out = y_block;
  p.saved = saved;
  p.relu = L.d.relu;
  p.round = 1;
  static bool attr = false;
  if (!attr) {
    CP_CUDA(cudaFuncSetAttribute(conv1_fwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CP_CUDA(cudaFuncSetAttribute(conv1_fwd_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  const int grid = std::min(p.balance ? p.nsets * p.mtiles : p.nsets, tc_num_sms());
  CP_TRY(tc_time_mark(L, 0, 0, s));
#ifdef C1F_TRACE
  static unsigned long long* tbuf = nullptr;
  if (!tbuf) CP_CUDA(cudaMalloc(&tbuf, 5 * 8 * 8));
  CP_CUDA(cudaMemsetAsync(tbuf, 0, 5 * 8 * 8, s));
  p.trace = tbuf;
#endif
  if (p.relu) conv1_fwd_kernel<true><<<grid, C1_THREADS, smem, s>>>(p);
  else conv1_fwd_kernel<false><<<grid, C1_THREADS, smem, s>>>(p);
#ifdef C1F_TRACE
  {   // experiment build: CTA 0's per-set stamps (us after its first patch issue) to stderr
    unsigned long long h[5 * 8];
    CP_CUDA(cudaStreamSynchronize(s));
    CP_CUDA(cudaMemcpy(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[c1f_trace] Kc=%d mtiles=%d nsets=%d grid=%d astages=%d nbuf=%d: set patch_issued build_start "
                    "build_done mma_start epi_done\n", L.Kc, p.mtiles, p.nsets, grid, p.astages, p.nbuf);
    for (int k = 0; k < 8; ++k)
      if (h[k])
        fprintf(stderr, "[c1f_trace] %d %8.2f %8.2f %8.2f %8.2f %8.2f\n", k, (h[k] - h[0]) * 1e-3, (h[8 + k] - h[0]) * 1e-3,
                (h[16 + k] - h[0]) * 1e-3, (h[24 + k] - h[0]) * 1e-3, (h[32 + k] - h[0]) * 1e-3);
  }
#endif
  CP_LAUNCHED();
  CP_TRY(tc_time_mark(L, 0, 1, s));
  return CP_OK;
}

// Plan of the fused image-layer backward-filter, or false outside its envelope.
static bool w1_plan(const Layer& L, W1Params& p, size_t* smem, int* grid) {
  if (!L.images || !L.d.pool || L.d.math != CP_MATH_TF32 || L.Kr == 0) return false;
  if (L.Kc > W1_MAXKC || L.Kcol > 128 || L.Bp % 8 || (L.Ho & 1) || (L.Wo & 1) || L.S > 7 || L.W % 4) return false;
  p.B = L.B; p.Bp = L.Bp; p.C = L.C; p.H = L.H; p.W = L.W; p.Hp = L.Hp; p.Wp = L.Wp;
  p.Kc = L.Kc; p.Kcol = L.Kcol; p.ncolr = L.R * L.S * L.C;
  p.ngrp8 = L.Bp / 8;
  p.nchunks = L.Hp * L.Wp * p.ngrp8;
  p.ntile = (L.Kc + 255) / 256;
  p.nkr = std::max(1, std::min(p.nchunks, tc_num_sms() / p.ntile));
  p.xpw = (L.S + 1 + 3 + 3) / 4 * 4;   // S+1 columns after a shift of up to 3 (aligned box start)
  p.pimg = L.C * (L.R + 1) * p.xpw;
  p.tile_bytes = 128 * 128 + 256 * 128;                 // A + B (a full 256-row B tile)
  p.raw_off_y = 8 * 256 * 4;
  p.raw_off_c = 2 * 8 * 256 * 4;
  p.raw_off_x = (p.raw_off_c + 8 * L.Kc + 127) / 128 * 128;
  p.raw_bytes = p.raw_off_x + 8 * p.pimg * 4;
  p.tstage_bytes = (p.tile_bytes + 1023) / 1024 * 1024;
  p.rstage_bytes = (p.raw_bytes + 1023) / 1024 * 1024;
  const size_t fixed = 1024 + 512 + 4 * C1_MAXK + 256;
  // two built tiles (the MMA of one overlaps the build of the next); the rest of shared memory holds
  // raw-input stages so that the TMA loads run several chunks ahead (CP_C1W_RSTAGES caps it, A/B)
  p.tstages = 2;
  p.rstages = 0;
  const int rcap = std::max(2, std::min(8, tc_env_int("CP_C1W_RSTAGES", 8)));
  for (int st = rcap; st >= 2; --st)
    if (fixed + (size_t)p.tstages * p.tstage_bytes + (size_t)st * p.rstage_bytes <= 227 * 1024) {
      p.rstages = st;
      break;
    }
  if (!p.rstages) return false;
  *smem = fixed + (size_t)p.tstages * p.tstage_bytes + (size_t)p.rstages * p.rstage_bytes;
  *grid = p.ntile * p.nkr;
  for (int kk = 0; kk < C1_MAXK; ++kk) {
    int o = -1;
    if (kk < p.ncolr) {
      const int ch = kk % L.C, tap = kk / L.C, r = tap / L.S, s = tap % L.S;
      o = (ch * (L.R + 1) + r) * p.xpw + s;
    }
    p.off[kk] = o;
  }
  return true;
}

bool c1_wgrad_supported(const Layer& L) {
  if (!tc_env_int("CP_C1_WGRAD", 1)) return false;
  W1Params p{};
  size_t smem = 0;
  int grid = 0;
  return w1_plan(L, p, &smem, &grid);
}

size_t c1_wgrad_workspace(const Layer& L) {
  W1Params p{};
  size_t smem = 0;
  int grid = 0;
  if (!w1_plan(L, p, &smem, &grid)) return 0;
  return (size_t)p.nkr * L.Kc * L.Kcol * 4 + (size_t)p.nkr * 2 * L.Kc * 4 + 512;
}

int c1_wgrad(Layer& L, const float* x, const float* da, const uint8_t* codes, const float* y, float* dw, float* db,
             float* part, cudaStream_t s, float* sgd_w, float* sgd_b, float lr) {
  W1Params p{};
  size_t smem = 0;
  int grid = 0;
  if (!w1_plan(L, p, &smem, &grid)) CP_FAIL(CP_ERR_UNSUPPORTED, "conv1 wgrad kernel: shape outside its envelope");
  {
    const uint64_t dims[2] = {(uint64_t)L.Kc, (uint64_t)L.Hp * L.Wp * L.Bp};
    const uint64_t str[1] = {(uint64_t)L.Kc * 4};
    const uint32_t box[2] = {256, 8};
    CP_TRY(tc_make_map_plain(&p.damap, da, 2, dims, str, box));
    CP_TRY(tc_make_map_plain(&p.ymap, y, 2, dims, str, box));
  }
  {
    const uint64_t dims[4] = {(uint64_t)L.W, (uint64_t)L.H, (uint64_t)L.C, (uint64_t)L.B};
    const uint64_t str[3] = {(uint64_t)L.W * 4, (uint64_t)L.H * L.W * 4, (uint64_t)L.C * L.H * L.W * 4};
    const uint32_t box[4] = {(uint32_t)p.xpw, (uint32_t)(L.R + 1), (uint32_t)L.C, 8};
    CP_TRY(tc_make_map_plain(&p.xmap, x, 4, dims, str, box));
  }
  p.codes = codes;
  p.part = part;
  p.dbpart = part + (size_t)p.nkr * L.Kc * L.Kcol;
  p.relu = L.d.relu;
  p.round = 1;
  static bool attr = false;
  if (!attr) {
    CP_CUDA(cudaFuncSetAttribute(conv1_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
#ifdef C1W_TRACE
  static unsigned long long* tbuf = nullptr;
  if (!tbuf) CP_CUDA(cudaMalloc(&tbuf, 4 * 64 * 8));
  CP_CUDA(cudaMemsetAsync(tbuf, 0, 4 * 64 * 8, s));
  p.trace = tbuf;
#endif
  CP_TRY(tc_time_mark(L, 2, 0, s));
  conv1_wgrad_kernel<<<grid, W1_THREADS, smem, s>>>(p);
  CP_LAUNCHED();
#ifdef C1W_TRACE
  {   // experiment build: CTA 0's per-chunk stamps (ns after the first producer issue) to stderr
    unsigned long long h[4 * 64];
    CP_CUDA(cudaStreamSynchronize(s));
    CP_CUDA(cudaMemcpy(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost));
    const int nc = std::min(64, p.nchunks / p.nkr);
    fprintf(stderr, "[c1w_trace] Kc=%d nkr=%d chunks=%d rstages=%d: chunk producer_issued mma_start builder_raw builder_tile\n",
            L.Kc, p.nkr, nc, p.rstages);
    for (int c = 0; c < nc; ++c)
      fprintf(stderr, "[c1w_trace] %2d %8.2f %8.2f %8.2f %8.2f\n", c, (h[c] - h[0]) * 1e-3, (h[64 + c] - h[0]) * 1e-3,
              (h[128 + c] - h[0]) * 1e-3, (h[192 + c] - h[0]) * 1e-3);
  }
#endif
  CP_TRY(tc_time_mark(L, 2, 1, s));
  const int n = L.Kr * L.Kcol + (db ? L.Kr : 0);
  conv1_wgrad_reduce<<<(n + 31) / 32, dim3(32, 8), 0, s>>>(p.part, p.dbpart, dw, db, p.nkr, L.Kr, L.Kc, L.Kcol,
                                                           sgd_w, db ? sgd_b : nullptr, lr);
  CP_LAUNCHED();
  return CP_OK;
}

}  // namespace cp
