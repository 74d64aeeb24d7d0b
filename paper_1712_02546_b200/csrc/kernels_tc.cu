// kernels_tc.cu — the three convolution passes of a rank's kernel slice as implicit GEMMs on
// the 5th-generation tensor cores (tcgen05, kind::tf32, fp32 accumulation in TMEM), operands
// staged by TMA into 128B-swizzled shared memory through a 4-stage mbarrier ring.
//
//   FWD   (conv of own kernels, P:L175-177 / P:L212-214):
//         Z[(p,q,b)][k] = sum_{tap,c'} A_in[p+r][q+s][b][c'] * W[k][tap][c']  (+bias, ReLU, 2x2 pool)
//   DGRAD (input gradient of own kernels = the rank's partial dX, north_star):
//         dX[(h,w,b)][c'] = sum_{tap,k} dY[h-r][w-s][b][k] * W[k][tap][c']
//   WGRAD (weight gradient of own kernels, stays local, north_star):
//         dW[k][(tap,c')] = sum_{(p,q,b)} dY[p][q][b][k] * A_in[p+r][q+s][b][c']
//
// M tiles of 128 rows: FWD/DGRAD rows are one 2x2 spatial window x 32 images (a 4-D TMA box
// {32 ch, 32 b, 2 w, 2 h}), so a pooling window's four positions sit in the four TMEM lane
// quadrants, i.e. in the four epilogue warps; WGRAD rows are 128 kernels.  N tiles <= 256.
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM allocator, w4-7 epilogue.
// Persistent: grid = min(units, #SMs); two TMEM accumulators (2 x 256 columns) let the
// epilogue of tile t overlap the MMAs of tile t+1.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <vector>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace cp {
using namespace tc;

namespace {

enum { PASS_FWD = 0, PASS_DGRAD = 1, PASS_WGRAD = 2 };
// operand element size / elements per 128-byte K-chunk of a layer (bf16 mode: 2 / 64, else 4 / 32)
inline int op_bytes(const Layer& L) { return L.d.math == CP_MATH_BF16 ? 2 : 4; }
inline int op_elems(const Layer& L) { return 128 / op_bytes(L); }
constexpr int BM = 128, BN = 256, BK = 32;
constexpr int A_BYTES = BM * BK * 4;          // 16 KB: this CTA's 128 rows x 32 k
constexpr int NUM_THREADS = 384;             // w0 TMA, w1 MMA, w2 TMEM alloc, w3 idle, w4-w11 epilogue
constexpr int EPI_WARP0 = 4;
constexpr int EPI_GROUPS = 2;                // two 4-warp epilogue groups share the 32-column chunks
constexpr int POOL_LD = 33;                   // padded row of the pooling exchange buffer
constexpr int POOL_BYTES = 4 * 32 * POOL_LD * 4;
constexpr int MAX_NT = 64;
constexpr int MAX_WIN = 512;                  // dgrad LPT window table (larger grids: natural order)
constexpr int MAX_GROUPS = 148;               // CTA groups (one per SM or SM pair)
constexpr int MAX_SCHED = 1024;               // units in an explicit per-group schedule
constexpr int MAX_PIECES = 2 * MAX_GROUPS + 8;  // stream-tail pieces (<= one or two per CTA group)
constexpr int MAX_PAIRS = 1024;               // dgrad pixel-pair table entries (input grids up to 2048 pixels)

// CG = CTAs per MMA (cta_group::1 or ::2).  With a CTA pair the MMA is M=256 (128 rows per CTA)
// and each CTA stages only half of B (N/2 columns), so per-SM operand traffic drops by 1/3 and
// the freed shared memory buys a deeper ring.
template <int CG, int PASS>
struct Cfg {
  static constexpr int B_BYTES = CG == 1 ? BN * BK * 4 : (BN / 2) * BK * 4;
  // forward: pooling exchange; dgrad: per-warp transpose for full-line (NVLink) peer stores
  static constexpr int POOL = PASS != 2 ? EPI_GROUPS * POOL_BYTES : 0;
#ifndef CP_TC_STAGES_CG2
#define CP_TC_STAGES_CG2 6   // experiment hook (-D via CP_NVCC_EXTRA)
#endif
  static constexpr int STAGES = CG == 1 ? 4 : CP_TC_STAGES_CG2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = 1024 + (size_t)STAGES * STAGE_BYTES + POOL + 256;
};

// forward timing diagnostics (experiment builds only: CP_NVCC_EXTRA=-DCP_TC_DIAG_HOOK, then
// CP_TC_DIAG = 1 no MMAs / 2 no A loads / 4 no B loads; results are wrong) - compiled out otherwise
#ifdef CP_TC_DIAG_HOOK
#define TC_DIAG(p, bit) ((p).diag & (bit))
#else
#define TC_DIAG(p, bit) 0
#endif
// forward halo A boxes (negative result): compiled in only with -DCP_TC_HALO_HOOK, because
// even a never-taken runtime check on the single producer / MMA threads costs ~1 % of the forward
#ifdef CP_TC_HALO_HOOK
#define TC_HALO(p) ((p).halo)
#else
#define TC_HALO(p) 0
#endif

struct TcParams {
  CUtensorMap maps[CP_MAX_RANKS + 1];  // per-block input maps [0..nblk) ; maps[16] = W (fwd/dgrad) or dY (wgrad); dgrad A = maps[0]
  int nblk;
  int kw[CP_MAX_RANKS], coff[CP_MAX_RANKS];
  long long start[CP_MAX_RANKS];
  int Cg;              // concatenated input slots (or Kcol for images)
  int R, S;
  int Ho, Wo;          // conv output grid
  int Hin, Win;        // conv input grid
  int Wp;              // pooled width (fwd)
  int Bp, B;
  int Kr, Kc;          // own kernels / own slots
  int Ktot;            // weight row length
  int relu, pool, images;
  int numM, numN, split, units, chunks_per_split, chunks_total;  // numM counts M tiles per CTA group
  int bn_box;          // fwd: B box rows
  int nw;              // fwd: N tile width (balanced: Kc split into equal tiles)
  int nlim;            // fwd (kernels on N): this launch computes own slots [0, nlim) (split forward: < Kc)
  float* sgd_w;        // wgrad with the fused SGD update: the own weights (w -= sgd_lr * dW where dW is final)
  float sgd_lr;
  int m_off;           // fwd transposed: first own slot of M tile 0 (split forward: the remainder)
  int nsched_groups;   // multicast forward: clusters the host planned for (resident at once)
  int fcl;             // fwd transposed, multicast cluster (conv_tc_kernel<..., MC = 1>): CTAs per cluster = the
                       // slice's M tiles; a unit = one position tile for the whole cluster, its activation
                       // tile loaded once (each CTA a slice, TMA multicast to all), weights per CTA
  int epi_groups;      // 1 or 2 epilogue warp groups (blockDim = 128 + 128*groups; CP_TC_EPI_GROUPS)
  int max_chunks;      // longest K loop of a unit (after split), for the launch heuristics
  int wide;            // MN-major operands loaded as one 5-D box of 32-column atoms (else per-atom boxes)
  int span;            // dgrad/wgrad N tiles run over the concatenated slots of all input blocks
  int unified;         // equal-width input blocks: ONE tensor map (block = outermost dim) in maps[0]
                       // for fwd A / wgrad B, so the TMA unit does not cycle through P descriptors
  int apb;             // wgrad span: atoms per B box (every block width is a multiple of 32*apb)
  int cpt;             // fwd: K-chunks per tap (sum over input blocks)
  long long part_stride;  // split-K: floats between split partial buffers (fwd/dgrad)
  int nt_rb[MAX_NT], nt_n0[MAX_NT], nt_n[MAX_NT];  // dgrad / wgrad N-tile list (per tap for wgrad)
  int tail_full, tail_np;  // stream tail: units >= tail_full are pieces (tail unit, K-chunk range)
  short tail_tu[MAX_PIECES], tail_lo[MAX_PIECES], tail_hi[MAX_PIECES];
  float* tail_buf;     // wgrad tail partials [tail unit][piece][CTA of pair][128 rows][256 cols]
  int nsched;          // >0: per-group unit lists (host LPT schedule); 0: static round-robin
  short sched_off[MAX_GROUPS + 1];
  short sched[MAX_SCHED];
  int bke;             // operand elements per K-chunk (one 128-byte row): 32 tf32, 64 bf16
  int l2hint;          // dgrad: L2 evict_last on the weights, evict_first on dY (CP_TC_L2HINT)
  int pix;             // dgrad pixel mode: a CTA's 128 rows = 128 images of ONE input pixel, a pair = two
                       // horizontally adjacent pixels (exact valid rows, s-union only at borders)
  int nwin_order;      // dgrad: windows listed in win_order (0: natural order)
  int npairs;          // dgrad pixel mode: >0 = the pair table below (pixels paired by tap class), 0 = adjacent
                       // columns (2j, 2j+1); entry = i0 | w0 << 8 | i1 << 16 | w1 << 24 (CTA 0 / CTA 1 pixel)
  uint32_t pair_tab[MAX_PAIRS];
  int wg_taps_slow;    // wgrad unit order: 0 = N (tap, slot tile) fastest; 1 = slot tile, kernel tile, tap
  int diag;            // fwd timing diagnostics (CP_TC_DIAG; results are wrong): 1 no MMAs, 2 no A loads,
                       // 4 no B loads
  int fwdT;            // transposed forward (CTA-local, tf32): own kernels on M (128-row tiles), the 2x2
                       // window x 64 images on N = 256; the pool runs in each thread's registers
  int halo;            // fwd (CTA pairs, tf32): one A box per (input block, tap row, channel chunk) holds the
                       // window's 2 x (S+1) input pixels; the S column taps are 8 KB offsets into it
                       // (accumulator rows ordered (dw, dh, image) instead of (dh, dw, image))
  short win_order[MAX_WIN];
  const float* bias;
  float* out;          // fwd: y block ; dgrad: dx (full gather) ; wgrad: dW or split partials
  uint8_t* saved;
  float* peer_out[CP_MAX_RANKS];  // fwd with fused AllGather: the own block inside each peer's buffer
  int npeers;
  float* dst[CP_MAX_RANKS];  // dgrad with fused reduce-scatter: base of input block rb's partial (own
  int fused_dx;              // receive slot, or this rank's slot in peer rb's receive area over NVLink)
  const uint32_t* arrive;  // fwd over a symmetric gathered input: per-sender arrival counters (else null);
  int self_blk;            // the own input block (ready at launch) is consumed first, a peer's block
                           // only after its counter reached arrive_target - the gather overlaps this GEMM
  uint32_t arrive_target;
  // fused all-gather -> GEMM: warp 3 of every CTA pushes a share of this rank's own input block into
  // every peer's copy (push_chunks fixed-size chunks; one release-add on the peer's counter per chunk)
  const float* push_src;
  float* push_dst[CP_MAX_RANKS];
  uint32_t* push_cnt[CP_MAX_RANKS];
  unsigned long long* push_stamp;  // timing only: globaltimer window of the push (atomic min start / max end)
  int push_mc;             // 1: push_dst[0] / push_cnt[0] are NVLink multicast addresses (multimem)
  int push_warps;          // warps per CTA pushing (1: warp 3; 2: warps 2 and 3), CP_TC_PUSH_WARPS
  uint32_t* push_claim;    // chunk claim counter (zero at launch): any resident CTA's warp 3 takes the next
  int npush, push_chunks;  // (peer, chunk) pair, so the gather completes as long as one CTA runs per rank
  long long push_n4;
};

static_assert(sizeof(TcParams) <= 32000, "TcParams exceeds the kernel parameter limit");

struct Unit {
  int mt, nt, sp;
  uint32_t pix2;       // dgrad pixel mode: both CTAs' pixels, i0 | w0 << 8 | i1 << 16 | w1 << 24
  int tail, tu, piece; // wgrad: K-piece `piece` of tail unit `tu` (last-round units split over all groups)
  int i, j, bc;        // spatial window / batch chunk (fwd, dgrad)
  int n0, n;           // N origin (within own slots or block) and width
  int rb, tap;         // dgrad: output block; wgrad: input block and tap
};

// Unit u of this CTA group -> the tile of CTA `rank` (rank = 0 for CG=1).  With CG=2 the pair's
// two M tiles are two consecutive 32-image chunks of the same 2x2 window (FWD/DGRAD: identical
// tap lists, so both CTAs run the same K loop) or two consecutive 128-kernel tiles (WGRAD).
// forward accumulator quadrant (32-row group) <-> row-major 2x2 window position (dh*2 + dw): the
// identity, or (halo rows ordered (dw, dh, image)) the swap of the two bits - an involution
__host__ __device__ __forceinline__ int win_pos(int q, int halo) { return halo ? ((q & 1) << 1) | (q >> 1) : q; }

template <int PASS, int CG>
__device__ __forceinline__ Unit decode_unit(const TcParams& p, int u, int rank) {
  Unit t{};
  int mg;
  if ((PASS == PASS_WGRAD || PASS == PASS_FWD) && p.tail_np > 0 && u >= p.tail_full) {
    // the last (partial) round of equal tiles, its K-chunks shared evenly by every CTA group
    const int v = u - p.tail_full;
    t.tail = 1;
    t.tu = p.tail_tu[v];
    t.piece = v;
    u = p.tail_full + t.tu;
  }
  if (PASS == PASS_FWD && CG == 1 && p.fwdT) {   // (compiled out of the pair kernels)
    // kernel tile fastest (the units of a wave share the window's activation tile), then image chunk;
    // multicast cluster: the unit is the position tile, the kernel tile the CTA's rank in the cluster
    t.mt = p.fcl ? rank : u % p.numM;
    const int rest = p.fcl ? u : u / p.numM, nb = p.Bp / 64;
    t.bc = rest % nb;
    const int ij = rest / nb;
    t.j = ij % p.Wp;
    t.i = ij / p.Wp;
    t.n0 = p.m_off + t.mt * BM;
    t.n = BN;
    return t;
  }
  if (PASS == PASS_WGRAD && p.wg_taps_slow) {
    // taps slowest: a wave covers every kernel tile x a few adjacent taps, so the activation rows
    // it reads span one tap row (large maps: R rows of activations exceed L2, see wgrad_plan)
    const int per_tap = p.numN / (p.R * p.S);
    const int e = u % per_tap;
    const int rest = u / per_tap;
    mg = rest % p.numM;
    const int rest2 = rest / p.numM;
    t.nt = (rest2 % (p.R * p.S)) * per_tap + e;
    t.sp = rest2 / (p.R * p.S);
  } else if (PASS == PASS_WGRAD) {
    // N fastest: a wave covers few kernel tiles x many (tap, slot) tiles, so it streams one
    // kernel slice of dY and the (shared, shifted) activations once per position
    t.nt = u % p.numN;
    const int rest = u / p.numN;
    mg = rest % p.numM;
    t.sp = rest / p.numM;
  } else if (PASS == PASS_DGRAD && p.nwin_order > 0) {
    // heaviest windows first: all tiles of a window are consecutive units, windows in descending
    // order of valid taps (host-sorted), so round-robin dispatch approximates LPT scheduling
    t.sp = u % p.split;
    const int rest = u / p.split;
    t.nt = rest % p.numN;
    const int rest2 = rest / p.numN;
    const int nbcg = p.Bp / 32 / CG;
    mg = p.win_order[rest2 / nbcg] * nbcg + rest2 % nbcg;
  } else {
    mg = u % p.numM;
    const int rest = u / p.numM;
    t.nt = rest % p.numN;
    t.sp = rest / p.numN;
  }
  if (PASS == PASS_DGRAD && p.pix) {
    const int nbc = p.Bp / 128, W2 = p.Win / 2;
    t.bc = mg % nbc;                  // 128-image chunk
    const int ij = mg / nbc;
    if (p.npairs > 0) {               // pixels paired by tap class (host table)
      t.pix2 = p.pair_tab[ij];
    } else {                          // adjacent columns 2j (CTA 0), 2j+1 (CTA 1) of input row i
      const int i = ij / W2, w = 2 * (ij - i * W2);
      t.pix2 = (uint32_t)i | ((uint32_t)w << 8) | ((uint32_t)i << 16) | ((uint32_t)(w + 1) << 24);
    }
    t.i = rank ? (t.pix2 >> 16) & 0xff : t.pix2 & 0xff;          // this CTA's input pixel (row, column)
    t.j = rank ? t.pix2 >> 24 : (t.pix2 >> 8) & 0xff;
    t.mt = mg;
  } else if (PASS == PASS_FWD || PASS == PASS_DGRAD) {
    const int nbcg = p.Bp / 32 / CG;
    const int W2 = (PASS == PASS_FWD ? p.Wo : p.Win) / 2;
    t.bc = (mg % nbcg) * CG + rank;
    const int ij = mg / nbcg;
    t.j = ij % W2;
    t.i = ij / W2;
    t.mt = mg;
  } else {
    t.mt = mg * CG + rank;
  }
  if (PASS == PASS_FWD) {
    t.n0 = t.nt * p.nw;
    t.n = min(p.nw, p.nlim - t.n0);
  } else if (PASS == PASS_DGRAD) {
    t.rb = p.nt_rb[t.nt];
    t.n0 = p.nt_n0[t.nt];
    t.n = p.nt_n[t.nt];
  } else {
    const int per_tap = p.numN / (p.R * p.S);
    t.tap = t.nt / per_tap;
    const int e = t.nt % per_tap;
    t.rb = p.nt_rb[e];
    t.n0 = p.nt_n0[e];
    t.n = p.nt_n[e];
  }
  return t;
}

// k-th unit processed by CTA group `group`: the host's per-group list (LPT-balanced, see
// tc_dgrad) or static round-robin; -1 when the group is done.  Producer, MMA issuer and
// epilogue walk the identical sequence.
__device__ __forceinline__ int unit_at(const TcParams& p, int group, int ngroups, int k) {
  if (p.nsched > 0) {
    const int b = p.sched_off[group], e = p.sched_off[group + 1];
    return b + k < e ? (int)p.sched[b + k] : -1;
  }
  const int u = group + k * ngroups;
  return u < p.units ? u : -1;
}

// Visit the K-chunks of a unit in order: f(ksteps, c0..c3 of A, ...) is pass specific, so the
// visitor hands back the raw loop indices and both warps derive coordinates identically.
struct Chunk {
  int tap, rb, c;     // fwd: tap, input block, channel chunk ; dgrad: tap, -, kernel chunk ; wgrad: -, -, k-chunk index
  int ksteps;
  int r, s;           // fwd / dgrad: the tap's row and column
  int bc, q, pp;      // wgrad: 32-image chunk and output position of k-chunk c
  int first, last;    // fwd halo: first / last chunk of its (block, tap row, channel chunk) group in this walk
};
// (coordinates are produced by the loops themselves: the single TMA producer thread issues one
// chunk per ~900 cycles of MMA, so integer divisions on its path cost tensor-pipe time)

// dgrad: taps (r,s) whose shifted 2x2 window hits the dY grid: r in [r_lo, r_hi], s in [s_lo, s_hi]
__device__ __forceinline__ void dgrad_taps(const TcParams& p, const Unit& t, int& r_lo, int& nr, int& s_lo, int& ns) {
  int r_hi, s_hi;
  if (p.pix) {
    // pixel mode: the union of the pair's two pixels' valid tap boxes (both CTAs run one K loop)
    const int i0 = t.pix2 & 0xff, w0 = (t.pix2 >> 8) & 0xff, i1 = (t.pix2 >> 16) & 0xff, w1 = t.pix2 >> 24;
    r_lo = max(0, min(i0, i1) - p.Ho + 1);
    r_hi = min(p.R - 1, max(i0, i1));
    s_lo = max(0, min(w0, w1) - p.Wo + 1);
    s_hi = min(p.S - 1, max(w0, w1));
  } else {
    // window mode: input rows 2i, 2i+1 and columns 2j, 2j+1
    r_lo = max(0, 2 * t.i - p.Ho + 1);
    r_hi = min(p.R - 1, 2 * t.i + 1);
    s_lo = max(0, 2 * t.j - p.Wo + 1);
    s_hi = min(p.S - 1, 2 * t.j + 1);
  }
  nr = r_hi - r_lo + 1;
  ns = s_hi - s_lo + 1;
}

// Visit the K-chunks of split `t.sp` of a unit, in order.  A unit's chunk sequence is
// FWD: (tap, input block, 32-channel chunk); DGRAD: (32-kernel chunk, valid tap);
// WGRAD: (position, 32-image chunk).  Split sp covers [sp*per, (sp+1)*per) of it.
// DT: operand type (0 tf32, 1 bf16): a K-chunk is one 128-byte row of elements (BKE = 32 / 64),
// four MMA K-steps of KSE = 8 / 16 elements.
template <int PASS, int DT, class F>
__device__ __forceinline__ void for_each_chunk(const TcParams& p, const Unit& t, F f) {
  constexpr int BKE = DT ? 64 : 32, KSE = DT ? 16 : 8;
  if (PASS == PASS_FWD) {
    const int RS = p.R * p.S;
    const int total = RS * p.cpt;
    const int per = (total + p.split - 1) / p.split;
    const int lo = t.tail ? p.tail_lo[t.piece] : t.sp * per;
    const int hi = t.tail ? p.tail_hi[t.piece] : min(total, lo + per);
    if (lo >= hi) return;
    // decode chunk `lo` once, then step the coordinates (this loop runs on the single producer and
    // MMA threads, one iteration per ~900 tensor cycles)
    if (TC_HALO(p)) {
      // input blocks outermost (own block first when gathering), then tap row, channel chunk, and the
      // tap column innermost: the S column taps of a group share one A halo box
      const int S = p.S, R = p.R;
      int rb = p.arrive ? p.self_blk : 0, rem = lo;
      int nc = (p.kw[rb] + BKE - 1) / BKE;
      while (rem >= nc * R * S) {
        rem -= nc * R * S;
        rb = rb + 1 == p.nblk ? 0 : rb + 1;
        nc = (p.kw[rb] + BKE - 1) / BKE;
      }
      int r = rem / (nc * S);
      rem -= r * nc * S;
      int c = rem / S, sx = rem - c * S;
      int kw = p.kw[rb];
      for (int idx = lo; idx < hi; ++idx) {
        Chunk ch{r * S + sx, rb, c, min(BKE, kw - c * BKE) / KSE, r, sx, 0, 0, 0};
        ch.first = sx == 0 || idx == lo;
        ch.last = sx == S - 1 || idx == hi - 1;
        f(ch);
        if (++sx == S) {
          sx = 0;
          if (++c == nc) {
            c = 0;
            if (++r == R) {
              r = 0;
              do {
                rb = rb + 1 == p.nblk ? 0 : rb + 1;
                nc = (p.kw[rb] + BKE - 1) / BKE;
              } while (nc == 0);
              kw = p.kw[rb];
            }
          }
        }
      }
      return;
    }
    if (p.arrive) {
      // overlapped gather: input blocks outermost (own block first), then tap, then channel chunk
      int rb = p.self_blk, rem = lo;
      int nc = (p.kw[rb] + BKE - 1) / BKE;
      while (rem >= nc * RS) {
        rem -= nc * RS;
        rb = rb + 1 == p.nblk ? 0 : rb + 1;
        nc = (p.kw[rb] + BKE - 1) / BKE;
      }
      int tap = rem / nc, c = rem - tap * nc;
      int r = tap / p.S, sx = tap - r * p.S;
      int kw = p.kw[rb];
      for (int idx = lo; idx < hi; ++idx) {
        f(Chunk{tap, rb, c, min(BKE, kw - c * BKE) / KSE, r, sx, 0, 0, 0});
        if (++c == nc) {
          c = 0;
          ++tap;
          if (++sx == p.S) {
            sx = 0;
            ++r;
          }
          if (tap == RS) {
            tap = r = sx = 0;
            do {
              rb = rb + 1 == p.nblk ? 0 : rb + 1;
              nc = (p.kw[rb] + BKE - 1) / BKE;
            } while (nc == 0);
            kw = p.kw[rb];
          }
        }
      }
      return;
    }
    // tap outermost, then input block, then channel chunk
    int tap = lo / p.cpt, rem = lo - tap * p.cpt;
    int rb = 0, nc = (p.kw[0] + BKE - 1) / BKE;
    while (rem >= nc) {
      rem -= nc;
      ++rb;
      nc = (p.kw[rb] + BKE - 1) / BKE;
    }
    int c = rem, r = tap / p.S, sx = tap - r * p.S;
    int kw = p.kw[rb];
    for (int idx = lo; idx < hi; ++idx) {
      f(Chunk{tap, rb, c, min(BKE, kw - c * BKE) / KSE, r, sx, 0, 0, 0});
      if (++c == nc) {
        c = 0;
        do {
          if (++rb == p.nblk) {
            rb = 0;
            ++tap;
            if (++sx == p.S) {
              sx = 0;
              ++r;
            }
          }
          nc = (p.kw[rb] + BKE - 1) / BKE;
        } while (nc == 0 && tap < RS);
        kw = p.kw[rb];
      }
    }
  } else if (PASS == PASS_DGRAD) {
    int r_lo, nr, s_lo, ns;
    dgrad_taps(p, t, r_lo, nr, s_lo, ns);
    const int kc = (p.Kc + BKE - 1) / BKE;
    const int total = nr * ns * kc;
    const int per = (total + p.split - 1) / p.split;
    const int lo = t.sp * per, hi = min(total, lo + per);
    // kernel chunk outermost: all CTAs of a wave stream the same 32-kernel slice of W and dY at
    // the same time (a few MB live in L2) instead of every tap of the whole tensors.  Nested loops
    // with a running index: no integer division on the MMA issue path.
    if (lo >= hi) return;
    const int nt = nr * ns;
    int c = lo / nt, rem = lo - c * nt;
    int r = r_lo + rem / ns, sx = s_lo + rem % ns;
    for (int idx = lo; idx < hi; ++idx) {
      f(Chunk{r * p.S + sx, 0, c, min(BKE, p.Kc - c * BKE) / KSE, r, sx, 0, 0, 0});
      if (++sx == s_lo + ns) {
        sx = s_lo;
        if (++r == r_lo + nr) {
          r = r_lo;
          ++c;
        }
      }
    }
  } else {
    const int c0 = t.tail ? p.tail_lo[t.piece] : t.sp * p.chunks_per_split;
    const int c1 = t.tail ? p.tail_hi[t.piece] : min(p.chunks_total, c0 + p.chunks_per_split);
    // k-chunk c = (pq, bc): decoded once, then stepped
    const int nbc = p.Bp / BKE;
    int bc = c0 % nbc, pq = c0 / nbc;
    int q = pq % p.Wo, pp = pq / p.Wo;
    for (int c = c0; c < c1; ++c) {
      f(Chunk{0, 0, c, BKE / KSE, 0, 0, bc, q, pp});
      if (++bc == nbc) {
        bc = 0;
        if (++q == p.Wo) {
          q = 0;
          ++pp;
        }
      }
    }
  }
}

// MMA N for a tile of n columns: multiple of 8 (1 CTA) / 16 (pair); with a pair and MN-major B
// each CTA's half must be whole 32-column atoms, so N is rounded to 64 (extra columns are zero
// or neighbouring data and are never stored).
template <int PASS, int CG, int DT = 0>
__host__ __device__ __forceinline__ int mma_n(int n) {
  if (CG == 1) return (n + 7) / 8 * 8;
  if (PASS == PASS_FWD) return (n + 15) / 16 * 16;
  return DT ? (n + 127) / 128 * 128 : (n + 63) / 64 * 64;   // whole MN-major groups per CTA half
}

// w[q] -= lr * v[q] for q < n (the fused SGD update; same fma as cp_sgd)
__device__ __forceinline__ void sgd_f32x32(float* w, const float (&v)[32], int n, float lr) {
  if (n >= 32 && ((reinterpret_cast<uintptr_t>(w) & 15) == 0)) {
    float4 a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = reinterpret_cast<const float4*>(w)[q];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      a[q].x = fmaf(-lr, v[4 * q], a[q].x);
      a[q].y = fmaf(-lr, v[4 * q + 1], a[q].y);
      a[q].z = fmaf(-lr, v[4 * q + 2], a[q].z);
      a[q].w = fmaf(-lr, v[4 * q + 3], a[q].w);
      reinterpret_cast<float4*>(w)[q] = a[q];
    }
  } else {
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (q < n) w[q] = fmaf(-lr, v[q], w[q]);
  }
}

__device__ __forceinline__ void store_f32x32(float* dst, const float (&v)[32], int n) {
  if (n >= 32 && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < 32; ++q)
      if (q < n) dst[q] = v[q];
  }
}

template <int PASS, int CG, int DT, int MC>
__global__ void __launch_bounds__(NUM_THREADS, 1) conv_tc_kernel(const __grid_constant__ TcParams p) {
  // MC = 1 (PASS_FWD, CG = 1, transposed): clusters of p.fcl CTAs share each activation tile (multicast)
  // DT = 1: bf16 operands (kind::f16), a K-chunk = 64 elements; MN-major 64-element groups ("atoms")
  constexpr int BKE = DT ? 64 : 32;          // elements per 128-byte row = per K-chunk
  constexpr int ASH = DT ? 6 : 5;            // log2 of the MN-major group width
  constexpr int GBYTES = BKE * 128;          // bytes of one MN-major group (BKE rows x 128 B)
  using C = Cfg<CG, PASS>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base (128B swizzle atoms); offsetting the __shared__ array keeps the
  // pointer in the shared address space (ld/st.shared, not generic accesses)
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * A_BYTES;
  float* pool_all = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES + C::POOL);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = bars + 2 * C::STAGES + 2;
  uint64_t* afull = bars + 2 * C::STAGES + 4;    // fwd halo ring (2 stages in the A region)
  uint64_t* aempty = bars + 2 * C::STAGES + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 8);
  const int halo_bytes = (p.S + 1) * 8192;       // 2 rows x (S+1) columns x 32 images x 128 B

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_ctarank() : 0u;
  const uint32_t crank = MC ? cluster_ctarank() : rank;   // multicast cluster: this CTA's kernel tile
  const int CS = MC ? p.fcl : CG;                 // CTAs per unit group
  const int group = blockIdx.x / CS, ngroups = gridDim.x / CS;
  const uint16_t mc_mask = (uint16_t)((1u << CS) - 1u);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC ? CS : 1);          // multicast: every CTA of the cluster releases the stage
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4 * p.epi_groups * CG);
      mbar_init(&afull[a], 1);
      mbar_init(&aempty[a], 1);
    }
    fence_barrier_init();
    for (int m = 0; m < (p.unified ? 1 : p.nblk); ++m) tma_prefetch(&p.maps[m]);
    tma_prefetch(&p.maps[CP_MAX_RANKS]);
  }
  if (warp == 2) tmem_alloc<CG>(tmem_slot, 512);
  tc_fence_before();
  if (CG == 2 || MC) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ======================= TMA producer (both CTAs of a pair load their own halves)
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int ast = 0;                                   // fwd halo ring stage / phase
      uint32_t aph = 0;
      uint32_t arrived = PASS == PASS_FWD && p.arrive ? 1u << p.self_blk : ~0u;  // input blocks known present
      const uint64_t pol_keep = l2_policy(true), pol_stream = l2_policy(false);
      for (int k = 0;; ++k) {
        const int u = unit_at(p, group, ngroups, k);
        if (u < 0) break;
        const Unit t = decode_unit<PASS, CG>(p, u, MC ? crank : rank);
        const int n_mma = mma_n<PASS, CG, DT>(t.n);
        const int nb_own = CG == 2 ? n_mma / 2 : n_mma;          // B columns staged by this CTA
        const int nb0 = t.n0 + (int)rank * nb_own;                // first B column of this CTA
        const int nboxes = p.wide ? (CG == 2 ? 4 : 8) : (nb_own + 31) / 32;  // MN-major B: 32-column atoms
        const uint32_t tx_cta = PASS == PASS_FWD ? ((CG == 1 && !DT && p.fwdT) ? A_BYTES + BN * BK * 4
                                                           : (TC_DIAG(p, 2) ? 0 : A_BYTES) + (TC_DIAG(p, 4) ? 0 : p.bn_box * BK * 4))
                                                 : A_BYTES + nboxes * 4096;
        // wgrad span: input block and atom of every B box of this unit, once per unit
        int wb_n = 0, wb_rb[8], wb_atom[8];
        const int wg_r = PASS == PASS_WGRAD ? t.tap / p.S : 0, wg_s = PASS == PASS_WGRAD ? t.tap % p.S : 0;
        if (PASS == PASS_WGRAD && p.span) {
          for (int jb = 0; jb * p.apb * BKE < (CG == 2 ? BN / 2 : BN) && jb < 8; ++jb) {
            const int sl = nb0 + jb * p.apb * BKE;  // concatenated slot of this box
            int rb = 0;
            while (rb + 1 < p.nblk && sl >= p.coff[rb + 1]) ++rb;
            wb_rb[jb] = rb;
            wb_atom[jb] = (sl - p.coff[rb]) >> ASH;
            wb_n = jb + 1;
          }
        }
        for_each_chunk<PASS, DT>(p, t, [&](const Chunk& ch) {
          if (PASS == PASS_FWD && !DT && TC_HALO(p)) {
            if (ch.first) {
              if (!((arrived >> ch.rb) & 1u)) {
                wait_flag_sys(p.arrive + ch.rb, p.arrive_target);
                asm volatile("fence.proxy.async.global;" ::: "memory");
                arrived |= 1u << ch.rb;
              }
              mbar_wait(&aempty[ast], aph ^ 1);
              if (rank == 0) mbar_arrive_expect_tx(&afull[ast], (uint32_t)halo_bytes * CG);
              uint8_t* ah = sA + ast * halo_bytes;
              // box (32 slots, 32 images, 2 rows, S+1 columns): rows land as (column, row, image)
              if (CG == 2) {
                const uint32_t abar = mapa(smem_u32(&afull[ast]), 0);
                if (p.unified) tma_load_5d_cg2(ah, &p.maps[0], abar, ch.c * BKE, t.bc * 32, 2 * t.i + ch.r, 2 * t.j, ch.rb);
                else tma_load_4d_cg2(ah, &p.maps[ch.rb], abar, ch.c * BKE, t.bc * 32, 2 * t.i + ch.r, 2 * t.j);
              } else {
                if (p.unified) tma_load_5d(ah, &p.maps[0], &afull[ast], ch.c * BKE, t.bc * 32, 2 * t.i + ch.r, 2 * t.j, ch.rb);
                else tma_load_4d(ah, &p.maps[ch.rb], &afull[ast], ch.c * BKE, t.bc * 32, 2 * t.i + ch.r, 2 * t.j);
              }
            }
            mbar_wait(&empty[stage], phase ^ 1);
            if (rank == 0) mbar_arrive_expect_tx(&full[stage], (uint32_t)(p.bn_box * BK * 4) * CG);
            uint8_t* bh = sB + stage * C::B_BYTES;
            if (CG == 2)
              tma_load_2d_cg2(bh, &p.maps[CP_MAX_RANKS], mapa(smem_u32(&full[stage]), 0),
                              ch.tap * p.Cg + p.coff[ch.rb] + ch.c * BKE, nb0);
            else
              tma_load_2d(bh, &p.maps[CP_MAX_RANKS], &full[stage], ch.tap * p.Cg + p.coff[ch.rb] + ch.c * BKE, nb0);
            if (ch.last && ++ast == 2) {
              ast = 0;
              aph ^= 1;
            }
            if (++stage == C::STAGES) {
              stage = 0;
              phase ^= 1;
            }
            return;
          }
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* a = sA + stage * A_BYTES;
          uint8_t* b = sB + stage * C::B_BYTES;
          if (rank == 0) mbar_arrive_expect_tx(&full[stage], tx_cta * CG);
          const uint32_t lbar = CG == 2 ? mapa(smem_u32(&full[stage]), 0) : 0u;
          auto ld2 = [&](void* d, const CUtensorMap* m, int c0, int c1) {
            if (CG == 2) tma_load_2d_cg2(d, m, lbar, c0, c1); else tma_load_2d(d, m, &full[stage], c0, c1);
          };
          auto ld3 = [&](void* d, const CUtensorMap* m, int c0, int c1, int c2) {
            if (CG == 2) tma_load_3d_cg2(d, m, lbar, c0, c1, c2); else tma_load_3d(d, m, &full[stage], c0, c1, c2);
          };
          auto ld4 = [&](void* d, const CUtensorMap* m, int c0, int c1, int c2, int c3) {
            if (CG == 2) tma_load_4d_cg2(d, m, lbar, c0, c1, c2, c3);
            else tma_load_4d(d, m, &full[stage], c0, c1, c2, c3);
          };
          auto ld4h = [&](void* d, const CUtensorMap* m, int c0, int c1, int c2, int c3, uint64_t pol) {
            if (CG == 2) tma_load_4d_cg2_hint(d, m, lbar, c0, c1, c2, c3, pol);
            else tma_load_4d_hint(d, m, &full[stage], c0, c1, c2, c3, pol);
          };
          auto ld5 = [&](void* d, const CUtensorMap* m, int c0, int c1, int c2, int c3, int c4) {
            if (CG == 2) tma_load_5d_cg2(d, m, lbar, c0, c1, c2, c3, c4);
            else tma_load_5d(d, m, &full[stage], c0, c1, c2, c3, c4);
          };
          if (PASS == PASS_FWD) {
            const int r = ch.r, s = ch.s;
            if (!((arrived >> ch.rb) & 1u)) {
              wait_flag_sys(p.arrive + ch.rb, p.arrive_target);
              asm volatile("fence.proxy.async.global;" ::: "memory");  // peer-written data -> TMA reads
              arrived |= 1u << ch.rb;
            }
            if (CG == 1 && !DT && p.fwdT) {
              // A = the own kernels' weight rows (K-major), B = 4 window pixels x 64 images (K-major)
              ld2(a, &p.maps[CP_MAX_RANKS], ch.tap * p.Cg + p.coff[ch.rb] + ch.c * BKE, t.n0);
              if (MC) {
                // this CTA's slice of the activation tile (rows = image + 64 w + 128 h), multicast to the
                // cluster: 2 CTAs one h row each (maps[1], 128 rows); 3 CTAs h = 0 (maps[1]) and the two
                // pixels of h = 1 (maps[2], 64 rows); 4 CTAs one pixel each (maps[2])
                const int hh = CS == 2 ? (int)crank : CS == 3 ? (crank > 0) : (int)(crank >> 1);
                const int ww = CS == 2 ? 0 : CS == 3 ? (crank > 0 ? (int)crank - 1 : 0) : (int)(crank & 1);
                const bool half = CS == 2 || (CS == 3 && crank == 0);
                tma_load_5d_mc(b + (hh * 128 + ww * 64) * 128, &p.maps[half ? 1 : 2], &full[stage], ch.c * BKE,
                               t.bc * 64, 2 * t.j + s + ww, 2 * t.i + r + hh, ch.rb, mc_mask);
              } else if (p.unified) ld5(b, &p.maps[0], ch.c * BKE, t.bc * 64, 2 * t.j + s, 2 * t.i + r, ch.rb);
              else ld4(b, &p.maps[ch.rb], ch.c * BKE, t.bc * 64, 2 * t.j + s, 2 * t.i + r);
            } else if (TC_DIAG(p, 2)) {
            } else if (p.unified)
              ld5(a, &p.maps[0], ch.c * BKE, t.bc * 32, 2 * t.j + s, 2 * t.i + r, ch.rb);
            else
              ld4(a, &p.maps[ch.rb], ch.c * BKE, t.bc * 32, 2 * t.j + s, 2 * t.i + r);
            if (!TC_DIAG(p, 4) && !(CG == 1 && !DT && p.fwdT)) ld2(b, &p.maps[CP_MAX_RANKS], ch.tap * p.Cg + p.coff[ch.rb] + ch.c * BKE, nb0);
          } else if (PASS == PASS_DGRAD) {
            const int r = ch.r, s = ch.s;
            if (p.l2hint && p.pix)
              ld4h(a, &p.maps[0], ch.c * BKE, t.bc * 128, t.j - s, t.i - r, pol_stream);
            else if (p.pix)
              ld4(a, &p.maps[0], ch.c * BKE, t.bc * 128, t.j - s, t.i - r);
            else
              ld4(a, &p.maps[0], ch.c * BKE, t.bc * 32, 2 * t.j - s, 2 * t.i - r);
            if (p.wide) {
              if (p.l2hint)
                ld4h(b, &p.maps[CP_MAX_RANKS], 0, ch.c * BKE, ((p.span ? 0 : p.coff[t.rb]) + nb0) >> ASH, ch.tap, pol_keep);
              else
                ld4(b, &p.maps[CP_MAX_RANKS], 0, ch.c * BKE, ((p.span ? 0 : p.coff[t.rb]) + nb0) >> ASH, ch.tap);
            } else {
              for (int q = 0; q < nboxes; ++q)
                ld3(b + q * 4096, &p.maps[CP_MAX_RANKS], p.coff[t.rb] + nb0 + 32 * q, ch.c * BKE, ch.tap);
            }
          } else {
            const int bc = ch.bc, q = ch.q, pp = ch.pp;
            const int r = wg_r, s = wg_s;
            if (p.span) {
              ld5(a, &p.maps[CP_MAX_RANKS], 0, bc * BKE, t.mt * (BM >> ASH), q, pp);
              for (int jb = 0; jb < wb_n; ++jb) {   // boxes of this unit (block / atom hoisted per unit)
                if (p.unified)
                  ld5(b + jb * p.apb * GBYTES, &p.maps[0], 0, bc * BKE, wb_atom[jb], (pp + r) * p.Win + q + s, wb_rb[jb]);
                else
                  ld5(b + jb * p.apb * GBYTES, &p.maps[wb_rb[jb]], 0, bc * BKE, wb_atom[jb], q + s, pp + r);
              }
            } else if (p.wide) {
              ld5(a, &p.maps[CP_MAX_RANKS], 0, bc * BKE, t.mt * (BM >> ASH), q, pp);
              ld5(b, &p.maps[t.rb], 0, bc * BKE, nb0 >> ASH, q + s, pp + r);
            } else {
              for (int m = 0; m < 4; ++m)
                ld4(a + m * 4096, &p.maps[CP_MAX_RANKS], t.mt * BM + 32 * m, bc * 32, q, pp);
              for (int m = 0; m < nboxes; ++m)
                ld4(b + m * 4096, &p.maps[t.rb], nb0 + 32 * m, bc * 32, q + s, pp + r);
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        });
      }
      if (MC) {   // drain: every CTA of the cluster released every stage this CTA multicast into
        for (int i = 0; i < C::STAGES; ++i) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (one thread of the leader CTA)
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int ast = 0;
      uint32_t aph = 0;
      int local = 0;
      for (int k = 0;; ++k, ++local) {
        const int u = unit_at(p, group, ngroups, k);
        if (u < 0) break;
        const Unit t = decode_unit<PASS, CG>(p, u, 0);
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        const int n_mma = mma_n<PASS, CG, DT>(t.n);
        const int a_mn = PASS == PASS_WGRAD, b_mn = PASS != PASS_FWD;
        const uint32_t idesc = DT ? idesc_bf16(BM * CG, n_mma, a_mn, b_mn) : idesc_tf32(BM * CG, n_mma, a_mn, b_mn);
        uint32_t accumulate = 0;
        const bool halo = PASS == PASS_FWD && !DT && TC_HALO(p);
        for_each_chunk<PASS, DT>(p, t, [&](const Chunk& ch) {
          if (halo && ch.first) {
            mbar_wait(&afull[ast], aph);
            tc_fence_after();
          }
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = halo ? smem_u32(sA + ast * halo_bytes + ch.s * 8192) : smem_u32(sA + stage * A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
          // descriptors built once per chunk; a K-step only advances the start-address field
          // (16-byte units: +32 B K-major, +1024 B MN-major)
          // (bf16 MN-major: 64-element groups of BKE K-rows, +2048 B per K=16 step)
          const uint64_t ad0 = a_mn ? (DT ? sdesc_mn16(a_addr, 0, BKE) : sdesc_mn(a_addr, 0)) : sdesc_k(a_addr, 0);
          const uint64_t bd0 = b_mn ? (DT ? sdesc_mn16(b_addr, 0, BKE) : sdesc_mn(b_addr, 0)) : sdesc_k(b_addr, 0);
          const uint64_t mnstep = DT ? 128 : 64;
          const uint64_t astep = a_mn ? mnstep : 2, bstep = b_mn ? mnstep : 2;
          auto mma = [&](int k) {
            if (DT) {
              if (CG == 2) mma_bf16_cg2(d_tmem, ad0 + k * astep, bd0 + k * bstep, idesc, accumulate);
              else mma_bf16(d_tmem, ad0 + k * astep, bd0 + k * bstep, idesc, accumulate);
            } else {
              if (CG == 2) mma_tf32_cg2(d_tmem, ad0 + k * astep, bd0 + k * bstep, idesc, accumulate);
              else mma_tf32(d_tmem, ad0 + k * astep, bd0 + k * bstep, idesc, accumulate);
            }
            accumulate = 1;
          };
          if (PASS == PASS_FWD && TC_DIAG(p, 1)) {
          } else if (ch.ksteps == 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) mma(k);
          } else {
            for (int k = 0; k < ch.ksteps; ++k) mma(k);
          }
          if (CG == 2) mma_commit_cg2(&empty[stage]);
          else if (MC) mma_commit_mc(&empty[stage], mc_mask);   // every CTA that multicast into the stage
          else mma_commit(&empty[stage]);
          if (halo && ch.last) {
            if (CG == 2) mma_commit_cg2(&aempty[ast]); else mma_commit(&aempty[ast]);
            if (++ast == 2) {
              ast = 0;
              aph ^= 1;
            }
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        });
        if (CG == 2) mma_commit_cg2(&tfull[acc]); else mma_commit(&tfull[acc]);
      }
    }
  } else if (PASS == PASS_FWD && (warp == 3 || (warp == 2 && p.push_warps > 1))) {
    // ======================= gather pushers (otherwise idle warps 3 and 2 - the latter after its TMEM
    // allocation): this rank's input block -> peers,
    // full 512 B per warp store instruction, while the MMA warps consume the own block
    // peers in the order they consume this block (host-sorted: the peer that needs it soonest
    // first), all CTAs on one peer at a time so each peer's block completes as early as possible;
    // 8 float4 loads in flight per lane (the source block is L2-resident: just written)
    // Chunks are claimed dynamically (one atomic per chunk), not assigned by blockIdx: a peer's GEMM
    // spins on these arrivals, so the push must not depend on every CTA of this grid being resident
    // (other streams' kernels, MPS / green-context SM limits) - one running CTA finishes the gather.
    if (p.npush > 0) {
      const long long per = (p.push_n4 + p.push_chunks - 1) / p.push_chunks;
      const float4* src = reinterpret_cast<const float4*>(p.push_src);
      const int total = p.npush * p.push_chunks;
      unsigned long long t_first = 0, t_last = 0;
      for (;;) {
        int idx = 0;
        if (lane == 0) idx = (int)atomicAdd(p.push_claim, 1u);
        idx = __shfl_sync(0xffffffffu, idx, 0);
        if (idx >= total) break;
        if (p.push_stamp && !t_first) t_first = globaltimer_ns();
        const int k = idx / p.push_chunks, c = idx - k * p.push_chunks;
        float4* dst = reinterpret_cast<float4*>(p.push_dst[k]);
        {
          const long long b = (long long)c * per, e = min(p.push_n4, b + per);
          for (long long i = b + lane; i < e; i += 256) {
            float4 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
              if (i + 32 * u < e) v[u] = __ldg(src + i + 32 * u);
            if (p.push_mc) {
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (i + 32 * u < e)
                  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};"
                               :: "l"(dst + i + 32 * u), "f"(v[u].x), "f"(v[u].y), "f"(v[u].z), "f"(v[u].w)
                               : "memory");
            } else {
#pragma unroll
              for (int u = 0; u < 8; ++u)
                if (i + 32 * u < e) dst[i + 32 * u] = v[u];
            }
          }
          __threadfence_system();
          __syncwarp();
          if (lane == 0) {
            if (p.push_mc)
              asm volatile("multimem.red.release.sys.global.add.u32 [%0], %1;" :: "l"(p.push_cnt[k]), "n"(1) : "memory");
            else
              red_add_release_sys(p.push_cnt[k], 1u);
          }
        }
        if (p.push_stamp) t_last = globaltimer_ns();
      }
      if (p.push_stamp && t_first && lane == 0) {
        atomicMin(p.push_stamp, t_first);
        atomicMax(p.push_stamp + 1, t_last);
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ======================= epilogue: TMEM -> registers -> global (each CTA its own 128 rows)
    const int quad = warp & 3;                     // TMEM lane quadrant this warp may access
    const int grp = (warp - EPI_WARP0) >> 2;       // epilogue group: handles chunks cc = grp (mod 2)
    const int row = quad * 32 + lane;              // accumulator row of this CTA = TMEM lane
    float* pool_buf = pool_all + grp * (POOL_BYTES / 4);
    int local = 0;
    for (int k = 0;; ++k, ++local) {
      const int u = unit_at(p, group, ngroups, k);
      if (u < 0) break;
      const Unit t = decode_unit<PASS, CG>(p, u, MC ? crank : rank);
      const int acc = local & 1;
      const int nchunk = (t.n + 31) / 32;
      // forward bias of this unit's chunks (one column per lane), loaded before the accumulator wait
      // so the load latency overlaps it instead of stalling every chunk
      float bias_l[BN / 32];
      if (PASS == PASS_FWD) {
#pragma unroll
        for (int j = 0; j < BN / 32; ++j) {
          const int col = t.n0 + (grp + j * p.epi_groups) * 32 + lane;
          bias_l[j] = (p.bias && !t.tail && p.split == 1 && grp + j * p.epi_groups < nchunk && col < p.Kr)
                          ? __ldg(p.bias + col) : 0.f;
        }
      }
      mbar_wait(&tfull[acc], (local >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN;
      if (grp >= p.epi_groups) break;
      if (PASS == PASS_FWD && CG == 1 && !DT && p.fwdT) {
        // transposed forward: TMEM lane = own kernel slot, columns = (window position, image); group
        // grp takes images [32 grp, 32 grp + 32) of the unit's 64; bias + ReLU + first-max pool over
        // the four positions in registers, then one coalesced 128 B store per image (lanes = slots)
        const int kk = t.n0 + row;
        for (int h2 = grp; h2 < 2; h2 += p.epi_groups) {
          if (t.tail) {
            const int64_t tile = MC ? (int64_t)t.piece * CS + crank : (int64_t)t.piece;   // [piece][cluster rank]
            for (int pp = 0; pp < 4; ++pp) {
              float v[32];
              tmem_ld_32x32b_x32(tbase + (pp * 2 + h2) * 32, v);
              store_f32x32(p.tail_buf + (tile * BM + row) * BN + (pp * 2 + h2) * 32, v, 32);
            }
            continue;
          }
          const float bs = (p.bias && kk < p.Kr) ? __ldg(p.bias + kk) : 0.f;
          float best[32];
          uint32_t code[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) code[q] = 0;
#pragma unroll 1
          for (int pp = 0; pp < 4; ++pp) {
            float v[32];
            tmem_ld_32x32b_x32(tbase + (pp * 2 + h2) * 32, v);
#pragma unroll
            for (int q = 0; q < 32; ++q) {
              float x = v[q] + bs;
              if (p.relu && !(x > 0.f)) x = 0.f;
              if (pp == 0) {
                best[q] = x;
              } else if (x > best[q]) {
                best[q] = x;
                code[q >> 2] = (code[q >> 2] & ~(0xffu << (8 * (q & 3)))) | ((uint32_t)pp << (8 * (q & 3)));
              }
            }
          }
          if (kk < p.Kc) {
#pragma unroll
            for (int q = 0; q < 32; ++q) {
              const int bb = t.bc * 64 + h2 * 32 + q;
              const int64_t o = ((int64_t)(t.i * p.Wp + t.j) * p.Bp + bb) * p.Kc + kk;
              const bool ok = bb < p.B && kk < p.Kr;
              const float ov = ok ? tf32_rna(best[q]) : 0.f;
              p.out[o] = ov;
              p.saved[o] = ok ? (uint8_t)((code[q >> 2] >> (8 * (q & 3))) & 0xffu) : (uint8_t)0;
              for (int k = 0; k < p.npeers; ++k) p.peer_out[k][o] = ov;
            }
          }
        }
      } else
      for (int cc = grp, jb = 0; cc < nchunk; cc += p.epi_groups, ++jb) {
        float v[32];
        tmem_ld_32x32b_x32(tbase + cc * 32, v);
        const int ncol = min(32, t.n - cc * 32);
        if ((PASS == PASS_FWD || PASS == PASS_WGRAD) && t.tail) {
          // tail piece: raw partial tile, finished by fwd_tail_finish / wgrad_tail_reduce
          float* dst = p.tail_buf + (((int64_t)t.piece * CG + rank) * BM + row) * BN + cc * 32;
          store_f32x32(dst, v, 32);
        } else if (PASS == PASS_FWD && p.split > 1) {
          // split-K partial of the pre-pool tile: [sp][Ho][Wo][Bp][Kc]
          const int pos = win_pos(quad, TC_HALO(p));
          const int dh = pos >> 1, dw = pos & 1;
          const int bb = t.bc * 32 + lane;
          const int64_t o = (int64_t)t.sp * p.part_stride +
                            ((int64_t)((2 * t.i + dh) * p.Wo + 2 * t.j + dw) * p.Bp + bb) * p.Kc + t.n0 + cc * 32;
          store_f32x32(p.out + o, v, ncol);
        } else if (PASS == PASS_FWD) {
          const int nbase = t.n0 + cc * 32;  // own slot index of column 0
          // bias: one column per lane (preloaded), broadcast by shuffle
          float bl = 0.f;
#pragma unroll
          for (int j = 0; j < BN / 32; ++j)
            if (j == jb) bl = bias_l[j];
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            float x = v[q] + __shfl_sync(0xffffffffu, bl, q);
            if (p.relu && !(x > 0.f)) x = 0.f;
            v[q] = x;
          }
          if (p.pool) {
            // exchange through smem: quadrant = window position (dh, dw), lane = image
            float* mine = pool_buf + (quad * 32 + lane) * POOL_LD;
#pragma unroll
            for (int q = 0; q < 32; ++q) mine[q] = v[q];
            asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
            // write mapping: 8 threads per image row, 4 columns each - every warp store instruction
            // writes 4 full 128 B lines (NVLink peer stores are full-line packets, not masked pieces).
            // Scalar smem reads stay conflict-free: bank = (b + c4 + q) mod 32 covers all 32 banks.
            const int et = quad * 32 + lane;  // 0..127 within the group
            const int c4 = (et & 7) * 4;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int b = h * 16 + (et >> 3);
              const int bb = t.bc * 32 + b;
              float best[4];
              uint32_t code[4];
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                best[q] = pool_buf[(0 * 32 + b) * POOL_LD + c4 + q];
                code[q] = 0;
              }
#pragma unroll
              for (int w4 = 1; w4 < 4; ++w4)      // window positions in row-major order (first-max ties)
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  const float x = pool_buf[(win_pos(w4, TC_HALO(p)) * 32 + b) * POOL_LD + c4 + q];
                  if (x > best[q]) {
                    best[q] = x;
                    code[q] = w4;
                  }
                }
              const int64_t o = ((int64_t)(t.i * p.Wp + t.j) * p.Bp + bb) * p.Kc + nbase + c4;
              const bool real_b = bb < p.B;
              float ov[4];
              uint32_t packed = 0;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const bool ok = real_b && (nbase + c4 + q) < p.Kr;
                ov[q] = ok ? tf32_rna(best[q]) : 0.f;
                packed |= (ok ? code[q] : 0u) << (8 * q);
              }
              if (c4 + 4 <= ncol) {
                const float4 o4 = make_float4(ov[0], ov[1], ov[2], ov[3]);
                *reinterpret_cast<float4*>(p.out + o) = o4;
                *reinterpret_cast<uint32_t*>(p.saved + o) = packed;
                // fused channel AllGather: the same pooled values straight into every peer's copy of
                // the gathered output over NVLink (same offset: the gather layout is identical on all ranks)
                for (int k = 0; k < p.npeers; ++k) *reinterpret_cast<float4*>(p.peer_out[k] + o) = o4;
              } else {
                for (int q = 0; q < 4 && c4 + q < ncol; ++q) {
                  p.out[o + q] = ov[q];
                  p.saved[o + q] = (uint8_t)(packed >> (8 * q));
                  for (int k = 0; k < p.npeers; ++k) p.peer_out[k][o + q] = ov[q];
                }
              }
            }
            asm volatile("bar.sync %0, 128;" ::"r"(1 + grp) : "memory");
          } else {
            const int pos = win_pos(quad, TC_HALO(p));
            const int dh = pos >> 1, dw = pos & 1;
            const int bb = t.bc * 32 + lane;
            const int64_t o = ((int64_t)((2 * t.i + dh) * p.Wo + 2 * t.j + dw) * p.Bp + bb) * p.Kc + nbase;
            const bool real_b = bb < p.B;
#pragma unroll
            for (int q = 0; q < 32; ++q) v[q] = (real_b && nbase + q < p.Kr) ? tf32_rna(v[q]) : 0.f;
            store_f32x32(p.out + o, v, ncol);
            for (int k = 0; k < p.npeers; ++k) store_f32x32(p.peer_out[k] + o, v, ncol);
          }
        } else if (PASS == PASS_DGRAD) {
          const int dh = quad >> 1, dw = quad & 1;
          const int bb = t.bc * 32 + lane;
          int rb = t.rb, slot = t.n0 + cc * 32;
          if (p.span) {  // 32-column chunk -> its input block (block widths are multiples of 32)
            rb = 0;
            while (rb + 1 < p.nblk && slot >= p.coff[rb + 1]) ++rb;
            slot -= p.coff[rb];
          }
          if (p.fused_dx) {
            // fused reduce-scatter: the partial goes to block rb's owner (own slot locally, a peer's
            // over NVLink).  Warp-local transpose through shared memory so that every store
            // instruction writes 4 full 128 B rows (8 lanes x float4 each) instead of 32 pieces.
            float* tb = pool_buf + (quad & 3) * 32 * POOL_LD;   // this warp's 32 x 33 tile
#pragma unroll
            for (int q = 0; q < 32; ++q) tb[lane * POOL_LD + q] = v[q];
            __syncwarp();
            const bool chunk_ok = !p.span || slot < p.kw[rb];
            if (chunk_ok) {
              const int kw = p.kw[rb];
              const int c4 = (lane & 7) * 4;
              float* base = p.dst[rb] + (p.pix ? ((int64_t)(t.i * p.Win + t.j) * p.Bp + t.bc * 128 + quad * 32)
                                                : ((int64_t)((2 * t.i + dh) * p.Win + 2 * t.j + dw) * p.Bp + t.bc * 32)) * kw + slot;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const int row = k * 4 + (lane >> 3);
                float4 o4;
                o4.x = tb[row * POOL_LD + c4 + 0];
                o4.y = tb[row * POOL_LD + c4 + 1];
                o4.z = tb[row * POOL_LD + c4 + 2];
                o4.w = tb[row * POOL_LD + c4 + 3];
                float* d = base + (int64_t)row * kw + c4;
                if (c4 + 4 <= ncol) {
                  *reinterpret_cast<float4*>(d) = o4;
                } else if (c4 < ncol) {
                  const float e[4] = {o4.x, o4.y, o4.z, o4.w};
                  for (int q = 0; q < ncol - c4; ++q) d[q] = e[q];
                }
              }
            }
            __syncwarp();
          } else if (!p.span || slot < p.kw[rb]) {
            const int kw = p.kw[rb];
            const int64_t o = (int64_t)t.sp * p.part_stride + p.start[rb] +
                              (p.pix ? ((int64_t)(t.i * p.Win + t.j) * p.Bp + t.bc * 128 + row)
                                     : ((int64_t)((2 * t.i + dh) * p.Win + 2 * t.j + dw) * p.Bp + bb)) * kw + slot;
            store_f32x32(p.out + o, v, ncol);
          }
        } else {
          const int kk = t.mt * BM + row;
          if (kk < p.Kr) {
            const int64_t col = (int64_t)t.tap * p.Cg + (p.span ? 0 : p.coff[t.rb]) + t.n0 + cc * 32;
            const int64_t o = ((int64_t)t.sp * p.Kr + kk) * p.Ktot + col;
            store_f32x32(p.out + o, v, ncol);
            if (p.sgd_w) sgd_f32x32(p.sgd_w + o, v, ncol, p.sgd_lr);   // final dW (no split): fused SGD
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2) mbar_arrive_cluster(mapa(smem_u32(&tempty[acc]), 0));
        else mbar_arrive(&tempty[acc]);
      }
    }
    // peer stores (fused gather from the epilogue, fused dX reduce-scatter) performed system-wide before
    // exit; the flag release that follows in the next launch then orders after them
    if ((PASS == PASS_FWD && p.npeers > 0) || (PASS == PASS_DGRAD && p.fused_dx)) __threadfence_system();
  }
  tc_fence_before();
  if (CG == 2 || MC) cluster_sync(); else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<CG>(tmem_base, 512);
  }
}

// wgrad tail: dW[kk0 + row][col0 + c] = sum over pieces (in order) of the partial tiles.
constexpr int MAX_TAIL = 148;
struct TailInfo {
  int n;                      // tail units
  int cg;                     // CTAs per tile
  short pbeg[MAX_TAIL + 1];   // pieces of tail unit tu: [pbeg[tu], pbeg[tu+1]) in K order
  int Kr, Ktot;
  int kk0[MAX_TAIL];          // first kernel row of the unit's tile (CTA 0)
  int col0[MAX_TAIL];         // first dW column
  int ncol[MAX_TAIL];         // valid columns
  float* sgd_w;               // fused SGD: w -= sgd_lr * dW (nullptr: none)
  float sgd_lr;
};
__global__ void wgrad_tail_reduce(const float* __restrict__ buf, float* __restrict__ dw, const __grid_constant__ TailInfo ti) {
  const int tu = blockIdx.z, rank = blockIdx.y, row = blockIdx.x;
  const int c = threadIdx.x;  // 256 columns
  const int kk = ti.kk0[tu] + rank * BM + row;
  if (kk >= ti.Kr || c >= ti.ncol[tu]) return;
  // the unit's pieces in K order (fixed order); four accumulators keep loads in flight
  const int64_t step = (int64_t)ti.cg * BM * BN;
  const int np = ti.pbeg[tu + 1] - ti.pbeg[tu];
  const float* src = buf + (((int64_t)ti.pbeg[tu] * ti.cg + rank) * BM + row) * BN + c;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  int pc = 0;
  for (; pc + 8 <= np; pc += 8) {   // 8 loads in flight, added in the same order (piece p -> a[p & 3])
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = src[(pc + k) * step];
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k & 3] += v[k];
  }
  for (; pc < np; ++pc) a[pc & 3] += src[pc * step];
  const int64_t o = (int64_t)kk * ti.Ktot + ti.col0[tu] + c;
  const float d = (a[0] + a[1]) + (a[2] + a[3]);
  dw[o] = d;
  if (ti.sgd_w) ti.sgd_w[o] = fmaf(-ti.sgd_lr, d, ti.sgd_w[o]);
}

// forward tail: the tile's pre-pool accumulator = sum over pieces (in order) of the partial tiles;
// then bias, ReLU, 2x2 max-pool (rows q*32+b of a CTA's tile are window position q, image b),
// argmax code and RN-tf32 rounding, exactly as the fused epilogue.
struct FwdTailInfo {
  int halo;   // accumulator quadrants in halo order (win_pos)
  int n, cg, Wo, Wp, Bp, B, Kr, Kc, relu, pool, npeers;
  short pbeg[MAX_TAIL + 1];   // pieces of tail unit tu: [pbeg[tu], pbeg[tu+1])
  float* peer[CP_MAX_RANKS];  // fused AllGather: own block inside each peer's buffer
  int i[MAX_TAIL], j[MAX_TAIL], bc0[MAX_TAIL], n0[MAX_TAIL], ncol[MAX_TAIL];
};
// Sum of one accumulator value over the pieces [pc, pe) (stride pstep floats), in piece order; loads
// batched 16 at a time (the pieces were just written: L2-latency bound, ~20-75 pieces per tail unit)
__device__ __forceinline__ float tail_sum(const float* __restrict__ src, int np, int64_t pstep) {
  float z = 0.f;
  int pc = 0;
  for (; pc + 16 <= np; pc += 16) {
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = src[(pc + u) * pstep];
#pragma unroll
    for (int u = 0; u < 16; ++u) z += v[u];
  }
  for (; pc < np; ++pc) z += src[pc * pstep];
  return z;
}

// blockDim (BN columns, 4 accumulator quadrants): each thread sums one pre-pool value over the pieces
// (four times the threads of one thread per pooling window; the same order per value), the quadrants
// meet in shared memory for the pool.  For tails of few units with many pieces each (P=1: ~20 per
// unit, 8.1 -> 7.4 us); with many units of few pieces (P=8) the window-per-thread kernel below is
// faster (9.1 vs 26.9 us, profiles/r02_tail_finish/)
__global__ void __launch_bounds__(4 * BN) fwd_tail_finish_q(const float* __restrict__ buf, const float* __restrict__ bias,
                                                           float* __restrict__ y, uint8_t* __restrict__ saved,
                                                           const __grid_constant__ FwdTailInfo ti) {
  __shared__ float zs[4][BN];
  const int tu = blockIdx.z, rank = blockIdx.y, b = blockIdx.x;
  const int c = threadIdx.x, qa = threadIdx.y;
  const bool col = c < ti.ncol[tu];
  if (col) {
    const int pb = ti.pbeg[tu];
    const float* src = buf + ((int64_t)pb * ti.cg + rank) * BM * BN + (int64_t)(qa * 32 + b) * BN + c;
    zs[qa][c] = tail_sum(src, ti.pbeg[tu + 1] - pb, (int64_t)ti.cg * BM * BN);
  }
  __syncthreads();
  if (qa != 0 || !col) return;
  const int n = ti.n0[tu] + c;
  const int bb = ti.bc0[tu] + rank * 32 + b;
  const bool ok = bb < ti.B && n < ti.Kr;
  const float bs = (bias && n < ti.Kr) ? bias[n] : 0.f;
  float best = 0.f;
  int code = 0;
  for (int q = 0; q < 4; ++q) {             // q: row-major window position
    float z = zs[win_pos(q, ti.halo)][c] + bs;
    if (ti.relu && !(z > 0.f)) z = 0.f;
    if (ti.pool) {
      if (q == 0 || z > best) {
        best = z;
        code = q;
      }
    } else {
      const int64_t o = ((int64_t)((2 * ti.i[tu] + (q >> 1)) * ti.Wo + 2 * ti.j[tu] + (q & 1)) * ti.Bp + bb) * ti.Kc + n;
      y[o] = ok ? tf32_rna(z) : 0.f;
      for (int k = 0; k < ti.npeers; ++k) ti.peer[k][o] = ok ? tf32_rna(z) : 0.f;
    }
  }
  if (ti.pool) {
    const int64_t o = ((int64_t)(ti.i[tu] * ti.Wp + ti.j[tu]) * ti.Bp + bb) * ti.Kc + n;
    y[o] = ok ? tf32_rna(best) : 0.f;
    saved[o] = ok ? (uint8_t)code : 0;
    for (int k = 0; k < ti.npeers; ++k) ti.peer[k][o] = ok ? tf32_rna(best) : 0.f;
  }
  if (ti.npeers) __threadfence_system();
}

// one thread per pooling window (4 pre-pool values), 8 pieces' loads in flight
__global__ void fwd_tail_finish(const float* __restrict__ buf, const float* __restrict__ bias, float* __restrict__ y,
                                uint8_t* __restrict__ saved, const __grid_constant__ FwdTailInfo ti) {
  const int tu = blockIdx.z, rank = blockIdx.y, b = blockIdx.x;
  const int c = threadIdx.x;
  if (c >= ti.ncol[tu]) return;
  const int n = ti.n0[tu] + c;
  const int bb = ti.bc0[tu] + rank * 32 + b;
  const bool ok = bb < ti.B && n < ti.Kr;
  const float bs = (bias && n < ti.Kr) ? bias[n] : 0.f;
  float best = 0.f;
  int code = 0;
  float zq[4] = {0.f, 0.f, 0.f, 0.f};   // the four window positions: independent load streams
  // pieces in K order; loads of 8 pieces batched (32 in flight), added in the same order
  int pc = ti.pbeg[tu];
  const int pe = ti.pbeg[tu + 1];
  for (; pc + 8 <= pe; pc += 8) {   // (8 pieces: 32 loads in flight)
    float v[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float* src = buf + ((int64_t)(pc + u) * ti.cg + rank) * BM * BN + (int64_t)b * BN + c;
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = src[q * 32 * BN];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) zq[q] += v[u][q];
  }
  for (; pc < pe; ++pc) {
    const float* src = buf + ((int64_t)pc * ti.cg + rank) * BM * BN + (int64_t)b * BN + c;
#pragma unroll
    for (int q = 0; q < 4; ++q) zq[q] += src[q * 32 * BN];
  }
  for (int q = 0; q < 4; ++q) {             // q: row-major window position
    float z = zq[win_pos(q, ti.halo)] + bs;
    if (ti.relu && !(z > 0.f)) z = 0.f;
    if (ti.pool) {
      if (q == 0 || z > best) {
        best = z;
        code = q;
      }
    } else {
      const int64_t o = ((int64_t)((2 * ti.i[tu] + (q >> 1)) * ti.Wo + 2 * ti.j[tu] + (q & 1)) * ti.Bp + bb) * ti.Kc + n;
      y[o] = ok ? tf32_rna(z) : 0.f;
      for (int k = 0; k < ti.npeers; ++k) ti.peer[k][o] = ok ? tf32_rna(z) : 0.f;
    }
  }
  if (ti.pool) {
    const int64_t o = ((int64_t)(ti.i[tu] * ti.Wp + ti.j[tu]) * ti.Bp + bb) * ti.Kc + n;
    y[o] = ok ? tf32_rna(best) : 0.f;
    saved[o] = ok ? (uint8_t)code : 0;
    for (int k = 0; k < ti.npeers; ++k) ti.peer[k][o] = ok ? tf32_rna(best) : 0.f;
  }
  if (ti.npeers) __threadfence_system();
}

// stream-tail finish of the transposed forward: tile rows = own kernel slots, columns = (window
// position, image of 64); pieces summed in K order, then bias + ReLU + first-max pool.  One block
// per (tile row, tail unit), one thread per (image, window position).
__global__ void __launch_bounds__(256) fwd_tail_finish_t(const float* __restrict__ buf, const float* __restrict__ bias,
                                                         float* __restrict__ y, uint8_t* __restrict__ saved,
                                                         const __grid_constant__ FwdTailInfo ti) {
  // blockIdx.z: the M tile within a multicast cluster's unit (ti.cg tiles per piece; 1 otherwise).
  // 256 threads = 64 images x 4 window positions: one pre-pool value each, summed over the pieces in
  // K order (~74 per tail unit at the P=4 slice), the positions meet in shared memory for the pool
  __shared__ float zs[4][64];
  const int tu = blockIdx.y, row = blockIdx.x, mt = blockIdx.z;
  const int b = threadIdx.x & 63, q = threadIdx.x >> 6;
  const int kk = ti.n0[tu] + mt * BM + row;
  if (kk >= ti.Kc) return;
  const int pb = ti.pbeg[tu];
  const float* src = buf + (((int64_t)pb * ti.cg + mt) * BM + row) * BN + q * 64 + b;
  zs[q][b] = tail_sum(src, ti.pbeg[tu + 1] - pb, (int64_t)ti.cg * BM * BN);
  __syncthreads();
  if (q != 0) return;
  const int bb = ti.bc0[tu] + b;
  const bool ok = bb < ti.B && kk < ti.Kr;
  const float bs = (bias && kk < ti.Kr) ? bias[kk] : 0.f;
  float best = 0.f;
  int code = 0;
  for (int w = 0; w < 4; ++w) {
    float z = zs[w][b] + bs;
    if (ti.relu && !(z > 0.f)) z = 0.f;
    if (w == 0 || z > best) {
      best = z;
      code = w;
    }
  }
  const int64_t o = ((int64_t)(ti.i[tu] * ti.Wp + ti.j[tu]) * ti.Bp + bb) * ti.Kc + kk;
  y[o] = ok ? tf32_rna(best) : 0.f;
  saved[o] = ok ? (uint8_t)code : 0;
  for (int k = 0; k < ti.npeers; ++k) ti.peer[k][o] = ok ? tf32_rna(best) : 0.f;
  if (ti.npeers) __threadfence_system();
}

// one thread per image (the four window positions), for tails of few pieces per unit
__global__ void fwd_tail_finish_t1(const float* __restrict__ buf, const float* __restrict__ bias, float* __restrict__ y,
                                  uint8_t* __restrict__ saved, const __grid_constant__ FwdTailInfo ti) {
  // blockIdx.z: the M tile within a multicast cluster's unit (ti.cg tiles per piece; 1 otherwise)
  const int tu = blockIdx.y, row = blockIdx.x, b = threadIdx.x, mt = blockIdx.z;
  const int kk = ti.n0[tu] + mt * BM + row;
  if (kk >= ti.Kc) return;
  const int bb = ti.bc0[tu] + b;
  const bool ok = bb < ti.B && kk < ti.Kr;
  const float bs = (bias && kk < ti.Kr) ? bias[kk] : 0.f;
  float zq[4] = {0.f, 0.f, 0.f, 0.f};
  // pieces in K order (~74 per tail unit at the P=4 slice): loads of 8 pieces batched (32 in flight),
  // added in the same order as one piece at a time
  int pc = ti.pbeg[tu];
  const int pe = ti.pbeg[tu + 1];
  const int64_t pstep = (int64_t)ti.cg * BM * BN;
  for (; pc + 8 <= pe; pc += 8) {
    const float* src = buf + (((int64_t)pc * ti.cg + mt) * BM + row) * BN + b;
    float v[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) v[u][q] = src[u * pstep + q * 64];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < 4; ++q) zq[q] += v[u][q];
  }
  for (; pc < pe; ++pc) {
    const float* src = buf + (((int64_t)pc * ti.cg + mt) * BM + row) * BN + b;
#pragma unroll
    for (int q = 0; q < 4; ++q) zq[q] += src[q * 64];
  }
  float best = 0.f;
  int code = 0;
  for (int q = 0; q < 4; ++q) {
    float z = zq[q] + bs;
    if (ti.relu && !(z > 0.f)) z = 0.f;
    if (q == 0 || z > best) {
      best = z;
      code = q;
    }
  }
  const int64_t o = ((int64_t)(ti.i[tu] * ti.Wp + ti.j[tu]) * ti.Bp + bb) * ti.Kc + kk;
  y[o] = ok ? tf32_rna(best) : 0.f;
  saved[o] = ok ? (uint8_t)code : 0;
  for (int k = 0; k < ti.npeers; ++k) ti.peer[k][o] = ok ? tf32_rna(best) : 0.f;
  if (ti.npeers) __threadfence_system();
}

// deterministic split-K reduction: dW[i] = sum_s part[s][i] in split order
// out = sum_s part[s] (split-K partials).  Block (32 float4, 8 split lanes): lane y adds splits
// y*per .. in ascending order, the 8 lane sums combine in fixed order (deterministic).  n % 4 == 0.
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float* __restrict__ part, float* __restrict__ out,
                                                            int64_t n, int S, float* __restrict__ sgd_w, float lr) {
  __shared__ float4 red[8][32];
  const int64_t i4 = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int per = (S + 7) / 8;
  const int s0 = threadIdx.y * per, s1 = min(S, s0 + per);
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i4 * 4 < n) {
    int s = s0;   // loads batched 4 at a time, added in ascending split order
    for (; s + 4 <= s1; s += 4) {
      float4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = reinterpret_cast<const float4*>(part + (int64_t)(s + u) * n)[i4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc.x += x[u].x; acc.y += x[u].y; acc.z += x[u].z; acc.w += x[u].w;
      }
    }
    for (; s < s1; ++s) {
      const float4 x = reinterpret_cast<const float4*>(part + (int64_t)s * n)[i4];
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
  }
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && i4 * 4 < n) {
    float4 t = red[0][threadIdx.x];
#pragma unroll
    for (int k = 1; k < 8; ++k) {
      const float4 u = red[k][threadIdx.x];
      t.x += u.x; t.y += u.y; t.z += u.z; t.w += u.w;
    }
    reinterpret_cast<float4*>(out)[i4] = t;
    if (sgd_w) {   // fused SGD on the final dW
      float4 a = reinterpret_cast<const float4*>(sgd_w)[i4];
      a.x = fmaf(-lr, t.x, a.x); a.y = fmaf(-lr, t.y, a.y); a.z = fmaf(-lr, t.z, a.z); a.w = fmaf(-lr, t.w, a.w);
      reinterpret_cast<float4*>(sgd_w)[i4] = a;
    }
  }
}
// S <= 8 splits: one thread per float4 adds the splits in ascending order with all S loads in flight
// (the 8-lane kernel above leaves 8 - S lanes idle and one load per thread: P=8 wgrad, S = 4,
// 21 us for 47 MB).  Same sums as the lane kernel (each lane held one split) up to the sign of zero.
__global__ void __launch_bounds__(256) splitk_reduce_few(const float* __restrict__ part, float* __restrict__ out,
                                                         int64_t n, int S, float* __restrict__ sgd_w, float lr) {
  const int64_t i4 = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i4 * 4 >= n) return;
  float4 x[8];
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (u < S) x[u] = reinterpret_cast<const float4*>(part + (int64_t)u * n)[i4];
  float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int u = 0; u < 8; ++u)
    if (u < S) {
      t.x += x[u].x; t.y += x[u].y; t.z += x[u].z; t.w += x[u].w;
    }
  reinterpret_cast<float4*>(out)[i4] = t;
  if (sgd_w) {   // fused SGD on the final dW
    float4 a = reinterpret_cast<const float4*>(sgd_w)[i4];
    a.x = fmaf(-lr, t.x, a.x); a.y = fmaf(-lr, t.y, a.y); a.z = fmaf(-lr, t.z, a.z); a.w = fmaf(-lr, t.w, a.w);
    reinterpret_cast<float4*>(sgd_w)[i4] = a;
  }
}
static int launch_splitk_reduce(const float* part, float* out, int64_t n, int S, cudaStream_t s,
                                float* sgd_w = nullptr, float lr = 0.f) {
  if (n % 4) CP_FAIL(CP_ERR_UNSUPPORTED, "split-K reduce: size not a multiple of 4");
  if (S <= 8 && tc_env_int("CP_TC_SPLITK_FEW", 1))
    splitk_reduce_few<<<(unsigned)((n / 4 + 255) / 256), 256, 0, s>>>(part, out, n, S, sgd_w, lr);
  else
    splitk_reduce_kernel<<<(unsigned)((n / 4 + 31) / 32), dim3(32, 8), 0, s>>>(part, out, n, S, sgd_w, lr);
  CP_LAUNCHED();
  return CP_OK;
}

// forward split-K finish: z = sum_s part[s] + bias, then ReLU, 2x2 max-pool (first max wins),
// argmax code and RN-tf32 rounding, exactly as the fused epilogue does.
// One thread per (pooled position, image, 4 slots).
struct PeerSet {
  float* p[CP_MAX_RANKS];
  int n;
};
__global__ void splitk_fwd_finish(const float* __restrict__ part, int S, long long stride,
                                  const float* __restrict__ bias, float* __restrict__ y, uint8_t* __restrict__ saved,
                                  int Wo, int Wp, int Bp, int B, int Kr, int Kc, long long total4, int relu, int pool,
                                  PeerSet peers) {
  const long long e4 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e4 >= total4) return;
  const int kc4 = Kc >> 2;
  const int slot = (int)(e4 % kc4) * 4;
  const long long rest = e4 / kc4;
  const int b = (int)(rest % Bp);
  const int ij = (int)(rest / Bp);
  float bs[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) bs[t] = (bias && slot + t < Kr) ? bias[slot + t] : 0.f;
  const int npos = pool ? 4 : 1;
  float best[4] = {0.f, 0.f, 0.f, 0.f};
  uint32_t code[4] = {0u, 0u, 0u, 0u};
  for (int pos = 0; pos < npos; ++pos) {
    long long zo;
    if (pool) {
      const int j = ij % Wp, i = ij / Wp;
      zo = ((long long)((2 * i + (pos >> 1)) * Wo + 2 * j + (pos & 1)) * Bp + b) * Kc + slot;
    } else {
      zo = rest * Kc + slot;
    }
    float4 acc = *reinterpret_cast<const float4*>(part + zo);
    for (int sp = 1; sp < S; ++sp) {
      const float4 x = *reinterpret_cast<const float4*>(part + sp * stride + zo);
      acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
    }
    float v[4] = {acc.x + bs[0], acc.y + bs[1], acc.z + bs[2], acc.w + bs[3]};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (relu && !(v[t] > 0.f)) v[t] = 0.f;
      if (pos == 0 || v[t] > best[t]) {
        best[t] = v[t];
        code[t] = pos;
      }
    }
  }
  float o[4];
  uint32_t packed = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const bool ok = b < B && slot + t < Kr;
    o[t] = ok ? tf32_rna(best[t]) : 0.f;
    packed |= (ok ? code[t] : 0u) << (8 * t);
  }
  *reinterpret_cast<float4*>(y + rest * Kc + slot) = make_float4(o[0], o[1], o[2], o[3]);
  for (int k = 0; k < peers.n; ++k)
    *reinterpret_cast<float4*>(peers.p[k] + rest * Kc + slot) = make_float4(o[0], o[1], o[2], o[3]);
  if (peers.n) __threadfence_system();
  if (pool) *reinterpret_cast<uint32_t*>(saved + rest * Kc + slot) = packed;
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int get_encoder(EncodeTiledFn* fn) {
  static EncodeTiledFn f = nullptr;
  if (!f) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !ptr)
      CP_FAIL(CP_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    f = (EncodeTiledFn)ptr;
  }
  *fn = f;
  return CP_OK;
}

// fp32 tensor map, zero OOB fill.  dims innermost first; strides in bytes for dims 1..
// K-major operand tiles: SWIZZLE_128B; MN-major tiles: SWIZZLE_128B_ATOM_32B (see tc_common.cuh).
// es: element size (4 = fp32 / tf32 operands, 2 = bf16 operands)
int make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
             const uint32_t* box, bool mn_major = false, int es = 4) {
  EncodeTiledFn enc;
  CP_TRY(get_encoder(&enc));
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], est[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    est[i] = 1;
    if (i + 1 < rank) gs[i] = strides[i];
  }
  CUresult r = enc(m, es == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank,
                   const_cast<void*>(base), gd, gs, bx, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   (mn_major && es == 4) ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) CP_FAIL(CP_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return CP_OK;
}

// 4-D map over an activation block [H][W][Bp][kw] with box {one 128-byte row, 32, bw, bh}
int map_act(CUtensorMap* m, const void* base, int kw, int Bp, int W, int H, int bw, int bh, bool mn_major,
            int es = 4) {
  const uint64_t dims[4] = {(uint64_t)kw, (uint64_t)Bp, (uint64_t)W, (uint64_t)H};
  const uint64_t str[3] = {(uint64_t)kw * es, (uint64_t)kw * Bp * es, (uint64_t)kw * Bp * W * es};
  const uint32_t box[4] = {(uint32_t)(128 / es), 32, (uint32_t)bw, (uint32_t)bh};
  return make_map(m, base, 4, dims, str, box, mn_major, es);
}

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

// 5-D map over an activation block [H][W][Bp][kw] as (32-slot atom lane, b, atom, w, h): one box
// {32, 32, natoms, 1, 1} lands as natoms stacked MN-major 32x32 atoms (the canonical layout).
// Slots past kw inside the last atom read neighbouring data: they only feed output columns/rows
// that are never stored, and every buffer carries read slack (conv_part_query).
// (bf16, es = 2: 64-element groups of 64 K-rows, the SWIZZLE_128B canonical MN-major layout)
int map_act_wide(CUtensorMap* m, const void* base, int kw, int Bp, int W, int H, int natoms, int es = 4) {
  const int E = 128 / es;
  const uint64_t dims[5] = {(uint64_t)E, (uint64_t)Bp, (uint64_t)((kw + E - 1) / E), (uint64_t)W, (uint64_t)H};
  const uint64_t str[4] = {(uint64_t)kw * es, 128, (uint64_t)kw * Bp * es, (uint64_t)kw * Bp * W * es};
  const uint32_t box[5] = {(uint32_t)E, (uint32_t)E, (uint32_t)natoms, 1, 1};
  return make_map(m, base, 5, dims, str, box, true, es);
}

// all input rank blocks have the same (nonzero) width and there are several of them
bool equal_blocks(const Layer& L) {
  if (L.images || L.in.n < 2 || !env_int("CP_TC_UNIFIED", 1)) return false;
  for (int r = 0; r < L.in.n; ++r)
    if (L.in.kw[r] != L.in.kw[0] || L.in.kw[r] == 0) return false;
  return true;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// launch shape of conv_tc_kernel<PASS, CG, DT, MC>: block size (epilogue groups) and, for the multicast
// clusters, how many clusters of `cs` CTAs can be resident at once (cluster placement is per GPC)
template <int PASS, int CG, int DT, int MC>
static void launch_shape(TcParams& p, cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at, int cs) {
  // short K loops (conv1: 3 chunks per tile) are epilogue-bound -> two epilogue warp groups;
  // long ones keep one group (fewer warps polling barriers next to the MMA issuer)
  if (p.epi_groups <= 0) p.epi_groups = p.max_chunks < 64 ? 2 : 1;
  p.epi_groups = std::max(1, std::min(EPI_GROUPS, p.epi_groups));
  cfg.blockDim = dim3(128 + 128 * p.epi_groups);
  cfg.dynamicSmemBytes = Cfg<CG, PASS>::SMEM;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
}

template <int PASS, int CG, int DT = 0, int MC = 0>
static int kernel_attr() {
  static bool attr = false;
  if (!attr) {
    CP_CUDA(cudaFuncSetAttribute(conv_tc_kernel<PASS, CG, DT, MC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)Cfg<CG, PASS>::SMEM));
    attr = true;
  }
  return CP_OK;
}

// clusters of `cs` CTAs of the multicast transposed forward that fit on the GPU at once
int fwd_mc_max_clusters(TcParams& p, int cs) {
  if (kernel_attr<PASS_FWD, 1, 0, 1>() != CP_OK) return 0;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  cfg.gridDim = dim3(cs * (num_sms() / cs));
  launch_shape<PASS_FWD, 1, 0, 1>(p, cfg, at, cs);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, conv_tc_kernel<PASS_FWD, 1, 0, 1>, &cfg) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return std::min(n, num_sms() / cs);
}

template <int PASS, int CG, int DT = 0, int MC = 0>
int launch_cg(const TcParams& p, cudaStream_t s) {
  if (p.units <= 0) return CP_OK;
  CP_TRY((kernel_attr<PASS, CG, DT, MC>()));
  TcParams* pp = const_cast<TcParams*>(&p);
  const int cs = MC ? p.fcl : CG;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  launch_shape<PASS, CG, DT, MC>(*pp, cfg, at, cs);
  const int max_groups = MC ? p.nsched_groups : num_sms() / CG;   // MC: the host planned this many clusters
  const int groups = std::min(p.units, max_groups);
  cfg.gridDim = dim3(groups * cs);
  cfg.stream = s;
  CP_CUDA(cudaLaunchKernelEx(&cfg, conv_tc_kernel<PASS, CG, DT, MC>, p));
  CP_LAUNCHED();
  return CP_OK;
}

// 2-CTA pairs unless disabled (CP_TC_CTA_GROUP=1) or the pass cannot pair its M tiles.
bool use_pairs() {
  const char* e = getenv("CP_TC_CTA_GROUP");   // read per plan (tests switch it between layers)
  return !(e && atoi(e) == 1);
}

void fill_blocks(TcParams& p, const Layer& L) {
  if (L.images) {
    p.nblk = 1;
    p.kw[0] = L.Kcol;
    p.coff[0] = 0;
    p.start[0] = 0;
    p.Cg = L.Kcol;
  } else {
    p.nblk = L.in.n;
    for (int r = 0; r < L.in.n; ++r) {
      p.kw[r] = L.in.kw[r];
      p.coff[r] = L.in.coff[r];
      p.start[r] = L.in.start[r];
    }
    p.Cg = L.in.Cg;
  }
}

void fill_common(TcParams& p, const Layer& L) {
  fill_blocks(p, L);
  p.bke = op_elems(L);
  p.l2hint = env_int("CP_TC_L2HINT", 0);
  p.epi_groups = env_int("CP_TC_EPI_GROUPS", 0);  // 0: decided per launch from the K-loop length
  p.R = L.images ? 1 : L.R;
  p.S = L.images ? 1 : L.S;
  p.Ho = L.Ho;
  p.Wo = L.Wo;
  p.Hin = L.images ? L.Ho : L.H;   // images: im2col rows live on the output grid
  p.Win = L.images ? L.Wo : L.W;
  p.Wp = L.Wp;
  p.Bp = L.Bp;
  p.B = L.B;
  p.Kr = L.Kr;
  p.Kc = L.Kc;
  p.Ktot = L.Ktot;
  p.relu = L.d.relu;
  p.pool = L.d.pool;
  p.images = L.images;
}

// Split-K factor from a small cost model, in units of one K-chunk's MMA time (~512 SM cycles):
// rounds(S) * chunks/S for the GEMM plus the HBM time to write and re-read S fp32 partials.
// Splitting fixes wave quantisation when a rank's slice yields fewer tiles than CTA groups.
int choose_split(int units, int groups, double chunks, double out_bytes, int maxS) {
  const double chunk_us = 512.0 / 1.4e3;  // ~1.4 GHz under load
  const double hbm_bytes_per_us = 6.0e6;
  int best = 1;
  double best_t = 1e300;
  for (int S = 1; S <= maxS; ++S) {
    if (S > 1 && chunks / S < 8) break;
    const double rounds = std::ceil((double)units * S / groups);
    double t = rounds * std::ceil(chunks / S) * chunk_us;
    if (S > 1) t += (2 * S + 1) * out_bytes / hbm_bytes_per_us;  // write + re-read partials, write result
    if (t < best_t * 0.9) {
      best_t = t;
      best = S;
    }
  }
  return best;
}

// N tiles span input blocks when every block width is a multiple of 32 (and there are several)
bool span_ok(const TcParams& p) {
  if (p.images || p.nblk < 2 || !env_int("CP_TC_SPAN", 1)) return false;
  for (int r = 0; r < p.nblk; ++r)
    if (p.kw[r] % p.bke) return false;
  return true;
}

int build_ntiles(TcParams& p) {
  int n = 0;
  if (p.span) {
    for (int n0 = 0; n0 < p.Cg; n0 += BN) {
      if (n >= MAX_NT) return -1;
      p.nt_rb[n] = 0;
      p.nt_n0[n] = n0;
      p.nt_n[n] = std::min(BN, p.Cg - n0);
      ++n;
    }
    return n;
  }
  for (int rb = 0; rb < p.nblk; ++rb)
    for (int n0 = 0; n0 < p.kw[rb]; n0 += BN) {
      if (n >= MAX_NT) return -1;
      p.nt_rb[n] = rb;
      p.nt_n0[n] = n0;
      p.nt_n[n] = std::min(BN, p.kw[rb] - n0);
      ++n;
    }
  return n;
}

}  // namespace

// ---------------------------------------------------------------- work decomposition (host)
// Shared by the workspace query and the launches so both agree on split factors.
struct Plan {
  bool pair;
  int numM, numN, S, per, chunks;  // chunks = K-chunks per unit before splitting (average for dgrad)
  int apb;                         // wgrad span: atoms per B box
};

static Plan fwd_plan(const Layer& L, TcParams& p, int kc = -1) {
  Plan w{};
  if (kc < 0) kc = L.Kc;   // own slots computed on N by this launch (split forward: the 256-multiple part)
  w.pair = use_pairs() && (L.Bp / 32) % 2 == 0;
  const int CG = w.pair ? 2 : 1;
  int cpt = 0;
  for (int r = 0; r < p.nblk; ++r) cpt += (p.kw[r] + op_elems(L) - 1) / op_elems(L);
  p.cpt = cpt;
  w.numM = (L.Ho / 2) * (L.Wo / 2) * (L.Bp / 32) / CG;
  // Balanced N tiles: Kc split into T equal tiles (width a multiple of 16 / 8).  Choose T by
  // rounds of CTA groups x per-chunk time, the latter ~ bytes staged per chunk (A 16 KB + B
  // columns): the kernel is bound by operand delivery, not by MMA issue.
  if (kc == 0) {   // a rank without kernels in this layer: no forward GEMM units
    p.nw = BN;
    w.numN = 0;
  } else {
    const int gran = CG == 2 ? 16 : 8, groups = num_sms() / CG;
    double best = 1e300;
    for (int T = (kc + BN - 1) / BN; T <= (kc + BN - 1) / BN + 4; ++T) {
      const int nw = ((kc + T - 1) / T + gran - 1) / gran * gran;
      if (nw > BN || nw <= 0) continue;
      const int tiles = (kc + nw - 1) / nw;
      const int units = w.numM * tiles;
      double rounds = std::ceil((double)units / groups);
      const int last = units - ((int)rounds - 1) * groups;    // tiles in the last round
      if (rounds > 1 && 2 * last <= groups && env_int("CP_TC_FWD_TAIL", 1))
        rounds = rounds - 1 + (double)last / groups * 1.1;    // tail split (tc_fwd), ~10 % overhead
      const double t = rounds * (16384.0 + 128.0 * nw / CG);
      if (t < best * 0.98) {
        best = t;
        p.nw = nw;
      }
    }
    if (env_int("CP_TC_FWD_NW", 0) > 0) p.nw = env_int("CP_TC_FWD_NW", 0);
    if (p.nw <= 0) p.nw = BN;
    w.numN = (kc + p.nw - 1) / p.nw;
  }
  w.chunks = p.R * p.S * cpt;
  // forward split-K re-reads the whole pre-pool tile from HBM; measured slower at every P, so it
  // is only used when forced (tests exercise it with CP_TC_SPLIT_FWD)
  w.S = env_int("CP_TC_SPLIT_FWD", 1);
  w.S = std::max(1, std::min(w.S, w.chunks));
  return w;
}

// Pixel-mode dgrad pairs two input pixels per CTA pair; both run the K loop over the UNION of their valid
// tap boxes, so pairing columns 2j, 2j+1 wastes MACs at every border column (paper net: 1.08x the exact
// work).  Pixels with the same (row tap range, column tap range) class need no union: pair them within
// their class (row-major), then the <= 1 leftover per class greedily by the fewest added MACs (paper net:
// 1.027x).  Entries sorted by the first pixel (spatial locality of the unit order).
static int build_pixel_pairs(const Layer& L, TcParams& p) {
  const int H = L.H, W = L.W;
  if (H * W / 2 > MAX_PAIRS || H > 255 || W > 255 || (W & 1) || !env_int("CP_TC_DGRAD_PAIRS", 1)) return 0;
  auto rlo = [&](int i) { return std::max(0, i - L.Ho + 1); };
  auto rhi = [&](int i) { return std::min(L.R - 1, i); };
  auto slo = [&](int w) { return std::max(0, w - L.Wo + 1); };
  auto shi = [&](int w) { return std::min(L.S - 1, w); };
  auto box = [&](int i0, int w0, int i1, int w1) {
    const int nr = std::max(rhi(i0), rhi(i1)) - std::min(rlo(i0), rlo(i1)) + 1;
    const int ns = std::max(shi(w0), shi(w1)) - std::min(slo(w0), slo(w1)) + 1;
    return nr * ns;
  };
  std::vector<std::pair<long long, int>> keyed;   // (class key, pixel) in row-major order
  for (int i = 0; i < H; ++i)
    for (int w = 0; w < W; ++w)
      keyed.push_back({((long long)(rlo(i) * 64 + rhi(i)) * 64 + slo(w)) * 64 + shi(w), i * W + w});
  std::stable_sort(keyed.begin(), keyed.end(),
                   [](const std::pair<long long, int>& a, const std::pair<long long, int>& b) { return a.first < b.first; });
  std::vector<std::pair<int, int>> pairs, singles;
  std::vector<int> left;
  for (size_t k = 0; k < keyed.size();) {
    size_t e = k;
    while (e < keyed.size() && keyed[e].first == keyed[k].first) ++e;
    size_t m = k;
    for (; m + 1 < e; m += 2) pairs.push_back({keyed[m].second, keyed[m + 1].second});
    if (m < e) left.push_back(keyed[m].second);
    k = e;
  }
  std::sort(left.begin(), left.end());
  std::vector<char> used(left.size(), 0);
  for (size_t a = 0; a < left.size(); ++a) {
    if (used[a]) continue;
    used[a] = 1;
    int best = -1, bc = 1 << 30;
    const int ia = left[a] / W, wa = left[a] % W;
    for (size_t b = a + 1; b < left.size(); ++b) {
      if (used[b]) continue;
      const int ib = left[b] / W, wb = left[b] % W;
      // the MACs the union adds over the two pixels' own tap boxes
      const int c = 2 * box(ia, wa, ib, wb) - box(ia, wa, ia, wa) - box(ib, wb, ib, wb);
      if (c < bc) {
        bc = c;
        best = (int)b;
      }
    }
    if (best < 0) return 0;   // (odd leftover: cannot happen for an even pixel count)
    used[best] = 1;
    pairs.push_back({left[a], left[best]});
  }
  for (auto& pr : pairs)
    if (pr.first > pr.second) std::swap(pr.first, pr.second);
  std::sort(pairs.begin(), pairs.end());
  if ((int)pairs.size() != H * W / 2) return 0;
  for (size_t k = 0; k < pairs.size(); ++k) {
    const int a = pairs[k].first, b = pairs[k].second;
    p.pair_tab[k] = (uint32_t)(a / W) | ((uint32_t)(a % W) << 8) | ((uint32_t)(b / W) << 16) | ((uint32_t)(b % W) << 24);
  }
  return (int)pairs.size();
}

// valid-tap box of pixel-mode pair entry e (host mirror of dgrad_taps)
static int pair_taps(const Layer& L, uint32_t e) {
  const int i0 = e & 0xff, w0 = (e >> 8) & 0xff, i1 = (e >> 16) & 0xff, w1 = e >> 24;
  const int nr = std::min(L.R - 1, std::max(i0, i1)) - std::max(0, std::min(i0, i1) - L.Ho + 1) + 1;
  const int ns = std::min(L.S - 1, std::max(w0, w1)) - std::max(0, std::min(w0, w1) - L.Wo + 1) + 1;
  return nr * ns;
}

static Plan dgrad_plan(const Layer& L, TcParams& p) {
  Plan w{};
  w.pair = use_pairs() && (L.Bp / 32) % 2 == 0;
  const int CG = w.pair ? 2 : 1;
  p.span = span_ok(p) ? 1 : 0;
  w.numN = build_ntiles(p);
  // pixel mode (pairs, 128-image chunks): valid taps per input row are exact, the pair's column
  // union wastes only at the borders (paper net: 1.08x the exact MACs vs 1.17x for 2x2 windows)
  p.pix = (w.pair && L.Bp % 128 == 0 && env_int("CP_TC_DGRAD_PIX", 1)) ? 1 : 0;
  w.numM = p.pix ? L.H * (L.W / 2) * (L.Bp / 128) : (L.H / 2) * (L.W / 2) * (L.Bp / 32) / CG;
  p.npairs = p.pix ? build_pixel_pairs(L, p) : 0;
  // average valid taps of a tile: (sum over tile rows of valid r) * (same for s) / tiles
  auto avg_valid = [](int Hin, int Ho, int R, int rows) {
    double t = 0;
    const int n = Hin / rows;
    for (int i = 0; i < n; ++i)
      t += std::min(R - 1, rows * i + rows - 1) - std::max(0, rows * i - Ho + 1) + 1;
    return t / n;
  };
  const double kc = (L.Kc + op_elems(L) - 1) / op_elems(L);
  w.chunks = (int)(avg_valid(L.H, L.Ho, L.R, p.pix ? 1 : 2) * avg_valid(L.W, L.Wo, L.S, 2) * kc + 0.5);
  if (p.npairs > 0) {
    double t = 0;
    for (int k = 0; k < p.npairs; ++k) t += pair_taps(L, p.pair_tab[k]);
    w.chunks = (int)(t / p.npairs * kc + 0.5);
  }
  w.S = env_int("CP_TC_SPLIT_DGRAD", 0);
  if (w.S <= 0) w.S = choose_split(w.numM * w.numN, num_sms() / CG, w.chunks, (double)L.in.start[L.in.n] * 4, 16);
  return w;
}

static Plan wgrad_plan(const Layer& L, TcParams& p) {
  Plan w{};
  // CTA pairs unless 128-row tiles cover the own kernels with less padding than 256-row pair tiles
  // (measured: P=4, Kc=376 -> 384 vs 512 rows: single CTAs 10 % faster; equal padding: pairs win)
  w.pair = use_pairs();
  if (w.pair && !getenv("CP_TC_CTA_GROUP") && roundup(L.Kc, BM) < roundup(L.Kc, 2 * BM)) w.pair = false;
  const int CG = w.pair ? 2 : 1;
  p.span = span_ok(p) ? 1 : 0;
  const int per_tap = build_ntiles(p);
  w.numM = ((L.Kc + BM - 1) / BM + CG - 1) / CG;
  w.numN = per_tap < 0 ? -1 : per_tap * p.R * p.S;
  w.chunks = L.Ho * L.Wo * (L.Bp / op_elems(L));   // K-chunks of op_elems images per position
  w.S = env_int("CP_TC_SPLIT_WGRAD", 0);
  if (w.S <= 0) {
    const int units = std::max(1, w.numM * w.numN), G = num_sms() / CG;
    // up to one split per CTA group: a skinny single-tile GEMM (conv1 wgrad) needs every SM streaming K
    w.S = choose_split(units, G, w.chunks, (double)L.Kr * L.Ktot * 4, G);
    if (w.S > 1 && env_int("CP_TC_WGRAD_TAIL", 1)) {
      // S = 1 with the last round split along K (tc_wgrad) vs the whole-tensor split-K
      const int rounds = (units + G - 1) / G, T = units - (rounds - 1) * G;
      const double chunk_us = 512.0 / 1.4e3;
      const double t_tail = (rounds - 1 + ((rounds > 1 && 2 * T <= G) ? 1.0 / std::max(1, G / std::max(T, 1)) : 1.0)) *
                            w.chunks * chunk_us;
      const double t_split = std::ceil((double)units * w.S / G) * std::ceil((double)w.chunks / w.S) * chunk_us +
                             (2 * w.S + 1) * (double)L.Kr * L.Ktot * 4 / 6.0e6;
      if (t_tail < t_split) w.S = 1;
    }
  }
  // Accuracy cap on the reduction length per TMEM accumulator.  The wgrad K (= B*Ho*Wo) grows with
  // batch and image size, and the tensor core's fp32 accumulation error grows linearly with the
  // number of MMAs accumulated (measured, scripts/wgrad_longk.py: scaled net conv2, 2.9 M terms ->
  // 6.0e-3 of max|dW|, 4x shorter -> 1.7e-3, 44x -> 1.6e-4).  At most kAccTerms terms per split
  // keep it near 2.5e-4 (north_star's TF32 bound is 2e-3); splits are summed in fp32 in order.
  {
    const int acc_terms = env_int("CP_TC_ACC_TERMS", 1 << 17);
    const int max_chunks = std::max(1, acc_terms / op_elems(L));
    w.S = std::max(w.S, (w.chunks + max_chunks - 1) / max_chunks);
  }
  w.S = std::max(1, std::min(w.S, w.chunks));
  // Unit order.  N fastest lets a wave share one kernel tile's dY slice, but it reads the
  // activations of all R tap rows at once; once those rows outgrow L2 (scaled net: 5 rows x 110 x
  // 256 images x 512 slots = 288 MB) every tap row is re-read from HBM (ncu: 0.9 TB per launch),
  // so large maps walk the taps slowest instead.
  {
    const double rows_bytes = (double)p.R * L.W * L.Bp * (p.images ? 0 : p.Cg) * op_bytes(L);
    p.wg_taps_slow = env_int("CP_TC_WGRAD_ORDER", rows_bytes > 48e6 ? 1 : 0);
  }
  w.per = (w.chunks + w.S - 1) / w.S;
  w.S = (w.chunks + w.per - 1) / w.per;
  // atoms per B box: every block holds whole boxes
  const int own_atoms = (CG == 2 ? BN / 2 : BN) / op_elems(L);
  w.apb = own_atoms;
  if (p.span)
    for (int r = 0; r < p.nblk; ++r)
      while (w.apb > 1 && (p.kw[r] / op_elems(L)) % w.apb) w.apb >>= 1;
  return w;
}

size_t tc_workspace_bytes(const Layer& L) {
  size_t need = 0;
  {
    TcParams p{};
    fill_common(p, L);
    const Plan w = fwd_plan(L, p);
    if (w.S > 1) need = std::max(need, (size_t)w.S * L.Ho * L.Wo * L.Bp * L.Kc * 4);
    need = std::max(need, (size_t)MAX_PIECES * BM * BN * 4);   // stream-tail partials (pieces x CG x tile)
  }
  if (!L.images && L.Kr > 0) {
    TcParams p{};
    fill_common(p, L);
    const Plan w = dgrad_plan(L, p);
    if (w.S > 1) need = std::max(need, (size_t)w.S * L.in.start[L.in.n] * 4);
  }
  if (L.Kr > 0) {
    TcParams p{};
    fill_common(p, L);
    const Plan w = wgrad_plan(L, p);
    if (w.numN > 0 && w.S > 1) need = std::max(need, (size_t)w.S * L.Kr * L.Ktot * 4);
    // tail-split partials: at most one round of CTA groups x CG tiles of 128 x 256 floats
    if (w.numN > 0 && w.S == 1) need = std::max(need, (size_t)MAX_PIECES * BM * BN * 4);
  }
  return need;
}

// Stream tail: the last partial round of T equal units (C K-chunks each) is shared evenly by all G
// CTA groups - group g takes chunks [g q, (g+1) q) of the T*C tail chunks (q = ceil(T*C / G)), cut at
// unit boundaries into one or two pieces.  Pieces are numbered in chunk order, so a unit's pieces
// are consecutive (pbeg) and its finish kernel sums them in K order (deterministic).  Each group's
// explicit list: its full-round units (round-robin order), then its pieces.  Applied when the last
// round is at most 90 % full (covers a single under-filled round, e.g. 50 units on 74 groups).
static bool plan_stream_tail(TcParams& p, int G, int chunks, int min_chunks, short* pbeg, int* T_out) {
  if (!env_int("CP_TC_STREAM_TAIL", 1)) return false;
  const int units = p.units;
  if (units <= 0 || chunks < min_chunks) return false;
  const int rounds = (units + G - 1) / G, T = units - (rounds - 1) * G, full = (rounds - 1) * G;
  if (T <= 0 || T > MAX_TAIL || 10 * T > 9 * G || G > MAX_GROUPS) return false;
  const long long W = (long long)T * chunks, q = (W + G - 1) / G;
  std::vector<std::vector<int>> lists(G);
  for (int g = 0; g < G; ++g)
    for (int u = g; u < full; u += G) lists[g].push_back(u);
  int np = 0;
  for (int g = 0; g < G; ++g) {
    long long st = (long long)g * q;
    const long long en = std::min(W, (long long)(g + 1) * q);
    while (st < en) {
      const int tu = (int)(st / chunks), lo = (int)(st - (long long)tu * chunks);
      const int hi = (int)std::min<long long>(chunks, lo + (en - st));
      if (np >= MAX_PIECES) return false;
      p.tail_tu[np] = (short)tu;
      p.tail_lo[np] = (short)lo;
      p.tail_hi[np] = (short)hi;
      lists[g].push_back(full + np);
      ++np;
      st += hi - lo;
    }
  }
  if (full + np > MAX_SCHED || chunks > 32767) return false;
  for (int tu = 0, v = 0; tu <= T; ++tu) {
    while (v < np && p.tail_tu[v] < tu) ++v;
    pbeg[tu] = (short)v;
  }
  int off = 0;
  for (int g = 0; g < G; ++g) {
    p.sched_off[g] = (short)off;
    for (int u : lists[g]) p.sched[off++] = (short)u;
  }
  p.sched_off[G] = (short)off;
  p.nsched = 1;
  p.tail_full = full;
  p.tail_np = np;
  p.units = full + np;
  *T_out = T;
  return true;
}

// Create-time check of every condition the three tensor-core passes would reject at launch, so a
// plan that cannot run fails in conv_part_create - never after a rank has entered a cross-rank
// barrier or started pushing its gather block (the peers would wait for it).
int tc_validate(const Layer& L) {
  if ((L.Ho & 1) || (L.Wo & 1))
    CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 forward needs an even conv output grid (2x2 window tiles), got " +
                                    std::to_string(L.Ho) + "x" + std::to_string(L.Wo));
  if (!L.images && L.Kr > 0 && L.Kc > 0) {
    if ((L.H & 1) || (L.W & 1)) CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 dgrad needs an even input grid");
    TcParams p{};
    fill_common(p, L);
    if (dgrad_plan(L, p).numN < 0) CP_FAIL(CP_ERR_UNSUPPORTED, "too many dgrad N tiles");
    if (L.d.math == CP_MATH_BF16)
      for (int r = 0; r < L.in.n; ++r)
        if (L.in.coff[r] % op_elems(L)) CP_FAIL(CP_ERR_UNSUPPORTED, "bf16 dgrad needs input block offsets in multiples of 64");
  }
  if (L.Kr > 0) {
    TcParams p{};
    fill_common(p, L);
    if (wgrad_plan(L, p).numN <= 0) CP_FAIL(CP_ERR_UNSUPPORTED, "too many wgrad N tiles");
  }
  return CP_OK;
}

// exported helpers (shared with kernels_conv1.cu)
int tc_make_map(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                const uint32_t* box, bool mn_major, int es) {
  return make_map(m, base, rank, dims, strides, box, mn_major, es);
}
int tc_num_sms() { return num_sms(); }
// fp32 tensor map without swizzle (dense boxes, e.g. an input patch read by CUDA-core threads)
int tc_make_map_plain(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                      const uint32_t* box) {
  EncodeTiledFn enc;
  CP_TRY(get_encoder(&enc));
  cuuint64_t gd[5], gs[4];
  cuuint32_t bx[5], est[5];
  for (int i = 0; i < rank; ++i) {
    gd[i] = dims[i];
    bx[i] = box[i];
    est[i] = 1;
    if (i + 1 < rank) gs[i] = strides[i];
  }
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rank, const_cast<void*>(base), gd, gs, bx, est,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) CP_FAIL(CP_ERR_CUDA, "cuTensorMapEncodeTiled (plain) failed (" + std::to_string((int)r) + ")");
  return CP_OK;
}
int tc_env_int(const char* name, int dflt) { return env_int(name, dflt); }

int tc_time_mark(Layer& L, int pass, int end, cudaStream_t s) {
  if (!L.timing) return CP_OK;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  CP_CUDA(cudaStreamIsCapturing(s, &st));
  CP_CUDA(cudaEventRecordWithFlags(L.ev_t[pass][end], s,
                                   st == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault));
  return CP_OK;
}

// multicast-cluster transposed forward (CP_TC_FWD_MC=1, with the transposed forward): 2-4 kernel tiles of
// 128 share each activation tile, loaded once per cluster (each CTA a slice, TMA multicast)
static bool fwd_mc_enabled(const Layer& L, int m_off) {
  const int tiles = (L.Kc - m_off + BM - 1) / BM;
  return env_int("CP_TC_FWD_MC", 0) && !L.images && op_bytes(L) == 4 && tiles >= 2 && tiles <= 4 &&
         L.Bp % 64 == 0 && equal_blocks(L);
}

// One forward GEMM launch over own slots [0, kc) on N (kernels-on-N kernels) or, transposed, over
// [m_off, Kc) on M; force_T: -1 = CP_TC_FWD_T, 0/1 = off/on.  `push`: this launch runs the gather push.
static int tc_fwd_part(Layer& L, const float* xin, const float* w, const float* b, float* y_block, uint8_t* saved,
                       void* ws, cudaStream_t s, float* const* peer_blocks, int npeers, const uint32_t* arrive,
                       const GatherPush* gp, int kc, int m_off, int force_T, bool push, bool mark0, bool mark1) {
  if ((L.Ho & 1) || (L.Wo & 1))
    CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 forward needs an even conv output grid (2x2 window tiles)");
  TcParams p{};
  fill_common(p, L);
  const Plan pl = fwd_plan(L, p, kc);
  p.nlim = kc;
  p.m_off = m_off;
  const int es = op_bytes(L), E = 128 / es;
  // halo A boxes (see TcParams::halo): CTA pairs (the 2-stage halo ring fills the 6-stage A region),
  // tf32, S <= 5 (2 x (S+1) x 8 KB <= 96 KB).  Measured 5-8 % SLOWER than one box per tap at P = 1/2/4
  // although it moves 40 % fewer A bytes (profiles/r01_fwd_p4/halo.txt), so it is off unless
  // CP_TC_FWD_HALO=1 (kept: parity-tested in tests/test_gpu_layers.py::test_planner_variants)
  p.diag = env_int("CP_TC_DIAG", 0);
  // transposed forward (TcParams::fwdT): tf32, gathered input, pooled, 64-image chunks.  A TF32 MMA
  // costs the same for any N <= 256, so own-kernel N tiles narrower than 256 waste tensor
  // time; the transposed CTA-local kernel pads the own kernels to 128 instead but moves 1.5x the
  // operand bytes per MAC (L2-bound, ~0.5 us per K-chunk): same-box A/B at P=4 0.206 vs 0.200 ms for
  // the pair kernel, slower at P=1/2/8 as well -> off unless CP_TC_FWD_T=1 (parity-tested; the base
  // for a CTA-pair transposed kernel)
  // default (gather input): transposed when its M tiles use the tensor core clearly better than the pair
  // kernel's N tiles (an N <= 256 MMA costs as much as N = 256): P=4 of the paper net, 376 slots -> 0.98
  // of 3 x 128 rows vs 0.73 of 2 x 256 columns: conv2 forward 0.200 -> 0.186 ms at N=4
  // (profiles/r02_fwdT_auto/); P=1/2 (>= 0.98 either way) and P=8 (0.75 both) keep the pair kernel
  int autoT = 0;
  if (!L.images && kc == L.Kc && m_off == 0 && pl.numN > 0) {
    const double eff_pair = (double)L.Kc / (pl.numN * (double)BN);
    const double eff_t = (double)L.Kc / (((L.Kc + BM - 1) / BM) * (double)BM);
    autoT = eff_t - eff_pair >= 0.15 ? 1 : 0;
  }
  p.fwdT = (es == 4 && L.d.pool && L.Bp % 64 == 0 &&
            (force_T >= 0 ? force_T : env_int(L.images ? "CP_TC_FWD_T_IMAGES" : "CP_TC_FWD_T", autoT))) ? 1 : 0;
#ifdef CP_TC_HALO_HOOK
  const bool halo_hook = true;
#else
  const bool halo_hook = false;
#endif
  p.halo = (halo_hook && pl.pair && es == 4 && !L.images && 2 * (p.S + 1) * 8192 <= Cfg<2, PASS_FWD>::STAGES * A_BYTES &&
            env_int("CP_TC_FWD_HALO", 0)) ? 1 : 0;
  if (p.fwdT && L.images) {
    // im2col rows [Ho][Wo][Bp][Kcol]: box (32 columns, 64 images, 2 w, 2 h)
    p.halo = 0;
    const uint64_t dims[4] = {(uint64_t)L.Kcol, (uint64_t)L.Bp, (uint64_t)L.Wo, (uint64_t)L.Ho};
    const uint64_t str[3] = {(uint64_t)L.Kcol * es, (uint64_t)L.Kcol * L.Bp * es, (uint64_t)L.Kcol * L.Bp * L.Wo * es};
    const uint32_t box[4] = {(uint32_t)E, 64, 2, 2};
    CP_TRY(make_map(&p.maps[0], xin, 4, dims, str, box, false, es));
    p.unified = 0;
  } else if (p.fwdT) {
    p.halo = 0;
    const int n = equal_blocks(L) ? 1 : L.in.n;
    for (int r = 0; r < n; ++r) {
      const int kw = L.in.kw[r];
      if (kw <= 0) continue;
      const uint64_t dims[5] = {(uint64_t)kw, (uint64_t)L.Bp, (uint64_t)L.W, (uint64_t)L.H, (uint64_t)L.in.n};
      const uint64_t str[4] = {(uint64_t)kw * es, (uint64_t)kw * L.Bp * es, (uint64_t)kw * L.Bp * L.W * es,
                               (uint64_t)kw * L.Bp * L.W * L.H * es};
      const uint32_t box[5] = {(uint32_t)E, 64, 2, 2, 1};
      CP_TRY(make_map(&p.maps[r], (const char*)xin + (n == 1 ? 0 : L.in.start[r] * es), n == 1 ? 5 : 4, dims, str,
                      box, false, es));
      if (n == 1 && fwd_mc_enabled(L, m_off)) {
        // multicast-cluster slices of the activation box: one h row (128 rows) / one pixel (64 rows)
        const uint32_t bh[5] = {(uint32_t)E, 64, 2, 1, 1}, bq[5] = {(uint32_t)E, 64, 1, 1, 1};
        CP_TRY(make_map(&p.maps[1], xin, 5, dims, str, bh, false, es));
        CP_TRY(make_map(&p.maps[2], xin, 5, dims, str, bq, false, es));
      }
    }
    p.unified = n == 1 ? 1 : 0;
  } else if (L.images) {
    CP_TRY(map_act(&p.maps[0], xin, L.Kcol, L.Bp, L.Wo, L.Ho, 2, 2, false, es));
  } else if (p.halo) {
    // dims (slot, b, h, w[, block]) - h before w, so a box lands as rows (w, h, b) and the 128 rows of
    // column tap s are the contiguous rows [64 s, 64 s + 128)
    const int n = equal_blocks(L) ? 1 : L.in.n;
    for (int r = 0; r < n; ++r) {
      const int kw = L.in.kw[r];
      if (kw <= 0) continue;
      const uint64_t dims[5] = {(uint64_t)kw, (uint64_t)L.Bp, (uint64_t)L.H, (uint64_t)L.W, (uint64_t)L.in.n};
      const uint64_t str[4] = {(uint64_t)kw * es, (uint64_t)kw * L.Bp * L.W * es, (uint64_t)kw * L.Bp * es,
                               (uint64_t)kw * L.Bp * L.W * L.H * es};
      const uint32_t box[5] = {(uint32_t)E, 32, 2, (uint32_t)(p.S + 1), 1};
      CP_TRY(make_map(&p.maps[r], (const char*)xin + (n == 1 ? 0 : L.in.start[r] * es), n == 1 ? 5 : 4, dims, str,
                      box, false, es));
    }
    p.unified = n == 1 ? 1 : 0;
  } else if (equal_blocks(L)) {
    // one 5-D map over all rank blocks: (slot, b, w, h, block)
    const int kw = L.in.kw[0];
    const uint64_t dims[5] = {(uint64_t)kw, (uint64_t)L.Bp, (uint64_t)L.W, (uint64_t)L.H, (uint64_t)L.in.n};
    const uint64_t str[4] = {(uint64_t)kw * es, (uint64_t)kw * L.Bp * es, (uint64_t)kw * L.Bp * L.W * es,
                             (uint64_t)kw * L.Bp * L.W * L.H * es};
    const uint32_t box[5] = {(uint32_t)E, 32, 2, 2, 1};
    CP_TRY(make_map(&p.maps[0], xin, 5, dims, str, box, false, es));
    p.unified = 1;
  } else {
    for (int r = 0; r < L.in.n; ++r)
      if (L.in.kw[r] > 0)
        CP_TRY(map_act(&p.maps[r], (const char*)xin + L.in.start[r] * es, L.in.kw[r], L.Bp, L.W, L.H, 2, 2, false, es));
  }
  p.bn_box = pl.pair ? p.nw / 2 : std::min(p.nw, L.Kc);

  {
    const uint64_t dims[2] = {(uint64_t)L.Ktot, (uint64_t)std::max(L.Kr, 1)};
    const uint64_t str[1] = {(uint64_t)L.Ktot * es};
    const uint32_t box[2] = {(uint32_t)E, (uint32_t)(p.fwdT ? BM : p.bn_box)};
    CP_TRY(make_map(&p.maps[CP_MAX_RANKS], w, 2, dims, str, box, false, es));
  }
  p.numM = pl.numM;
  p.numN = pl.numN;
  p.split = pl.S;
  p.units = p.numM * p.numN * pl.S;
  p.max_chunks = (pl.chunks + pl.S - 1) / pl.S;
  if (p.fwdT) {
    p.numM = (L.Kc - p.m_off + BM - 1) / BM;
    p.numN = L.Hp * L.Wp * (L.Bp / 64);
    p.split = 1;
    p.units = p.numM * p.numN;
    p.max_chunks = pl.chunks;
    if (p.unified && fwd_mc_enabled(L, p.m_off)) {
      // multicast clusters: one cluster per position tile, its CTAs = the kernel tiles
      const int g = fwd_mc_max_clusters(p, p.numM);
      if (g > 0) {
        p.fcl = p.numM;
        p.units = p.numN;
        p.nsched_groups = g;
      }
    }
  }
  p.bias = L.d.bias ? b : nullptr;
  p.saved = saved;
  p.npeers = npeers;
  for (int k = 0; k < npeers; ++k) p.peer_out[k] = peer_blocks[k];
  p.arrive = L.images ? nullptr : arrive;
  p.self_blk = L.d.rank;
  p.arrive_target = 1;
  if (gp && !L.images) {
    p.push_src = gp->src;
    p.npush = push ? gp->n : 0;
    for (int k = 0; k < gp->n; ++k) {
      p.push_dst[k] = gp->dst[k];
      p.push_cnt[k] = gp->cnt[k];
    }
    p.push_n4 = gp->n4;
    p.push_chunks = gp->chunks;
    p.push_claim = gp->claim;
    p.push_mc = gp->mc;
    p.push_warps = env_int("CP_TC_PUSH_WARPS", 1);
    p.push_stamp = push ? gp->stamp : nullptr;
    p.arrive_target = (uint32_t)gp->chunks;
  }
  float* part = (float*)((char*)ws + L.off_split);
  p.part_stride = (long long)L.Ho * L.Wo * L.Bp * L.Kc;
  p.out = (pl.S > 1 && !p.fwdT) ? part : y_block;
  // Stream tail of the last partial round (plan_stream_tail); the pooled epilogue of those tiles
  // runs in fwd_tail_finish after the deterministic sum of their pieces.
  FwdTailInfo ti{};
  {
    const int CG = (pl.pair && !p.fwdT) ? 2 : 1, G = p.fcl ? p.nsched_groups : num_sms() / CG;
    int T = 0;
    if ((pl.S == 1 || p.fwdT) && env_int("CP_TC_FWD_TAIL", 1) && plan_stream_tail(p, G, p.R * p.S * p.cpt, 16, ti.pbeg, &T)) {
      p.tail_buf = part;
      ti.n = T; ti.cg = p.fcl ? p.fcl : CG; ti.Wo = L.Wo; ti.Wp = L.Wp; ti.Bp = L.Bp; ti.B = L.B; ti.halo = p.halo;
      ti.Kr = L.Kr; ti.Kc = L.Kc; ti.relu = L.d.relu; ti.pool = L.d.pool;
      ti.npeers = npeers;
      for (int k = 0; k < npeers; ++k) ti.peer[k] = peer_blocks[k];
      const int nbcg = L.Bp / 32 / CG, W2 = L.Wo / 2;
      for (int k = 0; k < T && p.fwdT; ++k) {          // host mirror of decode_unit<FWD> (transposed)
        const int u = p.tail_full + k;
        const int mt = p.fcl ? 0 : u % p.numM, rest = p.fcl ? u : u / p.numM, nb = L.Bp / 64;
        const int ij = rest / nb;
        ti.bc0[k] = (rest % nb) * 64;
        ti.j[k] = ij % L.Wp;
        ti.i[k] = ij / L.Wp;
        ti.n0[k] = p.m_off + mt * BM;
        ti.ncol[k] = BM;
      }
      for (int k = 0; k < T && !p.fwdT; ++k) {         // host mirror of decode_unit<FWD>
        const int u = p.tail_full + k;
        const int mg = u % p.numM, nt = (u / p.numM) % p.numN;
        const int ij = mg / nbcg;
        ti.bc0[k] = (mg % nbcg) * CG * 32;
        ti.j[k] = ij % W2;
        ti.i[k] = ij / W2;
        ti.n0[k] = nt * p.nw;
        ti.ncol[k] = std::min(p.nw, kc - ti.n0[k]);
      }
    }
  }
  if (env_int("CP_TC_PLAN_LOG", 0))
    fprintf(stderr, "[tc_fwd] Kc=%d kc=%d m_off=%d fwdT=%d fcl=%d units=%d numM=%d numN=%d groups=%d tail_np=%d nw=%d\n",
            L.Kc, kc, m_off, p.fwdT, p.fcl, p.units, p.numM, p.numN, p.fcl ? p.nsched_groups : -1, p.tail_np, p.nw);
  if (mark0) CP_TRY(tc_time_mark(L, PASS_FWD, 0, s));
  if (es == 2) CP_TRY((pl.pair ? launch_cg<PASS_FWD, 2, 1>(p, s) : launch_cg<PASS_FWD, 1, 1>(p, s)));
  else if (p.fcl) CP_TRY((launch_cg<PASS_FWD, 1, 0, 1>(p, s)));
  else CP_TRY(((pl.pair && !p.fwdT) ? launch_cg<PASS_FWD, 2>(p, s) : launch_cg<PASS_FWD, 1>(p, s)));
  if (mark1) CP_TRY(tc_time_mark(L, PASS_FWD, 1, s));
  if (p.tail_np > 0 && p.fwdT) {
    int max_np = 0;
    for (int k = 0; k < ti.n; ++k) max_np = std::max(max_np, ti.pbeg[k + 1] - ti.pbeg[k]);
    // many pieces per tail unit (P=4 slice: 2 units x ~74 pieces): one thread per pre-pool value,
    // 22.0 -> 8.0 us (ncu, profiles/r02_tail_finish/); few: one thread per image
    if (max_np >= 16)
      fwd_tail_finish_t<<<dim3(BM, ti.n, p.fcl ? p.fcl : 1), 256, 0, s>>>(part, L.d.bias ? b : nullptr, y_block, saved, ti);
    else
      fwd_tail_finish_t1<<<dim3(BM, ti.n, p.fcl ? p.fcl : 1), 64, 0, s>>>(part, L.d.bias ? b : nullptr, y_block, saved, ti);
    CP_LAUNCHED();
  } else if (p.tail_np > 0) {
    int max_np = 0;
    for (int k = 0; k < ti.n; ++k) max_np = std::max(max_np, ti.pbeg[k + 1] - ti.pbeg[k]);
    if (max_np >= 16)
      fwd_tail_finish_q<<<dim3(32, ti.cg, ti.n), dim3(BN, 4), 0, s>>>(part, L.d.bias ? b : nullptr, y_block, saved, ti);
    else
      fwd_tail_finish<<<dim3(32, ti.cg, ti.n), BN, 0, s>>>(part, L.d.bias ? b : nullptr, y_block, saved, ti);
    CP_LAUNCHED();
  }
  if (pl.S > 1 && !p.fwdT) {
    PeerSet ps{};
    ps.n = npeers;
    for (int k = 0; k < npeers; ++k) ps.p[k] = peer_blocks[k];
    const long long total4 = (long long)L.Hp * L.Wp * L.Bp * (L.Kc / 4);
    splitk_fwd_finish<<<(unsigned)((total4 + 255) / 256), 256, 0, s>>>(
        part, pl.S, p.part_stride, L.d.bias ? b : nullptr, y_block, saved, L.Wo, L.Wp, L.Bp, L.B, L.Kr, L.Kc, total4,
        L.d.relu, L.d.pool, ps);
    CP_LAUNCHED();
  }
  return CP_OK;
}

// Split forward (CP_TC_FWD_SPLIT=1; off by default - measured no faster at P=4 on one GPU, 0.194 ->
// 0.192 ms, and 70 us slower inside the fused 4-GPU step, profiles/r02_fwd_split.txt): a TF32 MMA costs the same for any N <= 256,
// so an own-slot count just above a multiple of 256 (P=4 of the paper net: 375 = 256 + 119) wastes a
// whole N tile.  Then the CTA-pair kernel computes the 256-multiple part with full 256-wide N tiles
// and the transposed CTA-local kernel the remainder on M (119 of 128 TMEM lanes used, N = 256
// pixels x images): 375 slots cost 256 + 128 MMA columns instead of 2 x 256.  Both launches write
// disjoint slots of the same output block; the first runs the gather push, both wait for arrivals.
int tc_fwd(Layer& L, const float* xin, const float* w, const float* b, float* y_block, uint8_t* saved, void* ws,
           cudaStream_t s, float* const* peer_blocks, int npeers, const uint32_t* arrive, const GatherPush* gp) {
  if (L.Kc == 0) return CP_OK;
  const int rem = L.Kc % BN;
  const bool split = op_bytes(L) == 4 && !L.images && L.d.pool && L.Bp % 64 == 0 && use_pairs() &&
                     (L.Bp / 32) % 2 == 0 && L.Kc > BN && rem >= 64 && rem <= BM &&
                     env_int("CP_TC_FWD_SPLIT", 0) && !env_int("CP_TC_FWD_T", 0) && env_int("CP_TC_SPLIT_FWD", 1) == 1 &&
                     env_int("CP_TC_FWD_NW", 0) == 0 && !env_int("CP_TC_FWD_HALO", 0);
  if (!split)
    return tc_fwd_part(L, xin, w, b, y_block, saved, ws, s, peer_blocks, npeers, arrive, gp, L.Kc, 0, -1, true, true,
                       true);
  const int k1 = L.Kc - rem;
  CP_TRY(tc_fwd_part(L, xin, w, b, y_block, saved, ws, s, peer_blocks, npeers, arrive, gp, k1, 0, 0, true, true, false));
  return tc_fwd_part(L, xin, w, b, y_block, saved, ws, s, peer_blocks, npeers, arrive, gp, L.Kc, k1, 1, false, false,
                     true);
}

int tc_dgrad(Layer& L, const float* dY, const float* w, float* dx, void* ws, cudaStream_t s, float* const* dst_blocks) {
  if (L.images) CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 dgrad onto images");
  if ((L.H & 1) || (L.W & 1)) CP_FAIL(CP_ERR_UNSUPPORTED, "tcgen05 dgrad needs an even input grid");
  if (L.Kc == 0 || L.Kr == 0) {
    CP_CUDA(cudaMemsetAsync(dx, 0, (size_t)L.in.start[L.in.n] * 4, s));
    return CP_OK;
  }
  TcParams p{};
  fill_common(p, L);
  Plan pl = dgrad_plan(L, p);
  if (pl.numN < 0) CP_FAIL(CP_ERR_UNSUPPORTED, "too many dgrad N tiles");
  if (dst_blocks) {   // fused reduce-scatter: every partial tile is final (no split-K partials)
    pl.S = 1;
    p.fused_dx = 1;
    for (int r = 0; r < L.in.n; ++r) p.dst[r] = dst_blocks[r];
  }
  const int es = op_bytes(L), E = 128 / es;
  if (p.pix) {
    // A = dY rows of one pixel: box {one 128-byte row of kernels, 128 images, 1, 1}
    const uint64_t dims[4] = {(uint64_t)L.Kc, (uint64_t)L.Bp, (uint64_t)L.Wo, (uint64_t)L.Ho};
    const uint64_t str[3] = {(uint64_t)L.Kc * es, (uint64_t)L.Kc * L.Bp * es, (uint64_t)L.Kc * L.Bp * L.Wo * es};
    const uint32_t box[4] = {(uint32_t)E, 128, 1, 1};
    CP_TRY(make_map(&p.maps[0], dY, 4, dims, str, box, false, es));
  } else {
    CP_TRY(map_act(&p.maps[0], dY, L.Kc, L.Bp, L.Wo, L.Ho, 2, 2, false, es));
  }
  p.wide = 1;
  for (int r = 0; r < L.in.n; ++r)
    if (L.in.coff[r] % E) p.wide = 0;
  if (es == 2 && !p.wide) CP_FAIL(CP_ERR_UNSUPPORTED, "bf16 dgrad needs input block offsets in multiples of 64");
  if (p.wide) {
    // W [Kr][RS][Cg] viewed as (c' lane, k, c' group, tap): one box {E, E, groups, 1}
    const uint64_t dims[4] = {(uint64_t)E, (uint64_t)L.Kr, (uint64_t)((L.in.Cg + E - 1) / E), (uint64_t)(L.R * L.S)};
    const uint64_t str[3] = {(uint64_t)L.Ktot * es, 128, (uint64_t)L.in.Cg * es};
    const uint32_t box[4] = {(uint32_t)E, (uint32_t)E, (uint32_t)((pl.pair ? BN / 2 : BN) / E), 1};
    CP_TRY(make_map(&p.maps[CP_MAX_RANKS], w, 4, dims, str, box, true, es));
  } else {
    // W [Kr][RS][Cg] viewed as (c', k, tap): MN-major boxes {32 c', 32 k, 1}
    const uint64_t dims[3] = {(uint64_t)L.in.Cg, (uint64_t)L.Kr, (uint64_t)(L.R * L.S)};
    const uint64_t str[2] = {(uint64_t)L.Ktot * 4, (uint64_t)L.in.Cg * 4};
    const uint32_t box[3] = {32, 32, 1};
    CP_TRY(make_map(&p.maps[CP_MAX_RANKS], w, 3, dims, str, box, true));
  }
  p.numM = pl.numM;
  p.numN = pl.numN;
  p.split = pl.S;
  p.units = p.numM * p.numN * pl.S;
  p.max_chunks = (pl.chunks + pl.S - 1) / pl.S;
  {
    // LPT order of the 2x2 windows by valid-tap count (descending, stable)
    const int H2 = L.H / 2, W2 = L.W / 2;
    // off by default: measured slower at P=1/2/4 (heavy windows dispatched together lose the
    // spatial L2 locality of the natural order)
    if (!p.pix && H2 * W2 <= MAX_WIN && env_int("CP_TC_DGRAD_LPT", 0)) {
      std::vector<std::pair<int, int>> wk;
      for (int i = 0; i < H2; ++i)
        for (int j = 0; j < W2; ++j) {
          const int nr = std::min(L.R - 1, 2 * i + 1) - std::max(0, 2 * i - L.Ho + 1) + 1;
          const int ns = std::min(L.S - 1, 2 * j + 1) - std::max(0, 2 * j - L.Wo + 1) + 1;
          wk.push_back({-nr * ns, i * W2 + j});
        }
      std::stable_sort(wk.begin(), wk.end(), [](const std::pair<int, int>& a, const std::pair<int, int>& b) {
        return a.first < b.first;
      });
      p.nwin_order = H2 * W2;
      for (int k = 0; k < H2 * W2; ++k) p.win_order[k] = (short)wk[k].second;
    }
  }
  float* part = (float*)((char*)ws + L.off_split);
  p.part_stride = pl.S > 1 ? (long long)L.in.start[L.in.n] : 0;
  p.out = pl.S > 1 ? part : dx;
  {
    // Static LPT schedule: tiles carry 4..25 valid taps, so round-robin dispatch leaves SMs idle.
    // Assign each unit (heaviest first) to the least-loaded CTA group; a group then walks its units
    // in natural order (keeps the spatial L2 locality of neighbouring windows).
    const int CG = pl.pair ? 2 : 1, G = std::min(p.units, num_sms() / CG);
    if (p.nwin_order == 0 && p.units <= MAX_SCHED && G <= MAX_GROUPS && env_int("CP_TC_DGRAD_SCHED", 1)) {
      const int nbcg = p.pix ? L.Bp / 128 : L.Bp / 32 / CG, W2 = L.W / 2, kc = (L.Kc + op_elems(L) - 1) / op_elems(L);
      std::vector<std::pair<long long, int>> wk(p.units);
      for (int u = 0; u < p.units; ++u) {
        const int mg = u % p.numM;
        const int ij = mg / nbcg, i = ij / W2, j = ij % W2;
        int taps;
        if (p.pix && p.npairs > 0) {
          taps = pair_taps(L, p.pair_tab[ij]);
        } else {
          const int h0 = p.pix ? i : 2 * i, h1 = p.pix ? i : 2 * i + 1;
          const int nr = std::min(L.R - 1, h1) - std::max(0, h0 - L.Ho + 1) + 1;
          const int ns = std::min(L.S - 1, 2 * j + 1) - std::max(0, 2 * j - L.Wo + 1) + 1;
          taps = nr * ns;
        }
        const long long work = ((long long)taps * kc + pl.S - 1) / pl.S;
        wk[u] = {-work, u};
      }
      std::stable_sort(wk.begin(), wk.end());
      std::vector<long long> load(G, 0);
      std::vector<std::vector<int>> lists(G);
      for (const auto& e : wk) {
        int g = 0;
        for (int q = 1; q < G; ++q)
          if (load[q] < load[g]) g = q;
        load[g] += -e.first;
        lists[g].push_back(e.second);
      }
      int off = 0;
      for (int g = 0; g < G; ++g) {
        std::sort(lists[g].begin(), lists[g].end());
        p.sched_off[g] = (short)off;
        for (int u : lists[g]) p.sched[off++] = (short)u;
      }
      p.sched_off[G] = (short)off;
      p.nsched = off;
    }
  }
  CP_TRY(tc_time_mark(L, PASS_DGRAD, 0, s));
  if (es == 2) CP_TRY((pl.pair ? launch_cg<PASS_DGRAD, 2, 1>(p, s) : launch_cg<PASS_DGRAD, 1, 1>(p, s)));
  else CP_TRY((pl.pair ? launch_cg<PASS_DGRAD, 2>(p, s) : launch_cg<PASS_DGRAD, 1>(p, s)));
  CP_TRY(tc_time_mark(L, PASS_DGRAD, 1, s));
  if (pl.S > 1) {
    const int64_t n = L.in.start[L.in.n];
    CP_TRY(launch_splitk_reduce(part, dx, n, pl.S, s));
  }
  return CP_OK;
}

int tc_wgrad(Layer& L, const float* dY, const float* xin, float* dw, void* ws, cudaStream_t s, float* sgd_w,
             float sgd_lr) {
  if (L.Kr == 0) return CP_OK;
  TcParams p{};
  fill_common(p, L);
  const Plan w = wgrad_plan(L, p);
  if (w.numN <= 0) CP_FAIL(CP_ERR_UNSUPPORTED, "too many wgrad N tiles");
  p.wide = 1;
  p.apb = w.apb;
  const int es = op_bytes(L), E = 128 / es;
  const int nat = p.span ? w.apb : (w.pair ? BN / 2 : BN) / E;
  if (L.images) {
    CP_TRY(map_act_wide(&p.maps[0], xin, L.Kcol, L.Bp, L.Wo, L.Ho, nat, es));
  } else if (p.span && equal_blocks(L)) {
    // one 5-D map over all rank blocks: (slot lane, b, slot group, h*W + w, block)
    const int kw = L.in.kw[0];
    const uint64_t dims[5] = {(uint64_t)E, (uint64_t)L.Bp, (uint64_t)(kw / E), (uint64_t)L.H * L.W, (uint64_t)L.in.n};
    const uint64_t str[4] = {(uint64_t)kw * es, 128, (uint64_t)kw * L.Bp * es, (uint64_t)kw * L.Bp * L.W * L.H * es};
    const uint32_t box[5] = {(uint32_t)E, (uint32_t)E, (uint32_t)nat, 1, 1};
    CP_TRY(make_map(&p.maps[0], xin, 5, dims, str, box, true, es));
    p.unified = 1;
  } else {
    for (int r = 0; r < L.in.n; ++r)
      if (L.in.kw[r] > 0)
        CP_TRY(map_act_wide(&p.maps[r], (const char*)xin + L.in.start[r] * es, L.in.kw[r], L.Bp, L.W, L.H, nat, es));
  }
  CP_TRY(map_act_wide(&p.maps[CP_MAX_RANKS], dY, L.Kc, L.Bp, L.Wo, L.Ho, BM / E, es));
  p.numM = w.numM;
  p.numN = w.numN;
  p.chunks_total = w.chunks;
  p.split = w.S;
  p.chunks_per_split = w.per;
  p.max_chunks = w.per;
  p.units = p.numM * p.numN * w.S;
  float* part = w.S > 1 ? (float*)((char*)ws + L.off_split) : dw;
  p.out = part;
  p.sgd_w = w.S == 1 ? sgd_w : nullptr;   // split-K: the update runs in the split reduce
  p.sgd_lr = sgd_lr;
  // Tail split: when the last round of equal tiles is at most half full, split only those tiles
  // along K over all CTA groups (their partials are tiny; everything else is written directly).
  TailInfo ti{};
  const int CG = w.pair ? 2 : 1, G = num_sms() / CG;
  int T = 0;
  if (w.S == 1 && env_int("CP_TC_WGRAD_TAIL", 1) && plan_stream_tail(p, G, w.chunks, 8, ti.pbeg, &T)) {
    p.tail_buf = (float*)((char*)ws + L.off_split);
    ti.n = T;
    ti.cg = CG;
    ti.Kr = L.Kr;
    ti.Ktot = L.Ktot;
    ti.sgd_w = sgd_w;
    ti.sgd_lr = sgd_lr;
    const int per_tap = p.numN / (p.R * p.S);
    for (int k = 0; k < T; ++k) {                      // host mirror of decode_unit<WGRAD>
      const int u = p.tail_full + k;
      int tap, e, mg;
      if (p.wg_taps_slow) {
        e = u % per_tap;
        mg = (u / per_tap) % p.numM;
        tap = (u / per_tap / p.numM) % (p.R * p.S);
      } else {
        const int nt = u % p.numN;
        mg = (u / p.numN) % p.numM;
        tap = nt / per_tap;
        e = nt % per_tap;
      }
      ti.kk0[k] = mg * CG * BM;
      ti.col0[k] = tap * p.Cg + (p.span ? 0 : p.coff[p.nt_rb[e]]) + p.nt_n0[e];
      ti.ncol[k] = p.nt_n[e];
    }
  }
  CP_TRY(tc_time_mark(L, PASS_WGRAD, 0, s));
  if (es == 2) CP_TRY((w.pair ? launch_cg<PASS_WGRAD, 2, 1>(p, s) : launch_cg<PASS_WGRAD, 1, 1>(p, s)));
  else CP_TRY((w.pair ? launch_cg<PASS_WGRAD, 2>(p, s) : launch_cg<PASS_WGRAD, 1>(p, s)));
  CP_TRY(tc_time_mark(L, PASS_WGRAD, 1, s));
  if (p.tail_np > 0) {
    wgrad_tail_reduce<<<dim3(BM, CG, ti.n), BN, 0, s>>>(p.tail_buf, dw, ti);
    CP_LAUNCHED();
  }
  if (w.S > 1) {
    const int64_t n = (int64_t)L.Kr * L.Ktot;
    CP_TRY(launch_splitk_reduce(part, dw, n, w.S, s, sgd_w, sgd_lr));
  }
  return CP_OK;
}

void tc_release(Layer&) {}

}  // namespace cp
