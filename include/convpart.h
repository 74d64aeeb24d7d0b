/*
 * convpart.h — C ABI of the B200-native kernel-partitioned convolution library
 * (hot path of arXiv 1712.02546, "kernel-partitioned conv-layer training").
 *
 * The method (§4): every device receives the SAME layer
 * input and a DIFFERENT contiguous subset of the layer's kernels (Alg. 1 L9,
 * P:L169 "All slaves receive same inputs but different kernels"); each device
 * convolves its subset; the per-device feature maps are
 * gathered and "reshaped and rearranged" into channel order.  Kernel
 * counts per device follow Eq. 1 from a probe convolution timed on
 * every device.  Backward convolutions are distributed with the same
 * split ("forward and backward propagation included"; north_star): each
 * rank runs dgrad and wgrad for its slice, partial dX are summed across ranks,
 * weight gradients stay local.
 *
 * B200 realisation: one process per GPU.  With symmetric (peer-mapped) buffers the
 * channel gather overlaps the consumer GEMM (copy engines distribute each rank's block
 * over NVLink while the next layer's forward computes its own block first; or the GEMM
 * kernel pushes it itself) and the dX reduce-scatter overlaps the next GEMM (owners
 * fetch the partials by copy engine, or the dgrad epilogue stores them into the owners'
 * receive slots; summed in rank order); otherwise NCCL AllGather / ReduceScatter /
 * AllReduce.
 * Conv passes are implicit GEMMs on tcgen05/TMEM (kind::tf32, FP32 accumulation)
 * with TMA-staged tiles and a fused bias+ReLU+2x2 max-pool epilogue, or FP32
 * SIMT kernels in the reference math mode.
 *
 * CONVENTIONS (all entry points)
 *  - Return int status: CP_OK (0) or a negative CP_ERR_*; never abort; the
 *    message is available from cp_last_error() (thread-local), naming both
 *    shapes on a shape error ("dimension error naming both shapes").
 *  - Device pointers are caller-owned (PyTorch tensors), 16-byte aligned
 *    (TMA requirement), sized from conv_part_query().  The library owns only
 *    host state: the handle, cached TMA descriptors, a copy of the partition,
 *    and a borrowed cp_comm.
 *  - Calls enqueue work on the given CUDA streams and return; no device sync.
 *    Asynchronous kernel faults surface as CP_ERR_CUDA at a later call.
 *  - One host thread per handle.
 *
 * DATA LAYOUTS (fp32 unless stated)
 *  - Images (first-layer input): NCHW [B][C][H][W], replicated on every rank.
 *  - Gather layout of a layer's output ("y_gathered"): rank blocks in rank
 *    order; block r is [Hp][Wp][Bp][Kc_r] (channel slot innermost, batch next),
 *    Kc_r = k_width[r] = roundup(k_count[r], 8), Bp = roundup(B, 32).
 *    Logical channel c of rank r = owner(c) is slot c - k_begin[r].  Element
 *    (b,c,h,w) sits at  block_start[r] + ((h*Wp + w)*Bp + b)*Kc_r + slot,
 *    block_start[r] = sum_{r'<r} Hp*Wp*Bp*Kc_{r'}.  Padding slots and padded
 *    images (b >= B) are exactly 0.  (§8(c) item 9 of SURVEY.)
 *  - Conv weights on the GPU (the rank's own kernels only):
 *      image input : [K_r][Kcol], Kcol = roundup(R*S*C, 8), column (r*S+s)*C+c
 *      gather input: [K_r][R][S][Cg], Cg = sum_r k_width_in[r], column = the
 *                    input's gather slot order (zero at padded slots)
 *    cp_pack_conv_weights() builds these from KCRS.
 *  - saved: uint8 argmax code 2*di+dj per pooled output of the rank's block,
 *    [Hp][Wp][Bp][Kc_r]  (ties -> first in row-major order).
 */
#ifndef CONVPART_H_
#define CONVPART_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CP_MAX_RANKS 16

enum {
  CP_OK = 0,
  CP_ERR_ARG = -1,         /* null pointer / out-of-range argument            */
  CP_ERR_SHAPE = -2,       /* dimension error (message names both shapes)     */
  CP_ERR_CONFIG = -3,      /* invalid configuration (e.g. n_ranks < 1)        */
  CP_ERR_DATA = -4,        /* invalid data (e.g. nonpositive probe time)       */
  CP_ERR_CUDA = -5,        /* CUDA runtime / driver failure                   */
  CP_ERR_NCCL = -6,        /* NCCL failure (incl. async errors)               */
  CP_ERR_STATE = -7,       /* call order / handle state violated              */
  CP_ERR_UNSUPPORTED = -8  /* valid request this build does not implement     */
};

typedef enum {
  CP_MATH_TF32 = 0,      /* tcgen05 kind::tf32 implicit GEMMs, fp32 accumulate */
  CP_MATH_FP32_SIMT = 1, /* FP32 CUDA-core reference kernels                  */
  CP_MATH_BF16 = 2       /* NEXT row f4, report-only: the GEMM operands (weights, layer input, dY)
                            are rounded to bf16 copies inside the library, tcgen05 kind::f16,
                            fp32 accumulate and fp32 outputs.  Needs partition widths in multiples
                            of 64 (cp_partition_plan align 64) and a batch padded to a multiple of
                            64; error ~1e-2 of max|ref|, outside the 2e-3 TF32 bar */
} cp_math;

typedef enum {
  CP_DX_ALLREDUCE = 0,       /* full summed dX on every rank                       */
  CP_DX_REDUCE_SCATTER = 1,  /* rank r receives the summed dX of its own block only */
  CP_DX_LOCAL = 2,           /* no collective: dx holds this rank's partial sum     */
  CP_DX_ASYNC = 16,          /* OR-flag: do not make `stream` wait for the dX collective;
                                call conv_part_wait() before reading dx (lets independent
                                work such as wgrad overlap the reduction, §8(e))        */
  CP_DX_ORDERED = 64         /* OR-flag (fused reduce-scatter only).  PRECONDITION: between two
                                consecutive backward_data calls of this layer, every rank
                                passes a cross-rank synchronising operation that is ordered
                                after its previous dX sum on every rank (PartitionedNet: the
                                next forward's gather barrier or logits AllReduce, which all
                                ranks enter only after joining the dX stream).  Then no rank can
                                overwrite partials a peer is still summing, and the
                                overwrite-guard barrier is skipped.  Without that guarantee the
                                flag races: omit it.                                      */
} cp_dx_mode;

typedef enum {
  CP_INPUT_IMAGES = 0,  /* dense NCHW input replicated on all ranks (first layer)  */
  CP_INPUT_GATHER = 1   /* the previous layer's gather-layout output               */
} cp_input_kind;

/* Partition map: contiguous kernel ranges in rank order. */
typedef struct {
  int32_t n_ranks;
  int32_t num_k;
  int32_t k_begin[CP_MAX_RANKS];
  int32_t k_count[CP_MAX_RANKS];
  int32_t k_width[CP_MAX_RANKS]; /* Kc_r = roundup(k_count, align) */
} cp_partition;

/* cp_partition_plan — Eq. 1 weights w_i = (max t / t_i) / sum_j (max t / t_j),
 * then exact-integer largest-remainder apportionment (reading R11):
 * q_i = llround(2^20 * max(t)/t_i); floor_i = numK*q_i div sum q; leftover units to the
 * largest remainders numK*q_i mod sum q, ties to the lower rank; ranges = prefix sums;
 * k_width = roundup(count, align).  Pure host function, bit-exact, identical on all ranks.
 * Errors: t_i <= 0 or non-finite -> CP_ERR_DATA; n_ranks outside [1, CP_MAX_RANKS] or
 * align < 1 -> CP_ERR_CONFIG; num_k < 0 or null pointer -> CP_ERR_ARG. */
int cp_partition_plan(const double* times_s, int32_t n_ranks, int32_t num_k, int32_t align,
                      cp_partition* out);

/* Eq. 1 weights only (for reporting). */
int cp_eq1_weights(const double* times_s, int32_t n_ranks, double* weights_out);

/* ---------------------------------------------------------------- communicator
 * Library-owned ncclComm_t over NVLink/NVSwitch.  The 128-byte unique id is made
 * on rank 0 by cp_comm_unique_id and travels to the other ranks through
 * torch.distributed (the plumbing); every rank then calls cp_comm_create on its
 * own current CUDA device.  A NULL cp_comm means "no collectives" (single GPU, or
 * P ranks simulated on one GPU in tests). */
typedef struct cp_comm_s* cp_comm;
int cp_comm_unique_id(uint8_t id_out[128]);
int cp_comm_create(const uint8_t id[128], int32_t rank, int32_t world, cp_comm* out);
int cp_comm_destroy(cp_comm comm);

/* cp_comm_create_loopback — `world` simulated ranks in ONE process on the current GPU (tests of
 * the fused peer-memory paths on a single B200): out[r] is rank r's handle.  Symmetric buffers
 * are plain allocations (the k-th cp_symmetric_alloc of every handle forms one buffer); the
 * cross-rank barriers are no-ops; the comm-stream tail of a fused reduce-scatter (wait for the
 * peers' slots, rank-order sum) is held back until every rank has issued its backward_data
 * call for that layer and then enqueued behind all of their dgrads, so no kernel waits on a
 * later launch.  The caller issues the P ranks' calls of a layer back to back in rank order; the
 * fused gather's arrival counters of ranks that have not run yet must be satisfied by the caller
 * (cp_symmetric_peer gives the addresses).  NCCL collectives, cp_allreduce_sum and
 * cp_symmetric_wait return CP_ERR_UNSUPPORTED on a loopback handle.  Destroy every handle. */
int cp_comm_create_loopback(int32_t world, cp_comm* out);

/* Symmetric buffers for the fused collectives (the gather is Alg. 1's
 * "concatenate the output of all nodes").  cp_symmetric_alloc allocates `bytes` of
 * zeroed device memory on every rank (collective: all ranks, same size, same order), exchanges CUDA
 * IPC handles over the communicator and maps every peer's copy, plus a 256-byte flag line behind
 * the data: u32 word q = arrival counter of sender q; word 32 = the gather's chunk-claim counter.
 * Semantics when a layer's y_gathered is symmetric (conv_part_forward):
 *   producer: the GEMM writes this rank's block into its LOCAL copy only; a device-side
 *     cross-rank barrier (no rank may overwrite a copy a peer still reads) runs on comm_stream
 *     (on stream when comm_stream == stream) and the consumer's distribution waits for it;
 *   consumer: conv_part_forward whose x is a symmetric gathered buffer distributes this rank's
 *     input block into every peer's copy and consumes its own block first, each peer block once
 *     that peer's counter is raised (gather overlapped with the GEMM; no AllGather kernel), then
 *     resets its flag line.  Default (tensor-core consumer, comm_stream != stream): copy-engine
 *     copies on comm_stream, peers in the order they consume the block, then the counter set to
 *     CP_GATHER_CHUNKS.  CP_GATHER_MODE=push (environment): the GEMM kernel pushes the block
 *     itself (CP_GATHER_CHUNKS chunks claimed by any running CTA, one release-add on the peer's
 *     counter per chunk).  A rank without kernels in the consuming layer uses copy-engine copies
 *     on stream.  Any other reader of a symmetric gathered output calls cp_symmetric_wait (waits
 *     for all peers' flags on `stream`, then resets them) first.
 * cp_symmetric_peer returns rank `rank`'s copy of the buffer and of its flag line as addressable
 * from this process (tests; diagnostics).  cp_symmetric_free (collective) or cp_comm_destroy
 * releases the buffers.  Errors: CP_ERR_ARG for a pointer that is not a symmetric buffer of `comm`;
 * CUDA/NCCL errors as CP_ERR_CUDA/CP_ERR_NCCL. */
#define CP_GATHER_CHUNKS 256
int cp_symmetric_alloc(cp_comm comm, size_t bytes, void** local_out);
int cp_symmetric_free(cp_comm comm, void* local);
int cp_symmetric_wait(cp_comm comm, void* local, void* stream);
int cp_symmetric_peer(cp_comm comm, void* local, int32_t rank, void** data, uint32_t** flags);

/* ---------------------------------------------------------------- conv layer */
typedef struct {
  int32_t batch;               /* B (real images)                                 */
  int32_t in_c, in_h, in_w;    /* logical input NCHW (in_c = total input channels) */
  int32_t num_k, k_h, k_w;     /* kernels K, R, S (valid conv, stride 1)          */
  int32_t bias, relu, pool;    /* epilogue flags; pool = 2x2 stride 2 max         */
  int32_t math;                /* cp_math                                         */
  int32_t input_kind;          /* cp_input_kind                                   */
  cp_partition out_part;       /* this layer's kernel split (num_k == num_k)      */
  cp_partition in_part;        /* split of the input channels (CP_INPUT_GATHER)   */
  int32_t rank, world;         /* this rank; world == out_part.n_ranks            */
  int32_t local_output;        /* 0: all-gather the output along channels (default);
                                  1: keep only this rank's block (y_gathered holds the own block at
                                  its offset) - for a layer whose consumer is itself partitioned,
                                  e.g. the FC head with rank-local columns      */
} cp_conv_desc;

/* w, x, y and dx include 256 bytes of read slack past the tensor (TMA atoms of 32 columns may
 * read, but never use, a few elements beyond the last row). */
typedef struct {
  size_t w;         /* bytes of this rank's GPU-layout weights                    */
  size_t b;         /* bytes of this rank's bias                                  */
  size_t x;         /* bytes of the layer input (images NCHW or full gather)      */
  size_t y;         /* bytes of the full gather-layout output (all rank blocks)   */
  size_t y_block;   /* bytes of this rank's block of y                            */
  size_t y_offset;  /* byte offset of this rank's block inside y                  */
  size_t saved;     /* bytes of this rank's argmax codes (0 without pooling)      */
  size_t dx;        /* bytes of the input gradient (same shape as x)              */
  size_t workspace; /* bytes of per-layer scratch; must persist fwd -> bwd        */
  size_t dx_peer;   /* bytes of dx for the fused reduce-scatter: the gather layout
                       followed by n_ranks receive slots of the largest input block
                       (allocate with cp_symmetric_alloc; 0 for image input)       */
} cp_sizes;

typedef struct cp_layer_s* cp_layer;

/* conv_part_create — validate the descriptor and build the handle.  With a comm,
 * checks that every rank holds the same partition (an AllReduce of a hash):
 * mismatch -> CP_ERR_CONFIG.  comm may be NULL (no collectives). */
int conv_part_create(const cp_conv_desc* desc, cp_comm comm, cp_layer* out);
int conv_part_query(cp_layer layer, cp_sizes* out);
int conv_part_destroy(cp_layer layer);

/* conv_part_probe — the paper's throughput probe (§4.1.1): run this
 * rank's forward convolution on random data of the layer's shapes (the whole
 * layer's kernels on this device), warmups untimed, then the median of reps
 * (S:L178-186).  Blocking; host-timed with CUDA events.  scratch must hold
 * conv_part_probe_bytes(). */
int conv_part_probe_bytes(const cp_conv_desc* desc, size_t* bytes);
int conv_part_probe(const cp_conv_desc* desc, int32_t warmups, int32_t reps, void* scratch,
                    size_t scratch_bytes, void* stream, double* median_s);

/* conv_part_forward — Z = conv(x, own kernels) + b; ReLU; 2x2 max-pool; writes this
 * rank's block of y_gathered (and argmax codes into saved), then (with a comm) the
 * channel AllGather over NVLink fills the other ranks' blocks (Alg. 1 L19-22,
 * P:L178-182).  The collective runs on comm_stream, ordered after the compute on
 * stream via events; stream then waits for it.  comm_stream may equal stream. */
int conv_part_forward(cp_layer layer, const float* x, const float* w, const float* b,
                      float* y_gathered, uint8_t* saved, void* workspace,
                      void* stream, void* comm_stream);

/* conv_part_backward_data — unpool/ReLU' of this rank's block of dy_gathered (using
 * saved and y_gathered), then dX_partial = dgrad(dY, own kernels) for ALL input
 * channels, then the cross-rank sum selected by dx_mode.  dx has the shape of x.
 * For CP_DX_REDUCE_SCATTER only this rank's input block of dx is valid.  With the
 * CP_DX_ASYNC flag and comm_stream != stream, `stream` is not made to wait for the
 * collective: call conv_part_wait(layer, stream) before consuming dx.
 * Fused reduce-scatter (SURVEY §8(f) f1, TF32 path): when dx is a symmetric buffer of
 * at least dx_peer bytes (cp_symmetric_alloc) and dx_mode is CP_DX_REDUCE_SCATTER, no
 * NCCL collective runs.  Default ("ce"): the dgrad writes every input block's partial into
 * this rank's own copy of dx, sets this rank's ready flag at every peer, and on comm_stream
 * each owner waits for all flags, copies its block's partials from the peers' copies into
 * its receive slots behind the gather layout with the copy engines (NVLink, no SM) and
 * sums the n_ranks partials in ascending rank order into its block of dx.
 * CP_RS_MODE=pull (environment): the owner reads the partials with SM loads instead;
 * CP_RS_MODE=push: the dgrad epilogue stores each partial straight into its owner's receive
 * slot and the owner sums the slots - all three give the same bits.  Unless CP_DX_ORDERED is
 * given, a cross-rank barrier first guards the slots / partials against overwrite while an
 * owner still reads them. */
int conv_part_backward_data(cp_layer layer, const float* dy_gathered, const uint8_t* saved,
                            const float* y_gathered, const float* w, float* dx, int32_t dx_mode,
                            void* workspace, void* stream, void* comm_stream);

/* conv_part_backward_filter — dW_r = wgrad(dY, x) and db_r = sum dY for this rank's
 * kernels only (no communication).  dw has the GPU weight layout, db [K_r]. */
int conv_part_backward_filter(cp_layer layer, const float* dy_gathered, const uint8_t* saved,
                              const float* y_gathered, const float* x, float* dw, float* db,
                              void* workspace, void* stream);

/* conv_part_backward_filter_sgd — conv_part_backward_filter followed by this rank's SGD step
 * on its own slice: w -= lr*dw, b -= lr*db (b and db both given or both NULL; w, b
 * must not alias dw, db).  dw and db are still written.  TF32 / BF16 and the image-layer kernels
 * apply the update where the final dW / db are produced (the wgrad epilogue, its split-K or
 * stream-tail reduce, the bias reduce, the conv1 reduce) instead of a separate pass over W and dW
 * (the same fused multiply-add as cp_sgd: bitwise identical to backward_filter + sgd_step); the
 * FP32 SIMT mode runs the separate update. */
int conv_part_backward_filter_sgd(cp_layer layer, const float* dy_gathered, const uint8_t* saved,
                                  const float* y_gathered, const float* x, float* dw, float* db, float* w,
                                  float* b, float lr, void* workspace, void* stream);

/* conv_part_timing — enable (1) / disable (0) per-pass timing of this layer's tensor-core GEMM
 * launches: CUDA events recorded on the launching stream immediately before and after the GEMM
 * kernel (external records, so they also time inside a captured CUDA graph).  With a fused gather
 * input, also the gather window: events on comm_stream around the copy-engine distribution, or (in-
 * kernel push) %globaltimer stamps in the workspace from the first push chunk claimed to the last
 * chunk's arrival released; with the copy-engine reduce-scatter, events on comm_stream around the
 * partials' fetch (after all peers' ready flags).
 * conv_part_kernel_time — duration in ms of the last recorded GEMM of `pass` (0 forward,
 * 1 backward-data, 2 backward-filter), 3: the last gather window (push stamps: a blocking read),
 * 4: the last reduce-scatter fetch window.  The caller synchronizes first.  CP_ERR_STATE if timing
 * is off or (pass 3 / 4) no such window was recorded; a CUDA error if that pass never ran since
 * enabling.  (bench.py's roofline and NVLink measurements) */
int conv_part_timing(cp_layer layer, int32_t enable);
int conv_part_kernel_time(cp_layer layer, int32_t pass, float* ms);

/* conv_part_wait — make `stream` wait for the layer's last issued collective. */
int conv_part_wait(cp_layer layer, void* stream);

/* conv_part_sgd_step — w -= lr*dw, b -= lr*db on this rank's slice. */
int conv_part_sgd_step(cp_layer layer, float* w, float* b, const float* dw, const float* db,
                       float lr, void* stream);

/* Number of kernels this library launched since load (evidence counter). */
int64_t cp_launch_count(void);
/* Thread-local message of the last error. */
const char* cp_last_error(void);

/* ---------------------------------------------------------------- boundary helpers
 * All enqueue on `stream`.  Geometry is given by the partition and (H, W, B). */

/* NCHW [B][C][H][W] -> full gather layout (zero padding) and back (bit-exact). */
int cp_pack_nchw(const float* x_nchw, int32_t B, int32_t C, int32_t H, int32_t W,
                 const cp_partition* part, float* out_gathered, void* stream);
int cp_unpack_nchw(const float* gathered, int32_t B, int32_t C, int32_t H, int32_t W,
                   const cp_partition* part, float* out_nchw, void* stream);
/* argmax codes of rank `rank`'s block -> NCHW uint8 of that rank's channels [B][K_r][Hp][Wp]. */
int cp_unpack_saved(const uint8_t* saved, int32_t B, int32_t Hp, int32_t Wp,
                    const cp_partition* part, int32_t rank, uint8_t* out, void* stream);

/* KCRS conv weights (all K kernels, fp32) -> this rank's GPU layout; and back
 * (rows of this rank only, KCRS). */
int cp_pack_conv_weights(const cp_conv_desc* desc, const float* w_kcrs, float* out, void* stream);
int cp_unpack_conv_weights(const cp_conv_desc* desc, const float* w_gpu, float* out_kcrs_rows,
                           void* stream);

/* ---------------------------------------------------------------- replicated head
 * FC over a gather-layout input (features in gather order; the FC weight is
 * stored in that order, zero at padded slots: cp_pack_fc_weights), softmax
 * cross-entropy (mean over B, max-subtracted), FC backward.  Every
 * rank runs the head on identical data; reductions are fixed-order, so results
 * are bitwise identical on all ranks.  ws_bytes from cp_head_workspace_bytes. */
int cp_head_workspace_bytes(int32_t B, int32_t Hp, int32_t Wp, const cp_partition* part,
                            int32_t O, size_t* bytes);
int cp_pack_fc_weights(const float* wfc_nchw, int32_t O, int32_t Hp, int32_t Wp,
                       const cp_partition* part, float* out, void* stream);
int cp_unpack_fc_weights(const float* wfc_g, int32_t O, int32_t Hp, int32_t Wp,
                         const cp_partition* part, float* out_nchw, void* stream);
int cp_fc_forward(const float* x_gathered, int32_t B, int32_t Hp, int32_t Wp,
                  const cp_partition* part, const float* wfc_g, const float* bfc, int32_t O,
                  float* logits, void* ws, void* stream);
int cp_softmax_xent(const float* logits, const int32_t* labels, int32_t B, int32_t O,
                    float* loss, float* dlogits, void* stream);
int cp_fc_backward(const float* dlogits, const float* x_gathered, int32_t B, int32_t Hp,
                   int32_t Wp, const cp_partition* part, const float* wfc_g, int32_t O,
                   float* dx_gathered, float* dwfc_g, float* dbfc, void* ws, void* stream);
/* Cross-channel LRN followed by 2x2/2 max-pool (NEXT row f2: the paper's "Normalization layer",
 * Conv -> Norm -> Pool; form and default constants S:L89-97; ReLU before the
 * normalisation, reading R23):  s_c = bias + alpha * sum_{|j-c|<=depth/2} a_j^2,  n_c = a_c s_c^-beta.
 * cp_lrn_pool_forward: a_gathered is the conv layer's gathered pre-pool output (a layer created with
 * pool = 0: every rank holds all channels, H x W grid, B images); writes the pooled map for ALL
 * channels (gather layout over part, H/2 x W/2) and the uint8 argmax codes (2*di + dj, first max),
 * RN-tf32 rounded when round_tf32.  Every rank computes it (no second collective).
 * cp_lrn_pool_backward: dy_gathered is the gradient of the pooled map for ALL channels (the next
 * layer's dX summed with CP_DX_ALLREDUCE, or the replicated head's); writes this rank's block of
 * the gradient w.r.t. a (pre-pool gather layout), which is then the dy_gathered of
 * conv_part_backward_data / _filter of the pool = 0 conv layer (its ReLU' uses a).
 * Errors: depth even or < 1, bias <= 0 -> CP_ERR_CONFIG; odd H or W -> CP_ERR_SHAPE; more than 2048
 * channels -> CP_ERR_UNSUPPORTED. */
int cp_lrn_pool_forward(const float* a_gathered, int32_t B, int32_t H, int32_t W, const cp_partition* part,
                        int32_t depth, float alpha, float beta, float bias, int32_t round_tf32,
                        float* y_gathered, uint8_t* codes_gathered, void* stream);
int cp_lrn_pool_backward(const float* dy_gathered, const float* a_gathered, const uint8_t* codes_gathered,
                         int32_t B, int32_t H, int32_t W, const cp_partition* part, int32_t rank,
                         int32_t depth, float alpha, float beta, float bias, float* da_gathered, void* stream);

/* p -= lr*g over n floats. */
int cp_sgd(float* p, const float* g, int64_t n, float lr, void* stream);
/* The same SGD update for `count` tensors in one launch per 16 tensors: params[i]
 * -= lr*grads[i] over sizes[i] floats (host arrays of device pointers; a tensor may be empty). */
int cp_sgd_multi(float* const* params, const float* const* grads, const int64_t* sizes, int32_t count,
                 float lr, void* stream);

/* In-place sum over all ranks of n floats on `stream`; the result is bitwise identical on every
 * rank.  Once the communicator holds symmetric memory and n <= 65536, a one-CTA peer-memory kernel:
 * each rank writes its vector into slot [rank] of every peer's scratch (double-buffered by epoch
 * parity) and sums the slots in ascending rank order once every peer's data is there.  For
 * n <= 32768 (default) each value travels with the epoch in one 64-bit word and the reader polls
 * the data itself; otherwise (or CP_AR_LL=0) the rank raises an epoch flag after a system fence and
 * the readers wait for all flags.  Larger n: NCCL AllReduce.  Used by the partitioned head to sum
 * per-rank partial logits.  comm == NULL or a single rank: no-op. */
int cp_allreduce_sum(cp_comm comm, float* buf, int64_t n, void* stream);

/* cp_allreduce_sum of the [B][O] partial logits followed by cp_softmax_xent on the sum, in ONE
 * launch when the one-shot peer-memory path applies (the same block sums the slots in rank order,
 * then computes loss and dlogits: dlogits bitwise the same as the two calls, the loss too for
 * B <= 256 - beyond that its fixed-order tree runs over twice the threads).  logits is replaced by
 * the summed logits.  Otherwise (comm NULL / one rank: softmax only; NCCL path) the two calls.
 * B in [1,8192], O in [1,16]; CP_ERR_ARG otherwise; CP_ERR_UNSUPPORTED on a loopback handle. */
int cp_allreduce_softmax_xent(cp_comm comm, float* logits, const int32_t* labels, int32_t B, int32_t O,
                              float* loss, float* dlogits, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CONVPART_H_ */
