/*
 * smile.h -- C ABI of libsmile: the B200 (sm_100a) hot path of SMILE, the bi-level
 * Switch-style MoE layer of arXiv 2212.05191 ("SMILE: Scaling Mixture-of-Experts with
 * Efficient Bi-level Routing"), next to the flat single-All2All Switch baseline.
 *
 * Citations "P:Lx" are lines of the paper's text; "R<k>" are the readings of
 * ambiguous passages listed in DESIGN.md.
 *
 * ---------------------------------------------------------------------------------
 * Model.  G = n*m ranks form n groups ("nodes") of m ranks ("GPUs"); rank r = s*m + l
 * is local index l of group s (R10).  Each rank holds e experts and T
 * tokens.  Level 1 routes a token to a group (K1 = n destinations, the inter router W_p),
 * level 2 to an expert of that group (K2 = m*e destinations, the intra router W_q); the
 * token of source (s, l) travels first to the intermediate (i, l) and then to the expert
 * rank (i, j/e) (Eq. 3).  FLAT mode is the one-hop Switch layer with
 * K1 = G*e experts and no level 2.
 *
 * Ranks per process.  A process drives V = G / nprocs consecutive ranks on ONE device
 * ("resident ranks", r = proc*V + v).  nprocs == 1 emulates the whole G-rank layer on
 * one GPU (the exchanges become device copies); nprocs == G is one rank per GPU with the
 * exchanges as NCCL all-to-alls on the split inter / intra communicators.
 * Every per-rank array below has a leading dimension V.
 *
 * ---------------------------------------------------------------------------------
 * Conventions (all calls).
 *  - Ownership: the caller owns every buffer and the stream; the library owns only the
 *    context (its NCCL communicators, a sticky device error flag and small scratch sized
 *    at smile_create).  Nothing is allocated after smile_create.
 *  - Pointers: every buffer argument is a DEVICE pointer on the context's device unless
 *    its name starts with host_.  Rows are row-major, 16-byte aligned (d*b % 16 == 0).
 *  - Asynchrony: calls enqueue work on `stream` and return; there is no host sync on the
 *    hot path (smile_get_error and smile_forward_host excepted), so a sequence of calls
 *    is CUDA-graph capturable.
 *  - Errors: synchronous validation returns a status and launches nothing
 *    (SMILE_EINVAL bad value, SMILE_ESHAPE layout mismatch, SMILE_ENOTSUP unsupported
 *    combination).  Errors found on the device (non-finite logits, R27; an index out of
 *    range) set a sticky flag that smile_get_error returns.
 *  - T == 0 is a legal no-op for gate, dispatch, exchange, ffn and combine;
 *    smile_aux_loss returns SMILE_EINVAL for T == 0 (the loss divides by T).
 *  - Order: the calls of one layer must follow the sequence of smile_forward below; any
 *    other order is undefined behaviour.  A context is not thread-safe.
 * ---------------------------------------------------------------------------------
 */
#ifndef SMILE_H
#define SMILE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMILE_VERSION 100

typedef enum {
    SMILE_OK = 0,
    SMILE_EINVAL = 1,      /* invalid argument value (n, m, e < 1, cf <= 0, T < 0, ...) */
    SMILE_ESHAPE = 2,      /* layout / size mismatch */
    SMILE_ENONFINITE = 3,  /* device: a router logit was NaN or Inf (R27) */
    SMILE_ECUDA = 4,       /* a CUDA runtime call failed */
    SMILE_ENCCL = 5,       /* an NCCL call failed */
    SMILE_ENOTSUP = 6,     /* valid but unsupported combination */
    SMILE_EINDEX = 7,      /* device: routing index out of range (corrupt route input) */
    SMILE_ETIMEOUT = 8     /* device: a peer process did not reach a peer-exchange barrier within
                              the barrier timeout (smile_register_workspace); the step's data are
                              not valid */
} smile_status;

typedef enum { SMILE_FP32 = 0, SMILE_BF16 = 1 } smile_dtype;
typedef enum { SMILE_BILEVEL = 0, SMILE_FLAT = 1 } smile_mode;

/* Expert-FFN implementation.  AUTO picks tcgen05 for bf16 and SIMT FFMA for fp32. */
typedef enum { SMILE_FFN_AUTO = 0, SMILE_FFN_SIMT = 1, SMILE_FFN_TCGEN05 = 2 } smile_ffn_impl;

typedef struct {
    int32_t n, m, e;        /* groups, ranks per group, experts per rank */
    int32_t mode;           /* smile_mode */
    int32_t dtype;          /* smile_dtype of x, the exchanged rows and the expert weights */
    int32_t d, d_ff;        /* hidden and FFN sizes */
    int64_t T;              /* tokens per rank (static) */
    double cf;              /* capacity factor */
    int32_t nprocs;         /* processes of the job, each driving G/nprocs ranks */
    int32_t proc;           /* this process, 0 <= proc < nprocs */
    int32_t device;         /* CUDA device ordinal of this process */
    int32_t ffn_impl;       /* smile_ffn_impl */
    int32_t topk;           /* experts per token (Eq. 2): 0 or 1 = the
                               top-1 layers of the paper (Eq. 3); 2..4 = the FLAT top-k layer
                               (GShard-style, R29-R32; forward and backward).  BILEVEL requires
                               top-1 */
} smile_shape;

/* Sizes derived from a shape (R5, R7, R20, R31):
 *   K1 = BILEVEL ? n : G*e;   K2 = BILEVEL ? m*e : 1;
 *   C1 = K1 > 1 ? ceil(cf*k*T/K1) : k*T (k = topk, 1 for the paper's layers);
 *   C2 = BILEVEL ? (K2 > 1 ? ceil(cf*T/K2) : n*C1) : 0.
 * S = segments per local expert at the FFN (BILEVEL: m source ranks; FLAT: G);
 * Cseg = rows per segment (BILEVEL: C2; FLAT: C1). */
typedef struct {
    int32_t G, V, rank0;    /* ranks, ranks resident in this process, first resident rank */
    int32_t K1, K2, KW;     /* destinations per level; KW = logits row width (K1 + K2, FLAT: K1) */
    int64_t C1, C2;
    int32_t S;
    int64_t Cseg;
    size_t ws_bytes;        /* size of the workspace smile_forward needs (smile_forward_ws) */
    size_t router_partial_bytes;   /* scratch of smile_router_bwd */
} smile_sizes;

typedef struct smile_ctx_s *smile_ctx;

/* ---------------- context ---------------- */

int          smile_version(void);
/* Host-side count of kernels libsmile has launched in this process (every launch site
 * counts itself; NCCL's and CUDA's own kernels are not included).  Monotonic; a caller
 * takes the difference around a region to know how many library kernels it enqueued. */
int64_t      smile_launch_count(void);
/* sizeof of smile_shape, smile_sizes, smile_route, smile_stats, smile_layer_io,
 * smile_ws_view, smile_grad_io, smile_xop (in that order) into out[0..n), so a binding
 * can verify its mirrors of the structs. */
smile_status smile_struct_sizes(int64_t *out, int32_t n);
const char  *smile_strerror(smile_status s);
/* Pure host: the capacity of one (sending rank, destination) pair, ceil(cf * T / dests)
 * (the capacity factor of P:L207 applied to the equal-split buffers of P:L67-71; R5),
 * with a single-destination level having no capacity (dests == 1 -> T, R20) and T == 0
 * -> 0.  Computed in double then rounded up (exact for the paper's cf in {1, 1.25, 2}).
 * Returns -1 for T < 0, dests < 1 or cf <= 0 (or cf NaN). */
int64_t      smile_capacity(int64_t T, int64_t dests, double cf);
/* Pure host function, usable without a GPU: fills *out from *shape or returns
 * SMILE_EINVAL (n, m, e, d, d_ff < 1, T < 0, cf <= 0, nprocs not dividing G, ...). */
smile_status smile_plan(const smile_shape *shape, smile_sizes *out);
/* Pure host: the group of global rank r at `level` (1 = inter {(i, l)}, 2 = intra
 * {(s, g)}, 0 = world), written in position order to members[] (room for G ints); the
 * member count is returned through *count.  P:L148, R10. */
smile_status smile_group(const smile_shape *shape, int32_t level, int32_t r, int32_t *members,
                         int32_t *count);
/* Pure host: the point-to-point schedule smile_all2all posts for the pairs of `level`
 * whose two ranks live in different processes, for process shape->proc.  ops[] receives
 * every send (ordered by source rank, then destination rank) followed by every receive
 * (same order), so two processes list their common transfers in the same order, which is
 * how NCCL matches them inside one ncclGroupStart/End.  `chunk` indexes the caller's
 * [V, P] chunk array (send side: the chunk sent; receive side: where it lands).  Pairs
 * inside this process are device copies and are not listed.  count = #ops written
 * (SMILE_ESHAPE when more than `cap`). */
typedef struct {
    int32_t kind;        /* 0 = send, 1 = receive */
    int32_t peer_proc;   /* the other process */
    int32_t src, dst;    /* global ranks of the transfer */
    int32_t chunk;       /* v * P + p in this process's send / receive buffer */
} smile_xop;
smile_status smile_exchange_plan(const smile_shape *shape, int32_t level, smile_xop *ops, int32_t cap,
                                 int32_t *count);
/* 128-byte NCCL unique id, to be broadcast by the caller (e.g. torch.distributed) from
 * process 0 before smile_create when nprocs > 1. */
smile_status smile_get_unique_id(uint8_t out[128]);
/* Creates the context on shape->device.  nprocs > 1: initialises an NCCL world
 * communicator from `nccl_id` (collective: every process must call it) and, when
 * V == 1, splits it into the inter (color l, key s) and intra (color s, key l)
 * communicators.  nprocs == 1: nccl_id may be NULL. */
smile_status smile_create(smile_ctx *ctx, const smile_shape *shape, const uint8_t *nccl_id);
smile_status smile_destroy(smile_ctx ctx);
smile_status smile_query(smile_ctx ctx, smile_sizes *out);
/* Synchronises `stream`, then returns and clears the sticky device error flag. */
smile_status smile_get_error(smile_ctx ctx, void *stream);

/* ---------------- fused permute -> peer-store exchange ----------
 * SMILE_XCHG_COPY (default): the permutes fill send buffers and each level's All2All is an
 * explicit exchange (device copies between ranks of one process, NCCL between processes).
 * SMILE_XCHG_PEER: smile_forward (inference; train == 0) skips the send buffers -- the
 * level-1 / level-2 permutes store every kept row straight into the receive buffer of its
 * destination rank (on this GPU, or another GPU's workspace mapped with CUDA IPC and
 * written over NVLink), the return path loads rows straight from the peer's buffers, and
 * the four All2Alls become four process-level flag barriers over NVLink.  Only valid rows
 * move (no capacity padding on the wire).  One node only (CUDA IPC).
 * BILEVEL with the tcgen05 FFN: the level-2 permute also records, at the expert, the row
 * of the intermediate's ret1 each input row came from, and GEMM 2 of smile_expert_ffn /
 * smile_expert_ffn_train stores the output rows of intermediates in the same process
 * there instead of into Y -- the intra reverse exchange (a10) and the level-2 un-permute
 * (a11) of those rows happen inside the FFN's epilogue; the following smile_combine(2)
 * fetches only the rows of experts in other processes (with one process it returns at
 * once).  Level-2-dropped rows get their zero return row from the level-2 permute.
 * (Scattered 64-byte NVLink stores from the epilogue measured slower than the combine's
 * loads, hence the split.)  SMILE_RET_DIRECT=0 keeps Y + smile_combine(2) for all rows. */
typedef enum { SMILE_XCHG_COPY = 0, SMILE_XCHG_PEER = 1 } smile_xchg;

/* ---------------- emulated heterogeneous fabric ----------------
 * AN IN-BOX EMULATION, NOT A MEASUREMENT OF A REAL NETWORK.  The paper's premise is a
 * hierarchical interconnect: fast links inside a node, a slower, latency-bound network
 * between nodes, where the naive All2All issues O(mn) point-to-point messages per rank and
 * bi-level routing O(m + n) (tab:performance_table P:L325).  One B200
 * box has a uniform NVSwitch fabric, so the two levels cost the same per byte there.  With
 * a fabric set, every transfer of the COPY exchange between two ranks of DIFFERENT groups
 * (node s = rank / m) -- in both layers, every level, both directions -- is carried by an
 * emulated NIC of the sending rank: the NIC sends its cross-node messages one after
 * another, each taking latency_us + bytes / inter_gbps of wall time (bytes = the valid
 * rows of the message; every (sender, receiver) pair is one message, as in the NCCL loop
 * of P:L64-76), all ranks' NICs concurrently.  Same-node transfers stay device copies.
 * Data movement only: results are bit-identical to the plain COPY exchange.
 * Needs nprocs == 1 (every rank on this GPU) and the COPY exchange; inter_gbps <= 0
 * disables it.  Each emulated NIC copies with 16 CTAs; a message whose rows take longer to
 * copy than its window delays the next one, so bandwidths above that copy rate are not
 * emulated faithfully (the bench reports the model's expected exchange time beside the
 * measured one). */
typedef struct {
    double inter_gbps;        /* bytes per second / 1e9 of one rank's emulated NIC */
    double inter_latency_us;  /* fixed cost per cross-node message */
} smile_fabric;
smile_status smile_set_fabric(smile_ctx ctx, const smile_fabric *fabric);
/* The 72-byte IPC description of workspace `ws` (64-byte cudaIpcMemHandle of the
 * allocation containing it + the 8-byte offset of ws inside it), to be all-gathered by
 * the caller. */
smile_status smile_ipc_handle(smile_ctx ctx, const void *ws, uint8_t out[72]);
/* Registers `ws` (smile_sizes.ws_bytes, 256-byte aligned) as the workspace of every later
 * smile_forward and selects the exchange.  PEER with nprocs > 1: `handles` = the nprocs
 * handles from smile_ipc_handle in process order (collective; the caller must barrier all
 * processes after this call returns, before the first smile_forward); nprocs == 1:
 * handles may be NULL.  Synchronises the device.
 * Barriers: each All2All of the peer exchange is a flag barrier of the processes of the
 * level; its epoch counter lives on the device (one per level, advanced by the barrier
 * kernel itself), so a captured CUDA graph of the steps stays correct on every replay.
 * A barrier that waits longer than SMILE_BARRIER_TIMEOUT_MS (environment, read here;
 * default 60000, 0 = wait forever) for a peer gives up, sets the sticky device flag to
 * SMILE_ETIMEOUT (smile_get_error) and lets the stream continue (the step's results are
 * then invalid) instead of hanging or trapping the context. */
smile_status smile_register_workspace(smile_ctx ctx, void *ws, const uint8_t *handles, int32_t xchg);
/* Binds the layer output out [V, T, d] (dtype) for the following step calls (NULL unbinds;
 * smile_forward binds its io->out for the duration of an inference call by itself).  With
 * the peer-store exchange, bf16 and the tcgen05 FFN, an inference forward then also fuses
 * the level-1 return into the expert FFN's GEMM 2, in both modes:
 *  - BILEVEL: the level-1 permute records each row's source token at the intermediate,
 *    the level-2 permute forwards it to the expert, and GEMM 2 writes
 *    out[t] = bf16(gate[t] * bf16(y)) (R24, the same arithmetic as smile_combine(1)) for
 *    every token whose intermediate and expert share the process; tokens dropped at
 *    level 2 get their zero row from the level-2 permute.
 *  - FLAT (the Switch layer, P:L43-47 with k = 1): the level-1 permute records each row's
 *    source token at the expert, and GEMM 2 writes out[t] = bf16(p[t] * bf16(y)) for every
 *    token whose expert shares the process.
 * smile_combine(1) into the same out fills only the other tokens.  When every rank of the
 * job is in this process (G == V) the level-1 permute also writes the zero rows of tokens
 * dropped at level 1, and smile_combine(1) into the bound out returns without launching
 * anything.  After such a forward, smile_combine(1) into any other buffer fails with
 * SMILE_EINVAL -- every time, until the next level-1 dispatch (the fused rows were never
 * written to ret1 / Y; they are already in the bound buffer).  The gate used is the
 * route->gate passed to smile_dispatch(1).  Not used by smile_expert_ffn_train (the
 * backward needs the return rows).  SMILE_OUT_DIRECT=0 disables it. */
smile_status smile_set_output(smile_ctx ctx, void *out);

/* ---------------- the steps of the layer ---------------- */

/* Per-token routing decisions [V, T] (SoA).  Top-k FLAT layer (shape.topk = k > 1): dest1,
 * slot1 and gate are [k, V, T] choice-major -- choice j of token (v, t) at j*V*T + v*T + t,
 * dest1 = its expert (R29), gate = its weight p_e (Eq. 2, R30), slot1 = its capacity slot
 * in choice-major order (R31); p [V, T] = the top-1 probability. */
typedef struct {
    int32_t *dest1;   /* i: level-1 destination, first argmax of logits[0, K1) (R2, R3) */
    int32_t *dest2;   /* j: level-2 destination, first argmax of logits[K1, K1+K2) (FLAT: 0) */
    int32_t *slot1;   /* after smile_gate_inter: rank within its block; after
                         smile_dispatch(level 1): # earlier tokens of the rank with the same
                         dest1 -- kept iff slot1 < C1 */
    float *p;         /* top-1 inter probability 1/sum_k exp(r_k - r_i) (Eq. 1, R4) */
    float *q;         /* top-1 intra probability (FLAT: 1) */
    float *gate;      /* fp32(p*q) (Eq. 3, R24) */
} smile_route;

/* Load-balancing statistics per resident rank (R13): argmax counts before
 * capacity and sums of all softmax entries over the rank's T tokens. */
typedef struct {
    int32_t *hist1;   /* [V, K1] */
    int32_t *hist2;   /* [V, K2] */
    double *psum1;    /* [V, K1] */
    double *psum2;    /* [V, K2] */
} smile_stats;

/* a1-a3: level-1 gate at the source.  x [V, T, d] (dtype) with w_router [KW, d] fp32
 * (fused router, rows 0..K1-1 = W_p, then W_q) when logits == NULL, else the
 * caller-supplied fp32 logits [V, T, KW].  logits_out (optional, fused mode only)
 * receives the computed fp32 logits.  Writes route, stats, counts1 [V, K1] =
 * min(hist1, C1).  Scratch for the capacity scan lives in the context. */
smile_status smile_gate_inter(smile_ctx ctx, const void *x, const float *w_router,
                              const float *logits, float *logits_out, const smile_route *route,
                              const smile_stats *stats, int32_t *counts1, void *stream);

/* a1-a4 fused (fused router only): smile_gate_inter followed by smile_dispatch(level 1)
 * in one pass over x where the 128-token tensor-core gate applies (bf16, d % 64 == 0, the
 * context created with the 128-token tile: KW > 40 or SMILE_GATE_SWAP=0): the final
 * level-1 slots come from a decoupled look-back over the tiles' destination histograms
 * inside the gate kernel, which then moves every kept row to its slot (send_rows /
 * send_meta as smile_dispatch(1) writes them, or the destinations' receive buffers with
 * the peer-store exchange).  Same outputs as the two calls (route, stats, counts1, rows,
 * meta).  Returns SMILE_ENOTSUP (launching nothing) where the fused kernel does not apply,
 * so a caller always knows which path ran.  logits_out: optional [V, T, KW]. */
smile_status smile_gate_dispatch_inter(smile_ctx ctx, const void *x, const float *w_router, float *logits_out,
                                       const smile_route *route, const smile_stats *stats, int32_t *counts1,
                                       void *send_rows, int32_t *send_meta, void *stream);

/* a4 (level 1) / a7 (level 2): permute token rows into per-destination send buffers --
 * the per-peer offset layout of the paper's All2All ("sendbuff + r*rankdiff", P:L67-71,
 * Fig. code_all2all_nccl) filled in the routing order of P:L107 (a token goes first to a
 * node, then to a GPU of that node), capacity slots by R5/R8.
 * level 1: rows_in = x [V, T, d]; finalises route->slot1; send_rows [V, K1, C1, d];
 *   send_meta [V, K1, C1] = j of the token in that slot, -1 for empty slots (BILEVEL),
 *   unused (may be NULL) in FLAT.
 * level 2 (BILEVEL only): rows_in = recv1 [V, n, C1, d]; recv_meta [V, n, C1] from the
 *   inter exchange; slot2 [V, n, C1] as written by smile_gate_intra (finalised here:
 *   running count per j in received order, R8); send_rows [V, K2, C2, d] (= [V, m, e,
 *   C2, d]).  Padding rows are never written. */
smile_status smile_dispatch(smile_ctx ctx, int32_t level, const void *rows_in,
                            const smile_route *route, const int32_t *recv_meta, int32_t *slot2,
                            void *send_rows, int32_t *send_meta, void *stream);

/* a6: level-2 gate at the intermediate rank (i, l) -- the intra-node router's decision
 * "then assigned to a GPU via an intra-node router" applied where the token lands
 * after the first of the "four sequential All2All operations"; j itself was
 * computed at the source from the tied W_q (R12).  Ranks the valid received slots of
 * recv_meta [V, n, C1] per j in received order (source node ascending, then slot,
 * R8) into slot2 [V, n, C1] (block-local until smile_dispatch level 2) and writes
 * counts2 [V, K2] = min(#received per j, C2). */
smile_status smile_gate_intra(smile_ctx ctx, const int32_t *recv_meta, int32_t *slot2,
                              int32_t *counts2, void *stream);

/* a5/a12 (inter), a8/a10 (intra), flat world exchange (a15): the capacity-padded
 * equal-split All2All of one level.  Chunk p of send (rows
 * [V, P, rows_per_peer, d] and ints [V, P, ints_per_peer]) goes to the p-th member of
 * the rank's group, which receives it as chunk pos(sender).  level: 1 = inter
 * (rows_per_peer = C1, ints = C1 meta), 2 = intra (e*C2 rows, e counts), 0 = world
 * (FLAT: e*C1 rows, e counts).  reverse != 0 is the return trip of the same level
 * (rows only, send_ints/recv_ints ignored); `fwd_counts` is the forward trip's
 * per-chunk valid-row counts (level 1: counts1 [V, n]; level 2: counts2 [V, K2];
 * world: counts1 [V, K1]) used by the device-copy path to move only valid rows;
 * NCCL moves whole padded chunks (R25) -- or, with SMILE_XCHG_EXACT=1 in the environment,
 * only the valid rows of every (peer, sub-chunk): the counts travel first and the host
 * reads them (one stream synchronisation per forward trip, so not CUDA-graph capturable;
 * the reverse trip reuses them). */
smile_status smile_all2all(smile_ctx ctx, int32_t level, int32_t reverse, const void *send_rows,
                           void *recv_rows, const int32_t *send_ints, int32_t *recv_ints,
                           const int32_t *fwd_counts, void *stream);
smile_status smile_all2all_inter(smile_ctx ctx, int32_t reverse, const void *send_rows,
                                 void *recv_rows, const int32_t *send_meta, int32_t *recv_meta,
                                 const int32_t *fwd_counts, void *stream);
smile_status smile_all2all_intra(smile_ctx ctx, int32_t reverse, const void *send_rows,
                                 void *recv_rows, const int32_t *send_cnt, int32_t *recv_cnt,
                                 const int32_t *fwd_counts, void *stream);

/* a9: expert FFN -- E_e(x) of P:L45-47 ("the sub-model (e.g. multi-layer perceptron) for
 * expert e"), the FFN the MoE layer replaces with GELU activation (dropout omitted,
 * R21): Y = GELU(X W1 + b1) W2 + b2 (exact erf GELU) for every resident
 * expert over its S segments: X, Y [V, S, e, Cseg, d], counts [V, S, e] valid rows per
 * segment; W1t [V*e, d_ff, d] and W2t [V*e, d, d_ff] (K-major transposes, dtype);
 * b1 [V*e, d_ff], b2 [V*e, d] fp32; H_ws [V, S, e, Cseg, d_ff] (dtype).  bf16: tcgen05
 * MMA with fp32 accumulation in TMEM, H rounded to bf16; fp32: SIMT FFMA. */
smile_status smile_expert_ffn(smile_ctx ctx, const void *X, const int32_t *counts,
                              const void *W1t, const float *b1, const void *W2t, const float *b2,
                              void *H_ws, void *Y, void *stream);

/* a11 (level 2) / a13 (level 1): un-permute and combine.
 * level 2: ret1[s, c] = keep2 ? ret_rows[j, slot2] : 0 for every valid received slot
 *   (recv_meta >= 0); ret_rows [V, K2, C2, d], out = ret1 [V, n, C1, d].
 * level 1: out[t] = slot1 < C1 ? dtype(gate[t] * ret_rows[dest1, slot1]) : 0;
 *   ret_rows [V, K1, C1, d], out [V, T, d].  The residual is the caller's. */
smile_status smile_combine(smile_ctx ctx, int32_t level, const void *ret_rows,
                           const smile_route *route, const int32_t *recv_meta,
                           const int32_t *slot2, void *out, void *stream);

/* a14: Eq. (4) per resident rank in fp64: loss[v] = alpha*K1*sum_i (hist1_i/T)(psum1_i/T)
 * + beta*K2*sum_j (hist2_j/T)(psum2_j/T) (FLAT: first term only, the Switch loss). */
smile_status smile_aux_loss(smile_ctx ctx, const smile_stats *stats, double alpha, double beta,
                            double *loss, void *stream);

/* ---------------- training: the backward pass (configuration C3) ----
 * The paper trains the layer (Eq. 5) but gives no backward; these calls are
 * the chain rule of Eq. (3) and Eq. (4) for the objective
 *     J = sum_t <gout[t], out[t]> + lam * sum_v loss[v]
 * with the dispatch fractions f held constant (argmax indicators).  Gradient rows travel
 * the forward route (capacity slots and drops of the forward are reused, nothing is
 * re-routed), and dX travels the return route. */

/* Forward of the expert FFN that also stores Gp = GELU'(A1), the activation derivative at
 * the pre-activation A1 = X W1 + b1 (dtype, [V, S, e, Cseg, d_ff]), which is all the
 * backward needs of A1 (dZ = dH . GELU'(A1)); computed in GEMM 1's epilogue from the same
 * erf evaluation as H = GELU(A1). */
smile_status smile_expert_ffn_train(smile_ctx ctx, const void *X, const int32_t *counts, const void *W1t,
                                    const float *b1, const void *W2t, const float *b2, void *Gp_ws, void *H_ws,
                                    void *Y, void *stream);

/* a16 + a19 (router part): combine backward at the source.  gout [V, T, d] = dJ/dout;
 * back1 [V, K1, C1, d] the forward's returned expert rows (before the gate); logits
 * [V, T, KW] fp32 the forward's router logits; route / stats of the forward.  Writes
 * dsend [V, K1, C1, d] = gate * gout at (dest1, slot1) of every level-1-kept token and
 * dlogits [V, T, KW] fp32 = dJ/dlogits (Eq. 3 through p_i q_j, Eq. 4 through P, Q). */
smile_status smile_combine_bwd(smile_ctx ctx, const void *gout, const void *back1, const float *logits,
                               const smile_route *route, const smile_stats *stats, double alpha, double beta,
                               double lam, void *dsend, float *dlogits, void *stream);

/* a16 (level 2): gradient rows at the intermediate follow the forward route:
 * dsend2[v, j, slot2] = drecv1[v, s, c] for every kept received slot (BILEVEL).  With
 * the peer-store exchange the row is stored straight into the expert's Y buffer (the
 * row its forward input used), and dsend2 is not written. */
smile_status smile_dispatch_grad(smile_ctx ctx, const void *drecv1, const int32_t *recv_meta,
                                 const int32_t *slot2, void *dsend2, void *stream);

/* a17: backward of every resident expert over its segments.  X, dY [V, S, e, Cseg, d];
 * Gp = GELU'(A1), H [V, S, e, Cseg, d_ff] saved by smile_expert_ffn_train; W1 [V*e, d, d_ff]
 * and W2 [V*e, d_ff, d] in their math layouts (the transposes of the forward's W1t / W2t).
 * Writes dZ_ws = (dY W2^T) . Gp [V, S, e, Cseg, d_ff] (may alias Gp),
 * dX = dZ W1^T [V, S, e, Cseg, d] and fp32 dW1 [V*e, d, d_ff], db1 [V*e, d_ff],
 * dW2 [V*e, d_ff, d], db2 [V*e, d] summed over the valid rows.  dX may alias dY (every
 * read of dY precedes the dX GEMM).  bf16: dZ, dX on tcgen05, and dW1, dW2 too when d
 * and d_ff are multiples of 128 (MN-major operands; else SIMT); biases by fixed-order
 * two-pass column sums (deterministic). */
smile_status smile_expert_ffn_bwd(smile_ctx ctx, const void *X, const int32_t *counts, const void *Gp,
                                  const void *H, const void *dY, const void *W1, const void *W2, void *dZ_ws,
                                  void *dX, float *dW1, float *db1, float *dW2, float *db2, void *stream);

/* a18: the last step of the dX return: dx[t] = slot1 < C1 ? ret_rows[dest1, slot1] : 0
 * (rows already carry the gate factor from smile_combine_bwd). */
smile_status smile_combine_grad(smile_ctx ctx, const void *ret_rows, const smile_route *route, void *dx,
                                void *stream);

/* a19: fused-router gradient: dx += dlogits W (in place, dtype) and dW [KW, d] fp32 =
 * sum over every resident token of dlogits^T x (the router is tied; summing
 * across processes is the caller's data-parallel all-reduce).  partial_ws: scratch of
 * smile_sizes.router_partial_bytes. */
smile_status smile_router_bwd(smile_ctx ctx, const void *x, const float *w_router, const float *dlogits,
                              void *dx, float *dW, void *partial_ws, void *stream);

/* ---------------- whole layer ---------------- */

/* Caller-owned buffers of one layer; shapes as in the step calls. */
typedef struct {
    const void *x;            /* [V, T, d] */
    const float *logits;      /* [V, T, KW] or NULL for the fused router */
    const float *w_router;    /* [KW, d] (fused router) */
    const void *W1t; const float *b1; const void *W2t; const float *b2;
    void *out;                /* [V, T, d] */
    double *loss;             /* [V] */
    double alpha, beta;
    void *ws;                 /* smile_sizes.ws_bytes bytes, 256-byte aligned */
    int32_t train;            /* != 0: also save what smile_backward needs (GELU'(A1), router logits) */
} smile_layer_io;

/* Gradients of one layer (smile_backward).  gout [V, T, d] dtype in; dx [V, T, d] dtype,
 * dW_router [KW, d] fp32 (fused router only, else NULL), dW1 / db1 / dW2 / db2 fp32 out
 * (shapes of smile_expert_ffn_bwd); W1 / W2 the math layouts of the expert weights. */
typedef struct {
    const void *gout;
    void *dx;
    float *dW_router;
    const void *W1; const void *W2;
    float *dW1; float *db1; float *dW2; float *db2;
    double lam;               /* weight of the aux loss in J */
} smile_grad_io;

/* Device pointers into the workspace of smile_forward, for inspection. */
typedef struct {
    smile_route route; smile_stats stats;
    int32_t *counts1;                       /* [V, K1] */
    void *send1; int32_t *meta1;            /* [V, K1, C1, d], [V, K1, C1] */
    void *recv1; int32_t *rmeta1;           /* [V, n, C1, d], [V, n, C1] (BILEVEL) */
    int32_t *slot2, *counts2;               /* [V, n, C1], [V, K2] */
    void *send2; void *recv2;               /* [V, K2, C2, d] (BILEVEL) */
    int32_t *rcounts;                       /* [V, S, e] valid rows per FFN segment */
    void *ffn_in; void *H; void *Y;         /* [V, S, e, Cseg, d|d_ff] */
    void *ret2; void *ret1; void *back1;    /* return-path buffers */
    void *A1;                               /* [V, S, e, Cseg, d_ff] GELU'(pre-activation) (train) */
    float *logits; float *dlogits;          /* [V, T, KW] saved logits (train), their gradient */
    void *rpartial;                         /* router-gradient partial sums */
    void *flags;                            /* peer-exchange barrier flags */
} smile_ws_view;

smile_status smile_forward_ws(smile_ctx ctx, void *ws, smile_ws_view *view);

/* The whole forward of the layer on `stream`, in the paper's order (§3.2.3: four
 * sequential All2Alls): gate_inter, dispatch(1), all2all_inter, gate_intra, dispatch(2),
 * all2all_intra, expert_ffn, all2all_intra(rev), combine(2), all2all_inter(rev),
 * combine(1), aux_loss.  FLAT: gate, dispatch(1), all2all(world), ffn,
 * all2all(world, rev), combine(1), aux_loss.
 * T == 0: returns SMILE_OK without touching any buffer (x, out may be NULL; the loss,
 * which divides by T, is not written). */
smile_status smile_forward(smile_ctx ctx, const smile_layer_io *io, void *stream);

/* the paper's "pipe_overlapping" appendix: the layer
 * over c micro-batches ("chunks") of T/c tokens per rank, software-pipelined on two
 * streams: the expert FFN of chunk k (stream2) overlaps the gate + permutes + exchanges
 * of chunk k+1 and the return path of chunk k-1 (stream).  Each chunk is an independent
 * layer with its own capacities ceil(cf * (T/c) / K) (R5 applied to the chunk), so it
 * computes exactly what smile_forward computes for that chunk alone.
 * ctxs[k]: nchunks DISTINCT contexts created with identical shapes (T = tokens per chunk);
 * ios[k]: chunk k's layer io (x, out [V, T/c, d] contiguous, its own workspace -- the
 * registered one in peer mode -- weights and loss [V]); inference only (train == 0).
 * Enqueues on both streams (stream2 first waits for the work already on stream) and
 * returns; the result is complete when `stream` reaches the end of the enqueued work.
 * nchunks <= 64. */
smile_status smile_forward_chunked(smile_ctx const *ctxs, const smile_layer_io *ios, int32_t nchunks, void *stream,
                                   void *stream2);

/* The whole backward after a forward with io->train set, in reverse order of the forward:
 * combine_bwd, exchange(1, gradient rows), dispatch_grad, exchange(2), expert_ffn_bwd,
 * exchange(2, reverse), combine(2), exchange(1, reverse), combine_grad, router_bwd.
 * Works over both exchanges; with the peer-store exchange (smile_register_workspace)
 * the gradient rows are stored at / loaded from their owners and every exchange is a
 * barrier, as in the forward.
 * T == 0: the weight gradients (dW1, db1, dW2, db2 and dW_router when given) are sums
 * over no tokens and are set to 0; nothing else is touched (gout, dx may be NULL). */
smile_status smile_backward(smile_ctx ctx, const smile_layer_io *io, const smile_grad_io *g, void *stream);

/* End to end from HOST memory: copies host_x [V, T, d] (and host_logits when non-NULL)
 * to io->x / io->logits, runs smile_forward, copies io->out to host_out and io->loss to
 * host_loss, all on `stream`; synchronises `stream` before returning.  Host buffers
 * should be pinned for asynchronous copies. */
smile_status smile_forward_host(smile_ctx ctx, const smile_layer_io *io, const void *host_x,
                                const float *host_logits, void *host_out, double *host_loss,
                                void *stream);

/* Streams nb batches through the layer from pinned host memory with copy / compute
 * overlap: batch b's host->device copy (one copy engine) runs while batch b-1 is in the
 * layer and batch b-2's result is copied back (the other copy engine).  Every batch's
 * H2D and D2H are part of the call.  x_dev[2], out_dev[2]: caller-owned device
 * ping-pong buffers [V, T, d] (dtype); io->x / io->out are ignored (the ping-pong
 * buffers are used), io->loss holds V doubles (device) and is copied to
 * host_loss + b*V after each batch.  host_x[b] / host_out[b]: pinned [V, T, d].
 * Supplied logits are not streamed (io->logits must be NULL: fused router).  The
 * library's own copy streams and events are created with the context; `stream` is the
 * compute stream.  Blocks until the last D2H has completed. */
smile_status smile_forward_host_stream(smile_ctx ctx, const smile_layer_io *io, void *const *x_dev,
                                       void *const *out_dev, int32_t nb, const void *const *host_x,
                                       void *const *host_out, double *host_loss, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* SMILE_H */
