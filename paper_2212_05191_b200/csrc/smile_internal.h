// smile_internal.h -- private declarations shared by the libsmile translation units.
// Product code: never includes anything under oracle/.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <nccl.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/smile.h"

namespace smile {

constexpr int kWarp = 32;

// Host-side count of libsmile kernel launches (smile_launch_count); every launch site
// calls it immediately before its <<<>>> / cudaLaunchKernelEx.
void note_launch();

// Programmatic dependent launch (PDL) for the kernels of the forward chain: a kernel
// launched with launch_k may be scheduled while the previous kernel on the stream is still
// finishing; its first statement is pdl_wait() (griddepcontrol.wait: blocks until the
// previous grid has completed and its memory is visible -- so no global access happens
// before it), and the big kernels call pdl_trigger() after their main loop so the next
// grid's launch and prologue overlap their tail.  SMILE_PDL=0 disables the attribute.
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
#endif
bool pdl_enabled();

// Diagnostic per-CTA timelines (measurement only; tools/gpu/trace_kernels.py): with
// SMILE_TRACE=<name> ("gate", "ffn1", "ffn2") the named kernel gets a device buffer of
// kTraceSlots clock64 stamps per CTA (slot 0 / 1: %globaltimer at start / end, slots 2 / 3:
// clock64 at start / end, the rest kernel-specific), read back by smile_debug_trace (not part
// of smile.h).  Null otherwise: every stamp is one predicated branch.
constexpr int kTraceSlots = 1024;
unsigned long long *trace_buffer(const char *name);   // nullptr unless SMILE_TRACE == name
#ifdef __CUDACC__
__device__ __forceinline__ void trace_clock(unsigned long long *tr, int slot) {
    if (tr) {
        long long t = clock64();
        tr[(size_t)blockIdx.x * kTraceSlots + slot] = (unsigned long long)t;
    }
}
__device__ __forceinline__ void trace_begin(unsigned long long *tr) {
    if (tr && threadIdx.x == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        tr[(size_t)blockIdx.x * kTraceSlots + 0] = g;
        trace_clock(tr, 2);
    }
}
__device__ __forceinline__ void trace_end(unsigned long long *tr) {
    if (tr && threadIdx.x == 0) {
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        tr[(size_t)blockIdx.x * kTraceSlots + 1] = g;
        trace_clock(tr, 3);
    }
}
#endif
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Tokens per block of the level-1 gate (sized so the logits tile stays <= 32 KB of smem).
inline int gate_tokens_per_block(int KW) {
    if (KW <= 32) return 256;
    if (KW <= 64) return 128;
    if (KW <= 128) return 64;
    return 32;
}
constexpr int kRank2Items = 256;     // received slots per block of the level-2 gate

// Exchange topology of one level for the resident ranks (host-built at smile_create).
struct Level {
    int P = 1;                 // group size (peers incl. self)
    int nsub = 1;              // sub-chunks per peer chunk (e experts, or 1)
    int64_t Csub = 0;          // rows per sub-chunk
    int ints_per_peer = 0;     // side ints per peer chunk (meta or counts)
    int32_t *d_member_local = nullptr;  // [V, P] local index of member p, -1 if remote
    int32_t *d_mypos = nullptr;         // [V]   position of resident rank v in its group
    int32_t *h_member = nullptr;        // [V, P] global rank of member p (host)
    int32_t *h_mypos = nullptr;         // [V]
    int any_remote = 0;
    ncclComm_t comm = nullptr;          // split comm when V == 1 (inter/intra) or world
    // exact-size NCCL exchange (SMILE_XCHG_EXACT=1): per-chunk valid-row counts [V, P, nsub]
    int32_t *d_rcnt = nullptr;          // device: counts received from the peers (forward)
    int32_t *h_scnt = nullptr, *h_rcnt = nullptr;   // host copies of the last forward's counts
};

// Fused permute -> peer-store exchange (SMILE_XCHG_PEER): every process's workspace
// base (its own, or a CUDA-IPC mapping over NVLink) and the byte offsets of the receive
// buffers inside a workspace (all processes share one layout).  bases == nullptr: the
// classic path (permute into send buffers, then an explicit exchange).
struct PeerMap {
    char *const *bases;                // [nprocs] device array
    int V, rank0, n, m, e, G;
    int64_t off_recv1, off_rmeta1, off_recv2, off_rcounts, off_Y, off_ret1;
    int64_t off_rrow;                  // BILEVEL: [V, S, e, Cseg] i32 ret1 row of each expert input row
    int64_t off_rtok1;                 // BILEVEL: [V, n, C1] i32 source token of each received slot
    int64_t off_rtok2;                 // [V, S, e, Cseg] i32 source token of each expert input row
};
constexpr int kMaxProcs = 64;

}  // namespace smile

struct smile_ctx_s {
    smile_shape shape;
    smile_sizes sz;
    int TB1 = 256;             // gate tokens per block
    bool ret_direct = false;   // PEER: the last expert FFN stored its output in the intermediates' ret1
    void *out_bound = nullptr; // smile_set_output: the layer output [V, T, d] of the next steps
    bool rtok1_valid = false;  // PEER: the last level-1 permute recorded the source tokens
    bool out_planned = false;  // PEER: this forward writes in-process rows straight to out
    bool out_direct = false;   // ... and the last expert FFN did
    bool l1_zeroed = false;    // ... and the level-1 permute wrote the level-1-dropped zero rows
    bool l1_pending = false;   // the last expert FFN wrote out rows directly: until the next level-1
                               // dispatch, smile_combine(1) may only target the bound output
    const float *d1_gate = nullptr;   // route->gate of the last smile_dispatch(1)
    int nblk1 = 0;             // gate table blocks per rank (TB1 tokens each)
    bool gate_swapped = false; // the tensor-core gate is the swapped-role 256-token kernel
    int *gate_sync = nullptr;  // [3] swapped gate: split-ready, done, look-back epoch
    int nblk2 = 0;             // level-2 ranking blocks per rank
    int *d_err = nullptr;      // sticky device error flag (smile_status)
    int32_t *blk_hist1 = nullptr, *blk_off1 = nullptr, *blk_hist2a = nullptr;
    double *blk_psum = nullptr;
    int32_t *blk_hist2 = nullptr, *blk_off2 = nullptr;
    ncclComm_t world = nullptr, inter = nullptr, intra = nullptr;
    smile::Level lv[3];        // 0 world, 1 inter, 2 intra
    int num_sms = 148;
    smile_fabric fabric{};     // emulated inter-node fabric (COPY exchange, nprocs == 1)
    // peer-store exchange (smile_register_workspace)
    int xchg = 0;                            // smile_xchg
    void *reg_ws = nullptr;                  // the registered workspace
    char **d_bases = nullptr;                // [nprocs] device array of workspace bases
    char *h_bases[smile::kMaxProcs] = {};    // host copy (own + IPC-opened, + offset)
    void *h_ipc[smile::kMaxProcs] = {};      // bases returned by cudaIpcOpenMemHandle
    int64_t off_flags = 0;                   // barrier flags inside a workspace
    int32_t *d_peers[3] = {};                // per level: processes to synchronise with
    int npeers[3] = {};
    long long *d_epoch = nullptr;            // [3] device barrier epochs (advanced by the barrier kernel)
    unsigned long long barrier_timeout_ns = 0;   // 0: wait forever (SMILE_BARRIER_TIMEOUT_MS)
    smile::PeerMap peer{};
    // tensor-core gate (bf16 fused router): the three-piece bf16 split of the router
    __nv_bfloat16 *wsplit = nullptr;         // [gate_tc_np(KW), d], rewritten every fused gate call
    float *colsum_ws = nullptr;              // bias-gradient partials of smile_expert_ffn_bwd
    int *lb_flag = nullptr;                  // fused gate + permute: look-back flags [V * nblk1]
    int32_t *lb_agg = nullptr, *lb_inc = nullptr;   // tile aggregates / inclusive prefixes [V * nblk1 * K1]
    int *lb_scan_flag = nullptr;             // the gates' in-kernel level-1 scan: epoch-tagged flags [V * nblk1]
    // smile_forward_host_stream: copy streams and ping-pong events (created with the ctx)
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
    cudaEvent_t ev_chunk_front = nullptr, ev_chunk_ffn = nullptr;   // smile_forward_chunked
};

namespace smile {

// ---- launchers implemented in the .cu files (all asynchronous on `st`) ----
struct GateArgs {
    const void *x; const float *w; const float *logits; float *logits_out;
    smile_route route; int32_t *blk_hist1, *blk_hist2a; double *blk_psum;
    int *err; int V; int64_t T; int d; int K1, K2, KW; int TB, nblk; int flat; int bf16;
    int topk;                // FLAT top-k (tables [V][topk][nblk], route [topk][V][T] for dest1 / slot1 / gate)
    int swapped;             // tensor-core gate: the swapped-role 256-token kernel (KW <= 40)
    // fused level-1 permute (tensor-core gate only; smile_gate_dispatch_inter): final
    // slots by decoupled look-back over the tiles' destination histograms, then the
    // kept rows moved to their slots (send rows / meta, or the peers' receive buffers)
    int fuse_dispatch;
    void *send; int32_t *meta; int64_t rowbytes; int64_t C1;
    PeerMap peer;
    int *lb_flag; int32_t *lb_agg, *lb_inc;   // [V * nblk], [V * nblk * K1] x 2
};
void launch_gate1(const GateArgs &a, cudaStream_t st);

struct Scan1Args {
    const int32_t *blk_hist1, *blk_hist2a; const double *blk_psum; int32_t *blk_off1;
    smile_stats stats; int32_t *counts1; int V, nblk, K1, K2, KW; int64_t C1; int flat; int64_t T;
    PeerMap peer;            // nblk: table blocks per rank and choice
    int *lb_flag;            // reset for the next fused gate (may be null)
    int nlb;                 // look-back tiles per rank (lb_flag entries)
    int32_t *lb_inc;         // look-back inclusive prefixes (the swapped gate's in-kernel scan)
    int topk;
};
void launch_scan1(const Scan1Args &a, cudaStream_t st);

struct Rank2Args {
    const int32_t *recv_meta; int32_t *slot2; int32_t *blk_hist2; int32_t *blk_off2;
    int32_t *counts2; int *err; int V; int64_t items; int K2; int nblk; int64_t C2;
    PeerMap peer;
};
void launch_rank2(const Rank2Args &a, cudaStream_t st);

struct Dispatch1Args {
    const void *x; smile_route route; const int32_t *blk_off1; const int32_t *blk_hist1;
    void *send; int32_t *meta; int V; int64_t T; int64_t rowbytes; int K1; int64_t C1; int TB, nblk;
    int topk;                          // FLAT top-k: topk * V * T items, choice-major (R31)
    PeerMap peer;
    void *out;                         // PEER + output bound, every rank in this process: tokens
                                       // dropped at level 1 get their zero output row here
};
void launch_dispatch1(const Dispatch1Args &a, cudaStream_t st);
// meta = -1 for the empty slots [count, C1) (after the fused gate + permute)
void launch_meta_fill(const Dispatch1Args &a, cudaStream_t st);

struct Dispatch2Args {
    const void *recv1; const int32_t *recv_meta; int32_t *slot2; const int32_t *blk_off2;
    void *send2; int V; int64_t items; int64_t rowbytes; int K2; int64_t C2; int nblk;
    void *ret1;                        // PEER: level-2-dropped rows get their zero return row here
    void *out; int64_t T;              // PEER + output bound: ... or, for sources and experts in
                                       // this process, a zero row in the layer output
    PeerMap peer;
};
void launch_dispatch2(const Dispatch2Args &a, cudaStream_t st);

struct Combine2Args {
    const void *ret2; const int32_t *recv_meta; const int32_t *slot2; void *ret1;
    int V; int64_t items; int64_t rowbytes; int K2; int64_t C2;
    int skip_local;                    // PEER: rows of experts in this process are in ret1 already
    PeerMap peer;
};
void launch_combine2(const Combine2Args &a, cudaStream_t st);

struct Combine1Args {
    const void *back1; smile_route route; void *out; int V; int64_t T; int d; int K1; int64_t C1;
    int bf16; int nogate;      // nogate: gradient return (a18), rows copied unscaled
    PeerMap peer;
    int skip_direct;           // PEER: tokens whose intermediate and expert are in this process
                               // were written by the expert's GEMM 2 (smile_set_output)
    int topk;                  // FLAT top-k (> 1): out[t] = sum over kept choices of gate_j * row_j
};
void launch_combine1(const Combine1Args &a, cudaStream_t st);

// a7 for gradient rows (a16): dsend2[v, j, slot2] = drecv1[v, s, c] with the forward's final slot2.
void launch_grad_dispatch2(const Dispatch2Args &a, cudaStream_t st);

// a16 + a19 (router part): combine backward at the source.
struct CombineBwdArgs {
    const void *gout; const void *back1; const float *logits; smile_route route; smile_stats stats;
    void *dsend; float *dlogits; int V; int64_t T; int d; int K1, K2, KW; int64_t C1;
    double alpha, beta, lam; int flat; int bf16;
    PeerMap peer;            // PEER: back1 rows are loaded from, and gradient rows stored to, their owner
    int topk;                // FLAT top-k: every choice's gradient row and dgate (Eq. 2)
};
void launch_combine_bwd(const CombineBwdArgs &a, cudaStream_t st);

// a19: router weight / input gradient: dx[t] += dlogits[t] W;  dW = sum_t dlogits[t]^T x[t].
struct RouterBwdArgs {
    const void *x; const float *w; const float *dlogits; void *dx; float *dW; float *partial;
    int64_t rows; int d; int KW; int nchunk; int bf16;
};
void launch_router_bwd(const RouterBwdArgs &a, cudaStream_t st);
size_t router_bwd_partial_floats(int64_t rows, int d, int KW);

// Process-level barrier of one level over NVLink flags (peer-store exchange).
// The epoch is a device counter advanced by the kernel (CUDA-graph replay safe); a wait
// longer than timeout_ns (0 = forever) sets *err = SMILE_ETIMEOUT and returns.
void launch_peer_barrier(char *const *bases, int64_t off_flags, int me, const int32_t *peers, int npeers, int level,
                         long long *epoch, unsigned long long timeout_ns, int *err, cudaStream_t st);

void launch_aux(const smile_stats &s, double alpha, double beta, double *loss, int V, int K1,
                int K2, int64_t T, int flat, cudaStream_t st);

struct CopyXArgs {
    const char *send; char *recv; const int32_t *sint; int32_t *rint; const int32_t *cnt;
    const int32_t *member_local; const int32_t *mypos; int V, P, nsub; int64_t Csub;
    int64_t rowbytes; int ipp; int rev;
    // emulated heterogeneous fabric (smile_set_fabric): pairs whose ranks lie in different
    // groups ("nodes", rank / m) are skipped by the device copy and carried by the sender's
    // emulated NIC instead (launch_fabric_copy)
    int fabric; int rank0, m;
    double ns_per_byte; double latency_ns;
};
void launch_exchange_copy(const CopyXArgs &a, cudaStream_t st);
// The cross-node pairs of one exchange through per-rank emulated NICs: one CTA per sending
// rank handles its cross-node messages one after another, each costing latency + bytes /
// bandwidth of wall time (globaltimer), with the rows moved inside that window.
void launch_fabric_copy(const CopyXArgs &a, cudaStream_t st);

struct FfnArgs {
    const void *X; const int32_t *counts; const void *W1t; const float *b1; const void *W2t;
    const float *b2; void *H; void *Y; int V, S, e; int64_t Cseg; int d, d_ff; int bf16;
    int num_sms;
    // PEER, BILEVEL (ret.bases != nullptr): GEMM 2 stores each output row straight into
    // its intermediate's ret1 (the level-2 un-permute, a10 + a11) instead of Y, at the row
    // permute 2 recorded in rrow [V, S, e, Cseg] (this process's workspace)
    PeerMap ret;
    const int32_t *rrow;
    // inference with the layer output bound (smile_set_output): rows whose source rank is
    // in this process too go straight to out[t] as gate * y (a12 + a13 fused as well)
    void *out; const float *gate; const int32_t *rtok2; int64_t T, C1; int n;
    // FLAT: ret carries only the process layout; segment s of an expert is source rank s,
    // and rows of in-process sources go straight to out (rtok2 from the level-1 permute)
    int flat_out;
};
void launch_ffn_simt(const FfnArgs &a, cudaStream_t st);

// Training forward / backward of the expert FFN.
struct FfnBwdArgs {
    const void *X; const int32_t *counts; const void *A1; const void *H; const void *dY;
    const void *W1; const void *W2;          // math layouts: W1 [NE, d, d_ff], W2 [NE, d_ff, d]
    void *dZ; void *dX; float *dW1; float *db1; float *dW2; float *db2;
    int V, S, e; int64_t Cseg; int d, d_ff; int bf16; int num_sms;
    float *colsum_ws;                        // bias-gradient partials (colsum_ws_bytes)
};
cudaError_t launch_ffn_bwd(const FfnBwdArgs &a, bool tc, cudaStream_t st);
// Forward that also stores GELU'(A1), A1 = X W1 + b1 the pre-activation (training).
cudaError_t launch_ffn_fwd_train(const FfnArgs &a, void *A1, bool tc, cudaStream_t st);
// Returns cudaErrorNotSupported when the shape cannot run on the tcgen05 path.
cudaError_t launch_ffn_tcgen05(const FfnArgs &a, cudaStream_t st);

// Weight / bias gradients (wgrad_tcgen05.cu).
size_t colsum_ws_bytes(int NE, int S, int64_t Cseg, int maxN);
void launch_colsum(const void *B, float *db, float *part, const int32_t *counts, int NE, int e, int S, int64_t Cseg,
                   int N, int bf16, cudaStream_t st);
// db[E][n] = sum over the expert's valid 32-row strips of part[(g * nstr + u) * N + n]
// (strip partials written by the dZ GEMM's epilogue), fixed order.
void launch_colsum_strips(const float *part, float *db, const int32_t *counts, int NE, int e, int S, int nstr, int N,
                          cudaStream_t st);
bool wgrad_tc_supported(int bf16, int d, int d_ff, int S);
cudaError_t launch_wgrad_tc(const void *A, int M, const void *B, int N, float *Dw, const int32_t *counts, int V, int S,
                            int e, int64_t Cseg, int num_sms, cudaStream_t st);
void launch_pad_rows_zero(void *buf, const int32_t *counts, int nseg, int64_t Cseg, int cols, cudaStream_t st);

// Level-1 gate with the router on tcgen05 (gate_tcgen05.cu); needs TB == 128.
int gate_tc_np(int KW);
bool gate_tc_swapped(int KW);        // the swapped-role kernel (256-token tiles of 2 table blocks) for this KW
int gate_tc_rows(int KW);            // rows of the split-router buffer
bool gate_tc_supported(int bf16, int d, int KW);
// a.swapped: the swapped-role kernel, which also builds the split router (counters in
// gate_sync [2]); else the 128-token kernel (split by router_split_kernel).
// With `scan` (lb_flag, lb_inc set) the swapped kernel also runs the level-1 scan by
// look-back and sets *scanned (then no scan1_kernel is needed).
cudaError_t launch_gate1_tc(const GateArgs &a, __nv_bfloat16 *wsplit, int num_sms, int *gate_sync, const Scan1Args *scan,
                            bool *scanned, cudaStream_t st);

}  // namespace smile
