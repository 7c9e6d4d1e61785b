// api.cu -- the C ABI of libsmile (include/smile.h): validation, context, NCCL
// process groups, the exchange of each level, and the whole-layer sequence.
#include "smile_internal.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <algorithm>
#include <atomic>
#include <vector>

namespace smile {
bool ffn_simt_supported(int nseg, int d, int d_ff);
}

using namespace smile;

#define CUDA_TRY(x)                                   \
    do {                                              \
        if ((x) != cudaSuccess) return SMILE_ECUDA;   \
    } while (0)
#define NCCL_TRY(x)                                   \
    do {                                              \
        if ((x) != ncclSuccess) return SMILE_ENCCL;   \
    } while (0)

#define STEP(x)                            \
    do {                                   \
        smile_status _s = (x);             \
        if (_s != SMILE_OK) return _s;     \
    } while (0)

static inline cudaStream_t S(void *p) { return reinterpret_cast<cudaStream_t>(p); }

extern "C" int smile_version(void) { return SMILE_VERSION; }

extern "C" smile_status smile_struct_sizes(int64_t *out, int32_t n) {
    const int64_t s[8] = {(int64_t)sizeof(smile_shape),    (int64_t)sizeof(smile_sizes),  (int64_t)sizeof(smile_route),
                          (int64_t)sizeof(smile_stats),    (int64_t)sizeof(smile_layer_io), (int64_t)sizeof(smile_ws_view),
                          (int64_t)sizeof(smile_grad_io),  (int64_t)sizeof(smile_xop)};
    if (!out || n < 0) return SMILE_EINVAL;
    for (int i = 0; i < n && i < 8; ++i) out[i] = s[i];
    return SMILE_OK;
}

extern "C" const char *smile_strerror(smile_status s) {
    switch (s) {
        case SMILE_OK: return "ok";
        case SMILE_EINVAL: return "invalid argument";
        case SMILE_ESHAPE: return "shape or layout mismatch";
        case SMILE_ENONFINITE: return "non-finite router logit";
        case SMILE_ECUDA: return "CUDA error";
        case SMILE_ENCCL: return "NCCL error";
        case SMILE_ENOTSUP: return "unsupported configuration";
        case SMILE_EINDEX: return "routing index out of range";
        case SMILE_ETIMEOUT: return "peer-exchange barrier timed out";
    }
    return "unknown status";
}

// R5, R20: capacity ceil(cf*T/dests); one destination = no capacity.
static int64_t capacity(int64_t T, int64_t dests, double cf) {
    if (T <= 0) return 0;
    if (dests <= 1) return T;
    return (int64_t)ceil(cf * (double)T / (double)dests);
}

extern "C" int64_t smile_capacity(int64_t T, int64_t dests, double cf) {
    if (T < 0 || dests < 1 || !(cf > 0.0)) return -1;
    return capacity(T, dests, cf);
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Workspace carve-up for smile_forward (also gives ws_bytes).
struct WsLayout {
    size_t off[32];
    size_t total;
};

static void ws_layout(const smile_shape *s, const smile_sizes *z, WsLayout *L, smile_ws_view *view,
                      char *base, char **rrow_out = nullptr, char **rtok1_out = nullptr,
                      char **rtok2_out = nullptr) {
    const int64_t V = z->V, T = s->T;
    const int64_t eb = s->dtype == SMILE_BF16 ? 2 : 4;
    const int64_t rb = (int64_t)s->d * eb;
    const bool bi = s->mode == SMILE_BILEVEL;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += align256(bytes ? bytes : 1); return base ? base + r : nullptr; };
    smile_ws_view w;
    memset(&w, 0, sizeof(w));
    const int64_t k = s->topk > 1 ? s->topk : 1;           // choices per token (FLAT top-k)
    w.route.dest1 = (int32_t *)take(k * V * T * 4);
    w.route.dest2 = (int32_t *)take(V * T * 4);
    w.route.slot1 = (int32_t *)take(k * V * T * 4);
    w.route.p = (float *)take(V * T * 4);
    w.route.q = (float *)take(V * T * 4);
    w.route.gate = (float *)take(k * V * T * 4);
    w.stats.hist1 = (int32_t *)take(V * z->K1 * 4);
    w.stats.hist2 = (int32_t *)take(V * z->K2 * 4);
    w.stats.psum1 = (double *)take(V * z->K1 * 8);
    w.stats.psum2 = (double *)take(V * z->K2 * 8);
    w.counts1 = (int32_t *)take(V * z->K1 * 4);
    w.send1 = take(V * z->K1 * z->C1 * rb);
    w.meta1 = (int32_t *)take(V * z->K1 * z->C1 * 4);
    w.recv1 = take(V * z->K1 * z->C1 * rb);      // BILEVEL: [V, n, C1, d]; FLAT: [V, G, e, C, d]
    w.rmeta1 = (int32_t *)take(bi ? V * z->K1 * z->C1 * 4 : 0);
    if (bi) {
        w.slot2 = (int32_t *)take(V * z->K1 * z->C1 * 4);
        w.counts2 = (int32_t *)take(V * z->K2 * 4);
        w.send2 = take(V * z->K2 * z->C2 * rb);
        w.recv2 = take(V * z->K2 * z->C2 * rb);
    }
    w.rcounts = (int32_t *)take(V * z->S * s->e * 4);
    w.ffn_in = bi ? w.recv2 : w.recv1;
    const int64_t ffn_rows = V * z->S * s->e * z->Cseg;
    w.H = take(ffn_rows * s->d_ff * eb);
    w.Y = take(ffn_rows * rb);
    if (bi) {
        w.ret2 = take(V * z->K2 * z->C2 * rb);
        w.ret1 = take(V * z->K1 * z->C1 * rb);
    }
    w.back1 = take(V * z->K1 * z->C1 * rb);
    w.A1 = take(ffn_rows * s->d_ff * eb);
    w.logits = (float *)take(V * T * z->KW * 4);
    w.dlogits = (float *)take(V * T * z->KW * 4);
    w.rpartial = take(z->router_partial_bytes);
    w.flags = take(3 * kMaxProcs * 8);
    char *rrow = take(bi ? ffn_rows * 4 : 0);       // internal: ret1 row of each expert input row
    if (rrow_out) *rrow_out = rrow;
    char *rtok1 = take(bi ? V * z->K1 * z->C1 * 4 : 0);   // internal: source token per received slot
    char *rtok2 = take(ffn_rows * 4);                     // internal: source token per expert row
    if (rtok1_out) *rtok1_out = rtok1;
    if (rtok2_out) *rtok2_out = rtok2;
    if (L) L->total = o;
    if (view) *view = w;
}

extern "C" smile_status smile_plan(const smile_shape *s, smile_sizes *out) {
    if (!s || !out) return SMILE_EINVAL;
    if (s->n < 1 || s->m < 1 || s->e < 1 || s->d < 1 || s->d_ff < 1 || s->T < 0 || !(s->cf > 0.0))
        return SMILE_EINVAL;
    if (s->mode != SMILE_BILEVEL && s->mode != SMILE_FLAT) return SMILE_EINVAL;
    if (s->dtype != SMILE_FP32 && s->dtype != SMILE_BF16) return SMILE_EINVAL;
    const int G = s->n * s->m;
    if (s->nprocs < 1 || G % s->nprocs != 0 || s->proc < 0 || s->proc >= s->nprocs) return SMILE_EINVAL;
    if (s->T > (int64_t)1 << 30) return SMILE_ENOTSUP;
    const int topk = s->topk > 1 ? s->topk : 1;
    if (s->topk < 0) return SMILE_EINVAL;
    if (topk > 1 && (s->mode != SMILE_FLAT || topk > 4 || topk > G * s->e)) return SMILE_ENOTSUP;   // R29-R32
    const int eb = s->dtype == SMILE_BF16 ? 2 : 4;
    if ((s->d * eb) % 16 != 0 || (s->d_ff * eb) % 16 != 0) return SMILE_ESHAPE;
    smile_sizes z;
    memset(&z, 0, sizeof(z));
    z.G = G;
    z.V = G / s->nprocs;
    z.rank0 = s->proc * z.V;
    const bool bi = s->mode == SMILE_BILEVEL;
    z.K1 = bi ? s->n : G * s->e;
    z.K2 = bi ? s->m * s->e : 1;
    z.KW = bi ? z.K1 + z.K2 : z.K1;
    z.C1 = capacity((int64_t)topk * s->T, z.K1, s->cf);      // R31: k T items per rank
    z.C2 = bi ? (z.K2 > 1 ? capacity(s->T, z.K2, s->cf) : (int64_t)s->n * z.C1) : 0;
    z.S = bi ? s->m : G;
    z.Cseg = bi ? z.C2 : z.C1;
    if (z.KW > 512 || z.K2 > 256) return SMILE_ENOTSUP;   // gate smem tile / level-2 rank limits
    z.router_partial_bytes = router_bwd_partial_floats((int64_t)z.V * s->T, s->d, z.KW) * 4;
    WsLayout L;
    ws_layout(s, &z, &L, nullptr, nullptr);
    z.ws_bytes = L.total;
    *out = z;
    return SMILE_OK;
}

// Group of global rank r (R10): level 1 = inter {(i, l)}_i positioned by node,
// level 2 = intra {(s, g)}_g positioned by local index, level 0 = world.
static void group_of(int n, int m, int level, int r, std::vector<int> &mem, int *mypos) {
    const int s = r / m, l = r % m;
    mem.clear();
    if (level == 1) {
        for (int i = 0; i < n; ++i) mem.push_back(i * m + l);
        *mypos = s;
    } else if (level == 2) {
        for (int g = 0; g < m; ++g) mem.push_back(s * m + g);
        *mypos = l;
    } else {
        for (int q = 0; q < n * m; ++q) mem.push_back(q);
        *mypos = r;
    }
}

extern "C" smile_status smile_group(const smile_shape *shape, int32_t level, int32_t r, int32_t *members,
                                    int32_t *count) {
    if (!shape || !members || !count || shape->n < 1 || shape->m < 1) return SMILE_EINVAL;
    if (level < 0 || level > 2 || r < 0 || r >= shape->n * shape->m) return SMILE_EINVAL;
    std::vector<int> mem;
    int pos = 0;
    group_of(shape->n, shape->m, level, r, mem, &pos);
    for (size_t i = 0; i < mem.size(); ++i) members[i] = mem[i];
    *count = (int32_t)mem.size();
    return SMILE_OK;
}

// Remote transfers of one level for process shape->proc (see smile.h).
static void exchange_ops(const smile_shape *sh, int level, std::vector<smile_xop> &out) {
    const int G = sh->n * sh->m, V = G / sh->nprocs, rank0 = sh->proc * V;
    std::vector<int> mem;
    std::vector<smile_xop> sends, recvs;
    for (int v = 0; v < V; ++v) {
        int mp = 0;
        group_of(sh->n, sh->m, level, rank0 + v, mem, &mp);
        const int P = (int)mem.size();
        for (int p = 0; p < P; ++p) {
            const int q = mem[p];
            if (q / V == sh->proc) continue;                     // same process: device copy
            // chunk p of rank v goes to member q, which files it under our position mp;
            // q's chunk at position mp comes back into our chunk p (the level is an involution)
            sends.push_back({0, q / V, rank0 + v, q, v * P + p});
            recvs.push_back({1, q / V, q, rank0 + v, v * P + p});
        }
    }
    auto by_pair = [](const smile_xop &a, const smile_xop &b) { return a.src != b.src ? a.src < b.src : a.dst < b.dst; };
    std::sort(sends.begin(), sends.end(), by_pair);
    std::sort(recvs.begin(), recvs.end(), by_pair);
    out = sends;
    out.insert(out.end(), recvs.begin(), recvs.end());
}

extern "C" smile_status smile_exchange_plan(const smile_shape *shape, int32_t level, smile_xop *ops, int32_t cap,
                                            int32_t *count) {
    if (!shape || !count || level < 0 || level > 2) return SMILE_EINVAL;
    smile_sizes z;
    smile_status st = smile_plan(shape, &z);
    if (st != SMILE_OK) return st;
    std::vector<smile_xop> v;
    exchange_ops(shape, level, v);
    *count = (int32_t)v.size();
    if ((int32_t)v.size() > cap || (!ops && !v.empty())) return SMILE_ESHAPE;
    for (size_t i = 0; i < v.size(); ++i) ops[i] = v[i];
    return SMILE_OK;
}

extern "C" smile_status smile_get_unique_id(uint8_t out[128]) {
    if (!out) return SMILE_EINVAL;
    ncclUniqueId id;
    NCCL_TRY(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "nccl unique id size");
    memcpy(out, &id, 128);
    return SMILE_OK;
}

static smile_status build_level(smile_ctx c, int level, int P, int nsub, int64_t Csub, int ipp) {
    Level &L = c->lv[level];
    const int V = c->sz.V;
    L.P = P; L.nsub = nsub; L.Csub = Csub; L.ints_per_peer = ipp;
    std::vector<int32_t> mloc(V * P), mglob(V * P), pos(V);
    std::vector<int> mem;
    L.any_remote = 0;
    for (int v = 0; v < V; ++v) {
        int mp = 0;
        group_of(c->shape.n, c->shape.m, level, c->sz.rank0 + v, mem, &mp);
        pos[v] = mp;
        for (int p = 0; p < P; ++p) {
            mglob[v * P + p] = mem[p];
            const int ql = mem[p] - c->sz.rank0;
            mloc[v * P + p] = (ql >= 0 && ql < V) ? ql : -1;
            if (mloc[v * P + p] < 0) L.any_remote = 1;
        }
    }
    L.h_member = (int32_t *)malloc(sizeof(int32_t) * V * P);
    L.h_mypos = (int32_t *)malloc(sizeof(int32_t) * V);
    memcpy(L.h_member, mglob.data(), sizeof(int32_t) * V * P);
    memcpy(L.h_mypos, pos.data(), sizeof(int32_t) * V);
    CUDA_TRY(cudaMalloc(&L.d_member_local, sizeof(int32_t) * V * P));
    CUDA_TRY(cudaMalloc(&L.d_mypos, sizeof(int32_t) * V));
    CUDA_TRY(cudaMemcpy(L.d_member_local, mloc.data(), sizeof(int32_t) * V * P, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(L.d_mypos, pos.data(), sizeof(int32_t) * V, cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc(&L.d_rcnt, sizeof(int32_t) * V * P * nsub));
    CUDA_TRY(cudaMallocHost(&L.h_scnt, sizeof(int32_t) * V * P * nsub));
    CUDA_TRY(cudaMallocHost(&L.h_rcnt, sizeof(int32_t) * V * P * nsub));
    return SMILE_OK;
}

extern "C" smile_status smile_create(smile_ctx *out, const smile_shape *shape, const uint8_t *nccl_id) {
    if (!out || !shape) return SMILE_EINVAL;
    smile_sizes z;
    smile_status st = smile_plan(shape, &z);
    if (st != SMILE_OK) return st;
    if (shape->nprocs > 1 && !nccl_id) return SMILE_EINVAL;
    CUDA_TRY(cudaSetDevice(shape->device));
    smile_ctx c = new smile_ctx_s();
    c->shape = *shape;
    c->sz = z;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, shape->device);
    const int V = z.V;
    c->TB1 = gate_tokens_per_block(z.KW);
    {
        const char *e = getenv("SMILE_GATE_TC");
        const bool tc_on = !(e && e[0] == '0');
        if (tc_on && gate_tc_supported(shape->dtype == SMILE_BF16, shape->d, z.KW)) {
            c->gate_swapped = gate_tc_swapped(z.KW);
            c->TB1 = c->gate_swapped ? 256 : 128;   // the tensor-core gate's token tile = table block
            const size_t wb = (size_t)gate_tc_rows(z.KW) * shape->d * 2;
            if (cudaMalloc(&c->wsplit, wb) != cudaSuccess) { delete c; return SMILE_ECUDA; }
            // look-back state of the fused gate + permute (flags zero between calls)
            const int64_t nt = (int64_t)z.V * ((shape->T + 127) / 128);   // (the fused path's 128-token tiles)
            if (cudaMalloc(&c->lb_flag, (nt > 0 ? nt : 1) * 4) != cudaSuccess ||
                cudaMalloc(&c->lb_scan_flag, (nt > 0 ? nt : 1) * 4) != cudaSuccess ||
                cudaMemset(c->lb_scan_flag, 0, (nt > 0 ? nt : 1) * 4) != cudaSuccess ||
                cudaMalloc(&c->lb_agg, (nt > 0 ? nt : 1) * z.K1 * 4) != cudaSuccess ||
                cudaMalloc(&c->lb_inc, (nt > 0 ? nt : 1) * z.K1 * 4) != cudaSuccess ||
                cudaMemset(c->lb_flag, 0, (nt > 0 ? nt : 1) * 4) != cudaSuccess) {
                delete c;
                return SMILE_ECUDA;
            }
        }
    }
    c->nblk1 = (int)((shape->T + c->TB1 - 1) / c->TB1);
    const int64_t items2 = (int64_t)shape->n * z.C1;
    c->nblk2 = shape->mode == SMILE_BILEVEL ? (int)((items2 + kRank2Items - 1) / kRank2Items) : 0;
    const int topk = shape->topk > 1 ? shape->topk : 1;
    const size_t nb1 = (size_t)V * topk * (c->nblk1 > 0 ? c->nblk1 : 1);   // [V][topk][nblk] tables
    const size_t nb2 = (size_t)V * (c->nblk2 > 0 ? c->nblk2 : 1);
    CUDA_TRY(cudaMalloc(&c->d_err, sizeof(int)));
    CUDA_TRY(cudaMemset(c->d_err, 0, sizeof(int)));
    CUDA_TRY(cudaMalloc(&c->gate_sync, sizeof(int) * 3));
    CUDA_TRY(cudaMemset(c->gate_sync, 0, sizeof(int) * 3));
    CUDA_TRY(cudaMalloc(&c->blk_hist1, nb1 * z.K1 * 4));
    CUDA_TRY(cudaMalloc(&c->blk_off1, nb1 * z.K1 * 4));
    CUDA_TRY(cudaMalloc(&c->blk_hist2a, nb1 * z.K2 * 4));
    CUDA_TRY(cudaMalloc(&c->blk_psum, nb1 * (z.K1 + z.K2) * 8));
    CUDA_TRY(cudaMalloc(&c->blk_hist2, nb2 * z.K2 * 4));
    CUDA_TRY(cudaMalloc(&c->blk_off2, nb2 * z.K2 * 4));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_chunk_front, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&c->ev_chunk_ffn, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_h2d[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_comp[i], cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&c->ev_d2h[i], cudaEventDisableTiming));
    }
    {
        const size_t cb = colsum_ws_bytes(V * shape->e, (int)z.S, z.Cseg, std::max(shape->d, shape->d_ff));
        if (cudaMalloc(&c->colsum_ws, cb) != cudaSuccess) { smile_destroy(c); return SMILE_ECUDA; }
    }
    const int n = shape->n, m = shape->m, e = shape->e, G = z.G;
    if (shape->mode == SMILE_BILEVEL) {
        st = build_level(c, 1, n, 1, z.C1, (int)z.C1);
        if (st == SMILE_OK) st = build_level(c, 2, m, e, z.C2, e);
    } else {
        st = build_level(c, 0, G, e, z.C1, e);
    }
    if (st != SMILE_OK) { smile_destroy(c); return st; }
    if (shape->nprocs > 1) {
        ncclUniqueId id;
        memcpy(&id, nccl_id, sizeof(id));
        if (ncclCommInitRank(&c->world, shape->nprocs, id, shape->proc) != ncclSuccess) {
            smile_destroy(c);
            return SMILE_ENCCL;
        }
        c->lv[0].comm = c->world;
        if (V == 1) {
            // one inter-node and one intra-node process group per process.
            const int r = z.rank0, s = r / m, l = r % m;
            if (ncclCommSplit(c->world, l, s, &c->inter, nullptr) != ncclSuccess ||
                ncclCommSplit(c->world, s, l, &c->intra, nullptr) != ncclSuccess) {
                smile_destroy(c);
                return SMILE_ENCCL;
            }
            c->lv[1].comm = c->inter;
            c->lv[2].comm = c->intra;
        }
    }
    *out = c;
    return SMILE_OK;
}

extern "C" smile_status smile_destroy(smile_ctx c) {
    if (!c) return SMILE_EINVAL;
    cudaSetDevice(c->shape.device);
    if (c->inter) ncclCommDestroy(c->inter);
    if (c->intra) ncclCommDestroy(c->intra);
    if (c->world) ncclCommDestroy(c->world);
    cudaFree(c->d_err);
    cudaFree(c->gate_sync);
    cudaFree(c->wsplit);
    cudaFree(c->colsum_ws);
    cudaFree(c->lb_flag); cudaFree(c->lb_agg); cudaFree(c->lb_inc); cudaFree(c->lb_scan_flag);
    if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
    if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
    if (c->ev_chunk_front) cudaEventDestroy(c->ev_chunk_front);
    if (c->ev_chunk_ffn) cudaEventDestroy(c->ev_chunk_ffn);
    for (int i = 0; i < 2; ++i) {
        if (c->ev_h2d[i]) cudaEventDestroy(c->ev_h2d[i]);
        if (c->ev_comp[i]) cudaEventDestroy(c->ev_comp[i]);
        if (c->ev_d2h[i]) cudaEventDestroy(c->ev_d2h[i]);
    }
    cudaFree(c->blk_hist1); cudaFree(c->blk_off1); cudaFree(c->blk_hist2a); cudaFree(c->blk_psum);
    cudaFree(c->blk_hist2); cudaFree(c->blk_off2);
    for (int p = 0; p < kMaxProcs; ++p)
        if (c->h_ipc[p]) cudaIpcCloseMemHandle(c->h_ipc[p]);
    cudaFree(c->d_bases);
    for (int l = 0; l < 3; ++l) cudaFree(c->d_peers[l]);
    for (auto &L : c->lv) {
        cudaFree(L.d_member_local); cudaFree(L.d_mypos); cudaFree(L.d_rcnt);
        cudaFreeHost(L.h_scnt); cudaFreeHost(L.h_rcnt);
        free(L.h_member); free(L.h_mypos);
    }
    delete c;
    return SMILE_OK;
}

extern "C" smile_status smile_query(smile_ctx c, smile_sizes *out) {
    if (!c || !out) return SMILE_EINVAL;
    *out = c->sz;
    return SMILE_OK;
}

// ---- fused permute -> peer-store exchange ----------------------------------------
typedef int (*GetAddressRangeFn)(void **base, size_t *size, void *ptr);   // cuMemGetAddressRange_v2

extern "C" smile_status smile_ipc_handle(smile_ctx c, const void *ws, uint8_t out[72]) {
    if (!c || !ws || !out) return SMILE_EINVAL;
    cudaSetDevice(c->shape.device);
    static GetAddressRangeFn range_fn = nullptr;
    if (!range_fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return SMILE_ECUDA;
        range_fn = reinterpret_cast<GetAddressRangeFn>(p);
    }
    void *base = nullptr;
    size_t size = 0;
    if (range_fn(&base, &size, const_cast<void *>(ws)) != 0) return SMILE_ECUDA;
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, base));
    const uint64_t off = (uint64_t)((const char *)ws - (const char *)base);
    memcpy(out, &h, 64);
    memcpy(out + 64, &off, 8);
    return SMILE_OK;
}

extern "C" smile_status smile_register_workspace(smile_ctx c, void *ws, const uint8_t *handles, int32_t xchg) {
    if (!c || !ws || (xchg != SMILE_XCHG_COPY && xchg != SMILE_XCHG_PEER)) return SMILE_EINVAL;
    if (((uintptr_t)ws & 255) != 0) return SMILE_ESHAPE;
    const int P = c->shape.nprocs, me = c->shape.proc;
    if (P > kMaxProcs) return SMILE_ENOTSUP;
    if (xchg == SMILE_XCHG_PEER && P > 1 && !handles) return SMILE_EINVAL;
    if (xchg == SMILE_XCHG_PEER && c->fabric.inter_gbps > 0.0) return SMILE_ENOTSUP;   // fabric: COPY only
    cudaSetDevice(c->shape.device);
    c->reg_ws = ws;
    c->xchg = xchg;
    if (xchg == SMILE_XCHG_COPY) return SMILE_OK;
    smile_ws_view w;
    char *rrow = nullptr, *rtok1 = nullptr, *rtok2 = nullptr;
    ws_layout(&c->shape, &c->sz, nullptr, &w, (char *)ws, &rrow, &rtok1, &rtok2);
    auto off = [&](const void *ptr) { return (int64_t)((const char *)ptr - (const char *)ws); };
    c->off_flags = off(w.flags);
    CUDA_TRY(cudaMemset(w.flags, 0, 3 * kMaxProcs * 8));
    // barrier epochs live on the device (advanced by the barrier kernel: graph-replay safe)
    if (!c->d_epoch) CUDA_TRY(cudaMalloc(&c->d_epoch, 3 * sizeof(long long)));
    CUDA_TRY(cudaMemset(c->d_epoch, 0, 3 * sizeof(long long)));
    {
        const char *e = getenv("SMILE_BARRIER_TIMEOUT_MS");
        const long long ms = e ? atoll(e) : 60000;
        c->barrier_timeout_ns = ms > 0 ? (unsigned long long)ms * 1000000ull : 0ull;
    }
    for (int p = 0; p < P; ++p) {
        if (p == me) { c->h_bases[p] = (char *)ws; continue; }
        if (c->h_bases[p]) continue;                       // already opened
        cudaIpcMemHandle_t h;
        uint64_t o = 0;
        memcpy(&h, handles + (size_t)p * 72, 64);
        memcpy(&o, handles + (size_t)p * 72 + 64, 8);
        void *base = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        c->h_ipc[p] = base;
        c->h_bases[p] = (char *)base + o;
    }
    if (!c->d_bases) CUDA_TRY(cudaMalloc(&c->d_bases, sizeof(char *) * kMaxProcs));
    CUDA_TRY(cudaMemcpy(c->d_bases, c->h_bases, sizeof(char *) * kMaxProcs, cudaMemcpyHostToDevice));
    // processes each level must synchronise with: owners of the members of our ranks' groups
    const bool bi = c->shape.mode == SMILE_BILEVEL;
    for (int level = 0; level < 3; ++level) {
        std::vector<int32_t> peers;
        const bool used = bi ? level != 0 : level == 0;        // BILEVEL: inter + intra; FLAT: world
        if (used) {
            std::vector<int> mem;
            for (int v = 0; v < c->sz.V; ++v) {
                int mp = 0;
                group_of(c->shape.n, c->shape.m, level, c->sz.rank0 + v, mem, &mp);
                for (int q : mem) {
                    const int pq = q / c->sz.V;
                    if (pq != me && std::find(peers.begin(), peers.end(), pq) == peers.end()) peers.push_back(pq);
                }
            }
            std::sort(peers.begin(), peers.end());
        }
        c->npeers[level] = (int)peers.size();
        if (!c->d_peers[level]) CUDA_TRY(cudaMalloc(&c->d_peers[level], sizeof(int32_t) * kMaxProcs));
        if (!peers.empty())
            CUDA_TRY(cudaMemcpy(c->d_peers[level], peers.data(), sizeof(int32_t) * peers.size(), cudaMemcpyHostToDevice));
    }
    PeerMap &pm = c->peer;
    pm.bases = c->d_bases; pm.V = c->sz.V; pm.rank0 = c->sz.rank0; pm.n = bi ? c->shape.n : 0; pm.m = c->shape.m;
    pm.e = c->shape.e; pm.G = c->sz.G;
    pm.off_recv1 = off(w.recv1); pm.off_rmeta1 = bi ? off(w.rmeta1) : 0; pm.off_recv2 = bi ? off(w.recv2) : 0;
    pm.off_rcounts = off(w.rcounts); pm.off_Y = off(w.Y); pm.off_ret1 = bi ? off(w.ret1) : 0;
    pm.off_rrow = bi ? (int64_t)(rrow - (char *)ws) : 0;
    pm.off_rtok1 = bi ? (int64_t)(rtok1 - (char *)ws) : 0;
    pm.off_rtok2 = (int64_t)(rtok2 - (char *)ws);
    CUDA_TRY(cudaDeviceSynchronize());
    return SMILE_OK;
}

static void peer_barrier(smile_ctx c, int level, cudaStream_t st) {
    if (c->shape.nprocs <= 1 || c->npeers[level] == 0) return;
    launch_peer_barrier(c->d_bases, c->off_flags, c->shape.proc, c->d_peers[level], c->npeers[level], level,
                        c->d_epoch + level, c->barrier_timeout_ns, c->d_err, st);
}

extern "C" smile_status smile_get_error(smile_ctx c, void *stream) {
    if (!c) return SMILE_EINVAL;
    cudaSetDevice(c->shape.device);
    CUDA_TRY(cudaStreamSynchronize(S(stream)));
    int h = 0;
    CUDA_TRY(cudaMemcpy(&h, c->d_err, sizeof(int), cudaMemcpyDeviceToHost));
    CUDA_TRY(cudaMemset(c->d_err, 0, sizeof(int)));
    return (smile_status)h;
}

// Peer map of the step calls: active in SMILE_XCHG_PEER mode (smile_register_workspace).
static inline PeerMap peer_of(smile_ctx c) {
    return c->xchg == SMILE_XCHG_PEER ? c->peer : PeerMap{};
}

namespace smile {
static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
bool pdl_enabled() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SMILE_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v != 0;
}
static unsigned long long *g_trace = nullptr;
static int g_trace_ctas = 0;
unsigned long long *trace_buffer(const char *name) {
    const char *e = getenv("SMILE_TRACE");
    if (!e || strcmp(e, name) != 0) return nullptr;
    if (!g_trace) {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        g_trace_ctas = sms;
        if (cudaMalloc(&g_trace, (size_t)sms * kTraceSlots * 8) != cudaSuccess) return g_trace = nullptr;
        cudaMemset(g_trace, 0, (size_t)sms * kTraceSlots * 8);
    }
    return g_trace;
}
}  // namespace smile

extern "C" int64_t smile_launch_count(void) { return (int64_t)smile::g_launches.load(); }

// Diagnostic (not in smile.h): copy the SMILE_TRACE buffer ([CTAs][kTraceSlots] u64) of the
// last traced launch to host memory; returns the number of CTA rows copied (0: no trace).
extern "C" int64_t smile_debug_trace(void *host, int64_t bytes) {
    if (!smile::g_trace || !host) return 0;
    int64_t rows = bytes / (smile::kTraceSlots * 8);
    if (rows > smile::g_trace_ctas) rows = smile::g_trace_ctas;
    if (cudaMemcpy(host, smile::g_trace, (size_t)rows * smile::kTraceSlots * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
        return -1;
    return rows;
}

static smile_status post_launch() {
    return cudaGetLastError() == cudaSuccess ? SMILE_OK : SMILE_ECUDA;
}

extern "C" smile_status smile_gate_inter(smile_ctx c, const void *x, const float *w_router, const float *logits,
                                         float *logits_out, const smile_route *route, const smile_stats *stats,
                                         int32_t *counts1, void *stream) {
    if (!c || !route || !stats || !counts1) return SMILE_EINVAL;
    if (!logits && (!x || !w_router)) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    GateArgs a{};
    a.x = x; a.w = w_router; a.logits = logits; a.logits_out = logits_out;
    a.route = *route;
    a.blk_hist1 = c->blk_hist1; a.blk_hist2a = c->blk_hist2a; a.blk_psum = c->blk_psum;
    a.err = c->d_err; a.V = c->sz.V; a.T = c->shape.T; a.d = c->shape.d;
    a.K1 = c->sz.K1; a.K2 = c->sz.K2; a.KW = c->sz.KW; a.TB = c->TB1; a.nblk = c->nblk1;
    a.flat = c->shape.mode == SMILE_FLAT; a.bf16 = c->shape.dtype == SMILE_BF16;
    a.topk = c->shape.topk > 1 ? c->shape.topk : 1; a.swapped = c->gate_swapped;
    Scan1Args s{};
    s.blk_hist1 = c->blk_hist1; s.blk_hist2a = c->blk_hist2a; s.blk_psum = c->blk_psum; s.blk_off1 = c->blk_off1;
    s.stats = *stats; s.counts1 = counts1; s.V = c->sz.V; s.nblk = c->nblk1; s.K1 = c->sz.K1; s.K2 = c->sz.K2;
    s.KW = c->sz.KW; s.C1 = c->sz.C1; s.flat = a.flat; s.T = c->shape.T; s.peer = peer_of(c); s.topk = a.topk;
    bool scanned = false;                    // the swapped tensor-core gate scans by look-back itself
    if (!logits && c->wsplit) {
        Scan1Args sl = s;
        sl.lb_flag = c->lb_scan_flag; sl.lb_inc = c->lb_inc;   // epoch-tagged flags of the in-kernel scan
        const cudaError_t e = launch_gate1_tc(a, c->wsplit, c->num_sms, c->gate_sync, &sl, &scanned, S(stream));
        if (e != cudaSuccess) return SMILE_ECUDA;
    } else {
        launch_gate1(a, S(stream));
    }
    if (!scanned) launch_scan1(s, S(stream));
    return post_launch();
}

extern "C" smile_status smile_gate_dispatch_inter(smile_ctx c, const void *x, const float *w_router,
                                                  float *logits_out, const smile_route *route, const smile_stats *stats,
                                                  int32_t *counts1, void *send_rows, int32_t *send_meta, void *stream) {
    if (!c || !x || !w_router || !route || !stats || !counts1 || !send_rows) return SMILE_EINVAL;
    const bool bi = c->shape.mode == SMILE_BILEVEL;
    if (bi && !send_meta) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    // the fused kernel is the 128-token tensor-core gate; elsewhere refuse (the caller runs
    // smile_gate_inter + smile_dispatch(1) and knows which path ran)
    if (!c->wsplit || !c->lb_flag || c->TB1 != 128 || c->gate_swapped || c->shape.topk > 1) return SMILE_ENOTSUP;
    c->rtok1_valid = false;                  // this path does not record the source tokens
    c->out_planned = false;
    c->l1_zeroed = false;
    c->l1_pending = false;
    cudaSetDevice(c->shape.device);
    const int64_t rb = (int64_t)c->shape.d * (c->shape.dtype == SMILE_BF16 ? 2 : 4);
    GateArgs a{};
    a.x = x; a.w = w_router; a.logits = nullptr; a.logits_out = logits_out;
    a.route = *route;
    a.blk_hist1 = c->blk_hist1; a.blk_hist2a = c->blk_hist2a; a.blk_psum = c->blk_psum;
    a.err = c->d_err; a.V = c->sz.V; a.T = c->shape.T; a.d = c->shape.d;
    a.K1 = c->sz.K1; a.K2 = c->sz.K2; a.KW = c->sz.KW; a.TB = c->TB1; a.nblk = c->nblk1; a.topk = 1;
    a.flat = !bi; a.bf16 = c->shape.dtype == SMILE_BF16;
    a.fuse_dispatch = 1; a.send = send_rows; a.meta = bi ? send_meta : nullptr; a.rowbytes = rb; a.C1 = c->sz.C1;
    a.peer = peer_of(c); a.lb_flag = c->lb_flag; a.lb_agg = c->lb_agg; a.lb_inc = c->lb_inc;
    const cudaError_t e = launch_gate1_tc(a, c->wsplit, c->num_sms, nullptr, nullptr, nullptr, S(stream));
    if (e != cudaSuccess) return SMILE_ECUDA;
    Scan1Args s{};
    s.blk_hist1 = c->blk_hist1; s.blk_hist2a = c->blk_hist2a; s.blk_psum = c->blk_psum; s.blk_off1 = c->blk_off1;
    s.stats = *stats; s.counts1 = counts1; s.V = c->sz.V; s.nblk = c->nblk1; s.K1 = c->sz.K1; s.K2 = c->sz.K2;
    s.KW = c->sz.KW; s.C1 = c->sz.C1; s.flat = a.flat; s.T = c->shape.T; s.peer = peer_of(c); s.lb_flag = c->lb_flag;
    s.nlb = c->nblk1; s.topk = 1;
    launch_scan1(s, S(stream));
    Dispatch1Args d{};
    d.x = x; d.route = *route; d.blk_off1 = c->blk_off1; d.blk_hist1 = c->blk_hist1;
    d.send = send_rows; d.meta = bi ? send_meta : nullptr;
    d.V = c->sz.V; d.T = c->shape.T; d.rowbytes = rb; d.K1 = c->sz.K1; d.C1 = c->sz.C1;
    d.TB = c->TB1; d.nblk = c->nblk1; d.topk = 1; d.peer = peer_of(c);
    launch_meta_fill(d, S(stream));
    return post_launch();
}

static bool out_direct_enabled(smile_ctx c);
static bool out_direct_possible(smile_ctx c);

extern "C" smile_status smile_dispatch(smile_ctx c, int32_t level, const void *rows_in, const smile_route *route,
                                       const int32_t *recv_meta, int32_t *slot2, void *send_rows, int32_t *send_meta,
                                       void *stream) {
    if (!c || !rows_in || !send_rows) return SMILE_EINVAL;
    const int64_t rb = (int64_t)c->shape.d * (c->shape.dtype == SMILE_BF16 ? 2 : 4);
    const bool bi = c->shape.mode == SMILE_BILEVEL;
    cudaSetDevice(c->shape.device);
    if (level == 1) {
        if (!route || (bi && !send_meta)) return SMILE_EINVAL;
        if (c->shape.T == 0) return SMILE_OK;
        Dispatch1Args a{};
        a.x = rows_in; a.route = *route; a.blk_off1 = c->blk_off1; a.blk_hist1 = c->blk_hist1;
        a.send = send_rows; a.meta = bi ? send_meta : nullptr;
        a.V = c->sz.V; a.T = c->shape.T; a.rowbytes = rb; a.K1 = c->sz.K1; a.C1 = c->sz.C1;
        a.TB = c->TB1; a.nblk = c->nblk1; a.peer = peer_of(c);
        a.topk = c->shape.topk > 1 ? c->shape.topk : 1;
        // every rank in this process: the whole level-1 return fuses into GEMM 2, so the
        // zero rows of level-1-dropped tokens are written here and combine(1) is skipped
        c->l1_zeroed = out_direct_enabled(c) && c->sz.V == c->sz.G;
        if (c->l1_zeroed) a.out = c->out_bound;
        c->l1_pending = false;               // a new forward: the previous one's fused rows are history
        c->d1_gate = route->gate;            // the gate GEMM 2 scales in-process rows by
        launch_dispatch1(a, S(stream));
        c->rtok1_valid = a.peer.bases != nullptr;   // the source token of each row is recorded
        // FLAT: the permute wrote the rows' source tokens straight to the experts' rtok2
        if (!bi) c->out_planned = out_direct_possible(c);
        return post_launch();
    }
    if (level == 2) {
        if (!bi) return SMILE_EINVAL;
        if (!recv_meta || !slot2) return SMILE_EINVAL;
        if (c->shape.T == 0) return SMILE_OK;
        Dispatch2Args a{};
        a.recv1 = rows_in; a.recv_meta = recv_meta; a.slot2 = slot2; a.blk_off2 = c->blk_off2;
        a.send2 = send_rows; a.V = c->sz.V; a.items = (int64_t)c->shape.n * c->sz.C1; a.rowbytes = rb;
        a.K2 = c->sz.K2; a.C2 = c->sz.C2; a.nblk = c->nblk2; a.peer = peer_of(c);
        if (a.peer.bases) a.ret1 = static_cast<char *>(c->reg_ws) + c->peer.off_ret1;
        c->out_planned = out_direct_possible(c);
        if (c->out_planned) { a.out = c->out_bound; a.T = c->shape.T; }
        launch_dispatch2(a, S(stream));
        return post_launch();
    }
    return SMILE_EINVAL;
}

extern "C" smile_status smile_gate_intra(smile_ctx c, const int32_t *recv_meta, int32_t *slot2, int32_t *counts2,
                                         void *stream) {
    if (!c || !recv_meta || !slot2 || !counts2) return SMILE_EINVAL;
    if (c->shape.mode != SMILE_BILEVEL) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    Rank2Args a{};
    a.recv_meta = recv_meta; a.slot2 = slot2; a.blk_hist2 = c->blk_hist2; a.blk_off2 = c->blk_off2;
    a.counts2 = counts2; a.err = c->d_err; a.V = c->sz.V; a.items = (int64_t)c->shape.n * c->sz.C1;
    a.K2 = c->sz.K2; a.nblk = c->nblk2; a.C2 = c->sz.C2; a.peer = peer_of(c);
    launch_rank2(a, S(stream));
    return post_launch();
}

// SMILE_XCHG_EXACT=1: the NCCL part of an exchange moves only the valid rows of every
// (peer, sub-chunk) -- the counts travel first (a small NCCL exchange), the host reads them
// (one stream sync per forward exchange; the reverse trip reuses them), then grouped
// ncclSend / ncclRecv of exact sizes land the rows at the padded layout's offsets.  Not
// graph-capturable (host sync); the default keeps the equal-split padded chunks (R25).
static bool exact_exchange() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("SMILE_XCHG_EXACT");
        v = (e && e[0] == '1') ? 1 : 0;
    }
    return v != 0;
}

static smile_status all2all_exact(smile_ctx c, int level, int reverse, const void *send_rows, void *recv_rows,
                                  const int32_t *send_ints, int32_t *recv_ints, const int32_t *fwd_counts,
                                  bool split_comm, cudaStream_t st) {
    Level &L = c->lv[level];
    const int V = c->sz.V, P = L.P, ns = L.nsub;
    const int64_t rb = (int64_t)c->shape.d * (c->shape.dtype == SMILE_BF16 ? 2 : 4);
    // the remote transfers of this process: (send?, peer, comm, chunk)
    struct Op { int send; int peer; int chunk; };
    std::vector<Op> ops;
    ncclComm_t comm = split_comm ? L.comm : c->world;
    if (split_comm) {
        // V == 1: comm rank = position in the group; every chunk, our own included (the
        // padded path's ncclAlltoAll covers the self chunk too -- no device copy runs here)
        for (int p = 0; p < P; ++p) ops.push_back({1, p, p});
        for (int p = 0; p < P; ++p) ops.push_back({0, p, p});
    } else {
        std::vector<smile_xop> xo;
        exchange_ops(&c->shape, level, xo);
        for (const smile_xop &o : xo) ops.push_back({o.kind == 0 ? 1 : 0, o.peer_proc, o.chunk});   // kind 0 = send
    }
    const size_t ncnt = (size_t)V * P * ns;
    if (!reverse) {
        // 1. counts: ours to the peers, theirs into d_rcnt (at our chunk of the transfer)
        NCCL_TRY(ncclGroupStart());
        for (const Op &o : ops) {
            if (o.send) NCCL_TRY(ncclSend(fwd_counts + (size_t)o.chunk * ns, ns, ncclInt32, o.peer, comm, st));
            else NCCL_TRY(ncclRecv(L.d_rcnt + (size_t)o.chunk * ns, ns, ncclInt32, o.peer, comm, st));
        }
        NCCL_TRY(ncclGroupEnd());
        CUDA_TRY(cudaMemcpyAsync(L.h_scnt, fwd_counts, ncnt * 4, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaMemcpyAsync(L.h_rcnt, L.d_rcnt, ncnt * 4, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        if (send_ints) {                               // side ints (meta / counts): whole, small
            const int ipp = L.ints_per_peer;
            NCCL_TRY(ncclGroupStart());
            for (const Op &o : ops) {
                if (o.send) NCCL_TRY(ncclSend(send_ints + (size_t)o.chunk * ipp, ipp, ncclInt32, o.peer, comm, st));
                else NCCL_TRY(ncclRecv(recv_ints + (size_t)o.chunk * ipp, ipp, ncclInt32, o.peer, comm, st));
            }
            NCCL_TRY(ncclGroupEnd());
        }
    }
    // 2. rows: exact sizes per (peer, sub-chunk); the reverse trip sends back what came in
    const size_t sub = (size_t)L.Csub * rb;
    NCCL_TRY(ncclGroupStart());
    for (const Op &o : ops) {
        for (int k = 0; k < ns; ++k) {
            const size_t ci = (size_t)o.chunk * ns + k;
            int32_t rows = o.send ? (reverse ? L.h_rcnt[ci] : L.h_scnt[ci]) : (reverse ? L.h_scnt[ci] : L.h_rcnt[ci]);
            if (rows > L.Csub) rows = (int32_t)L.Csub;
            if (rows <= 0) continue;
            const size_t off = ci * sub, bytes = (size_t)rows * rb;
            if (o.send) NCCL_TRY(ncclSend((const char *)send_rows + off, bytes, ncclUint8, o.peer, comm, st));
            else NCCL_TRY(ncclRecv((char *)recv_rows + off, bytes, ncclUint8, o.peer, comm, st));
        }
    }
    NCCL_TRY(ncclGroupEnd());
    return SMILE_OK;
}

// One level's equal-split All2All.  Pairs of ranks resident on this
// device are a device copy; V == 1 uses ncclAlltoAll on the level's split communicator;
// several resident ranks per process plus remote peers use grouped ncclSend/ncclRecv
// on the world communicator, posted in (source rank, destination rank) order on both
// sides so NCCL matches them.
extern "C" smile_status smile_all2all(smile_ctx c, int32_t level, int32_t reverse, const void *send_rows,
                                      void *recv_rows, const int32_t *send_ints, int32_t *recv_ints,
                                      const int32_t *fwd_counts, void *stream) {
    if (!c || !send_rows || !recv_rows || level < 0 || level > 2) return SMILE_EINVAL;
    const bool bi = c->shape.mode == SMILE_BILEVEL;
    if (bi == (level == 0)) return SMILE_EINVAL;
    const Level &L = c->lv[level];
    const bool with_ints = !reverse && send_ints && recv_ints;
    if (!reverse && (!send_ints != !recv_ints)) return SMILE_EINVAL;   // forward: both or neither (rows only)
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    cudaStream_t st = S(stream);
    if (c->xchg == SMILE_XCHG_PEER) {
        // the permute already stored every row at its destination (and the combine loads
        // from its source): the All2All of the level is a barrier of its processes
        peer_barrier(c, level, st);
        return cudaGetLastError() == cudaSuccess ? SMILE_OK : SMILE_ECUDA;
    }
    const int64_t rb = (int64_t)c->shape.d * (c->shape.dtype == SMILE_BF16 ? 2 : 4);
    const size_t chunk = (size_t)L.nsub * L.Csub * rb;
    const int V = c->sz.V, P = L.P;
    const bool nccl_alltoall = c->shape.nprocs > 1 && V == 1 && L.comm;
    if (!nccl_alltoall) {
        CopyXArgs a{};
        a.send = (const char *)send_rows; a.recv = (char *)recv_rows;
        a.sint = with_ints ? send_ints : nullptr; a.rint = with_ints ? recv_ints : nullptr;
        a.cnt = fwd_counts; a.member_local = L.d_member_local; a.mypos = L.d_mypos;
        a.V = V; a.P = P; a.nsub = L.nsub; a.Csub = L.Csub; a.rowbytes = rb; a.ipp = L.ints_per_peer;
        a.rev = reverse ? 1 : 0;
        const bool fab = c->fabric.inter_gbps > 0.0 && c->shape.nprocs == 1;
        if (fab) {
            a.fabric = 1; a.rank0 = c->sz.rank0; a.m = c->shape.m;
            a.ns_per_byte = 1.0 / c->fabric.inter_gbps;          // GB/s = bytes per ns
            a.latency_ns = c->fabric.inter_latency_us * 1e3;
        }
        launch_exchange_copy(a, st);
        if (fab) launch_fabric_copy(a, st);
        if (cudaGetLastError() != cudaSuccess) return SMILE_ECUDA;
    }
    if (c->shape.nprocs == 1) return SMILE_OK;
    if (exact_exchange() && fwd_counts && (nccl_alltoall || L.any_remote))
        return all2all_exact(c, level, reverse, send_rows, recv_rows, with_ints ? send_ints : nullptr,
                             with_ints ? recv_ints : nullptr, fwd_counts, nccl_alltoall, st);
    if (nccl_alltoall) {
        if (with_ints) NCCL_TRY(ncclAlltoAll(send_ints, recv_ints, L.ints_per_peer, ncclInt32, L.comm, st));
        NCCL_TRY(ncclAlltoAll(send_rows, recv_rows, chunk, ncclUint8, L.comm, st));
        return SMILE_OK;
    }
    if (!L.any_remote) return SMILE_OK;
    // mixed: remote pairs over the world communicator, in smile_exchange_plan order.  The
    // side ints (meta / counts) go in their own group first: interleaving them with the
    // multi-MB row messages of the same peer pair in one group serialised NCCL's p2p
    // (measured 8 ms instead of 0.4 ms for the C2 inter exchange on 2 B200).
    std::vector<smile_xop> ops;
    exchange_ops(&c->shape, level, ops);
    const int ipp = L.ints_per_peer;
    if (with_ints) {
        NCCL_TRY(ncclGroupStart());
        for (const smile_xop &o : ops) {
            if (o.kind == 0) NCCL_TRY(ncclSend(send_ints + (size_t)o.chunk * ipp, ipp, ncclInt32, o.peer_proc, c->world, st));
            else NCCL_TRY(ncclRecv(recv_ints + (size_t)o.chunk * ipp, ipp, ncclInt32, o.peer_proc, c->world, st));
        }
        NCCL_TRY(ncclGroupEnd());
    }
    NCCL_TRY(ncclGroupStart());
    for (const smile_xop &o : ops) {
        if (o.kind == 0)
            NCCL_TRY(ncclSend((const char *)send_rows + (size_t)o.chunk * chunk, chunk, ncclUint8, o.peer_proc, c->world, st));
        else
            NCCL_TRY(ncclRecv((char *)recv_rows + (size_t)o.chunk * chunk, chunk, ncclUint8, o.peer_proc, c->world, st));
    }
    NCCL_TRY(ncclGroupEnd());
    return SMILE_OK;
}

extern "C" smile_status smile_all2all_inter(smile_ctx c, int32_t reverse, const void *send_rows, void *recv_rows,
                                            const int32_t *send_meta, int32_t *recv_meta, const int32_t *fwd_counts,
                                            void *stream) {
    return smile_all2all(c, 1, reverse, send_rows, recv_rows, send_meta, recv_meta, fwd_counts, stream);
}

extern "C" smile_status smile_all2all_intra(smile_ctx c, int32_t reverse, const void *send_rows, void *recv_rows,
                                            const int32_t *send_cnt, int32_t *recv_cnt, const int32_t *fwd_counts,
                                            void *stream) {
    return smile_all2all(c, 2, reverse, send_rows, recv_rows, send_cnt, recv_cnt, fwd_counts, stream);
}

// PEER inference with the output bound (smile_set_output) and the tcgen05 FFN: GEMM 2
// writes rows whose source rank is in this process straight to out (BILEVEL: a12 + a13;
// FLAT: the world reverse exchange + a13) -- both layers get the same fusion.
static bool out_direct_enabled(smile_ctx c) {
    if (c->xchg != SMILE_XCHG_PEER || !c->out_bound) return false;
    if (c->shape.topk > 1) return false;            // several experts write each token's output
    if (c->shape.dtype != SMILE_BF16 || c->shape.ffn_impl == SMILE_FFN_SIMT) return false;
    const char *e = getenv("SMILE_OUT_DIRECT");
    if (e && e[0] == '0') return false;
    e = getenv("SMILE_RET_DIRECT");
    return !(e && e[0] == '0');
}

static bool out_direct_possible(smile_ctx c) { return c->rtok1_valid && out_direct_enabled(c); }

// PEER + BILEVEL + tcgen05: GEMM 2 stores its rows into the intermediates' ret1 (the
// level-2 un-permute fused into the FFN); smile_combine(2) then has nothing left to do.
static void set_ret_direct(smile_ctx c, FfnArgs &f) {
    if (c->xchg != SMILE_XCHG_PEER || c->shape.mode != SMILE_BILEVEL) return;
    if (getenv("SMILE_RET_DIRECT") && getenv("SMILE_RET_DIRECT")[0] == '0') return;
    f.ret = c->peer;
    f.rrow = reinterpret_cast<const int32_t *>(static_cast<char *>(c->reg_ws) + c->peer.off_rrow);
}

extern "C" smile_status smile_expert_ffn(smile_ctx c, const void *X, const int32_t *counts, const void *W1t,
                                         const float *b1, const void *W2t, const float *b2, void *H_ws, void *Y,
                                         void *stream) {
    if (!c || !X || !counts || !W1t || !b1 || !W2t || !b2 || !H_ws || !Y) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    FfnArgs f{};
    f.X = X; f.counts = counts; f.W1t = W1t; f.b1 = b1; f.W2t = W2t; f.b2 = b2; f.H = H_ws; f.Y = Y;
    f.V = c->sz.V; f.S = c->sz.S; f.e = c->shape.e; f.Cseg = c->sz.Cseg; f.d = c->shape.d; f.d_ff = c->shape.d_ff;
    f.bf16 = c->shape.dtype == SMILE_BF16; f.num_sms = c->num_sms;
    int impl = c->shape.ffn_impl;
    if (impl == SMILE_FFN_AUTO) impl = f.bf16 ? SMILE_FFN_TCGEN05 : SMILE_FFN_SIMT;
    c->ret_direct = false;
    c->out_direct = false;
    if (impl == SMILE_FFN_TCGEN05) {
        if (!f.bf16) return SMILE_ENOTSUP;
        set_ret_direct(c, f);
        if (c->shape.mode == SMILE_FLAT && c->out_planned && c->xchg == SMILE_XCHG_PEER) {
            f.ret = c->peer;                 // bases / rank layout only (FLAT has no ret1)
            f.flat_out = 1;
        }
        if (f.ret.bases && c->out_planned) {
            f.out = c->out_bound; f.gate = c->d1_gate; f.T = c->shape.T; f.C1 = c->sz.C1; f.n = c->shape.n;
            f.rtok2 = reinterpret_cast<const int32_t *>(static_cast<char *>(c->reg_ws) + c->peer.off_rtok2);
        }
        cudaError_t e = launch_ffn_tcgen05(f, S(stream));
        if (e == cudaErrorNotSupported) return SMILE_ENOTSUP;
        c->ret_direct = f.ret.bases != nullptr && !f.flat_out;
        c->out_direct = f.out != nullptr;
        if (c->out_direct) c->l1_pending = true;
        return e == cudaSuccess ? post_launch() : SMILE_ECUDA;
    }
    if (!ffn_simt_supported(f.V * f.S * f.e, f.d, f.d_ff)) return SMILE_ENOTSUP;
    launch_ffn_simt(f, S(stream));
    return post_launch();
}

extern "C" smile_status smile_combine(smile_ctx c, int32_t level, const void *ret_rows, const smile_route *route,
                                      const int32_t *recv_meta, const int32_t *slot2, void *out, void *stream) {
    if (!c || !ret_rows || !out) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    const bool bf = c->shape.dtype == SMILE_BF16;
    if (level == 1) {
        if (!route) return SMILE_EINVAL;
        Combine1Args a{};
        a.back1 = ret_rows; a.route = *route; a.out = out; a.V = c->sz.V; a.T = c->shape.T; a.d = c->shape.d;
        a.K1 = c->sz.K1; a.C1 = c->sz.C1; a.bf16 = bf; a.nogate = 0; a.peer = peer_of(c);
        a.topk = c->shape.topk > 1 ? c->shape.topk : 1;
        if (c->l1_pending && out != c->out_bound) {
            // GEMM 2 wrote the in-process tokens to the bound output, not to ret1 / Y: a
            // combine into another buffer would read stale rows -- refused until the next
            // level-1 dispatch starts a new forward (sticky)
            return SMILE_EINVAL;
        }
        c->l1_pending = false;
        a.skip_direct = (a.peer.bases && c->out_direct) ? 1 : 0;
        c->out_direct = false;
        if (a.skip_direct && c->l1_zeroed && c->sz.V == c->sz.G) {
            // every token's intermediate and expert are in this process: GEMM 2 wrote the
            // kept tokens, the level-1 permute the dropped ones -- nothing left to move
            c->l1_zeroed = false;
            return SMILE_OK;
        }
        c->l1_zeroed = false;
        launch_combine1(a, S(stream));
        return post_launch();
    }
    if (level == 2) {
        if (c->shape.mode != SMILE_BILEVEL || !recv_meta || !slot2) return SMILE_EINVAL;
        const bool skip_local = c->xchg == SMILE_XCHG_PEER && c->ret_direct;
        c->ret_direct = false;
        // the expert FFN stored the rows of this process's experts in ret1 already; when
        // every node (m consecutive ranks) lies inside one process that is every row
        if (skip_local && (c->shape.nprocs == 1 || c->sz.V % c->shape.m == 0)) return SMILE_OK;
        Combine2Args a{};
        a.ret2 = ret_rows; a.recv_meta = recv_meta; a.slot2 = slot2; a.ret1 = out; a.V = c->sz.V;
        a.items = (int64_t)c->shape.n * c->sz.C1; a.rowbytes = (int64_t)c->shape.d * (bf ? 2 : 4);
        a.K2 = c->sz.K2; a.C2 = c->sz.C2; a.peer = peer_of(c); a.skip_local = skip_local ? 1 : 0;
        launch_combine2(a, S(stream));
        return post_launch();
    }
    return SMILE_EINVAL;
}

extern "C" smile_status smile_aux_loss(smile_ctx c, const smile_stats *stats, double alpha, double beta,
                                       double *loss, void *stream) {
    if (!c || !stats || !loss) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_EINVAL;
    cudaSetDevice(c->shape.device);
    launch_aux(*stats, alpha, beta, loss, c->sz.V, c->sz.K1, c->sz.K2, c->shape.T,
               c->shape.mode == SMILE_FLAT, S(stream));
    return post_launch();
}

static bool ffn_use_tc(smile_ctx c) {
    int impl = c->shape.ffn_impl;
    if (impl == SMILE_FFN_AUTO) impl = c->shape.dtype == SMILE_BF16 ? SMILE_FFN_TCGEN05 : SMILE_FFN_SIMT;
    return impl == SMILE_FFN_TCGEN05;
}

extern "C" smile_status smile_expert_ffn_train(smile_ctx c, const void *X, const int32_t *counts, const void *W1t,
                                               const float *b1, const void *W2t, const float *b2, void *A1_ws,
                                               void *H_ws, void *Y, void *stream) {
    if (!c || !X || !counts || !W1t || !b1 || !W2t || !b2 || !A1_ws || !H_ws || !Y) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    FfnArgs f{};
    f.X = X; f.counts = counts; f.W1t = W1t; f.b1 = b1; f.W2t = W2t; f.b2 = b2; f.H = H_ws; f.Y = Y;
    f.V = c->sz.V; f.S = c->sz.S; f.e = c->shape.e; f.Cseg = c->sz.Cseg; f.d = c->shape.d; f.d_ff = c->shape.d_ff;
    f.bf16 = c->shape.dtype == SMILE_BF16; f.num_sms = c->num_sms;
    const bool tc = ffn_use_tc(c);
    if (tc && !f.bf16) return SMILE_ENOTSUP;
    if (!tc && !ffn_simt_supported(f.V * f.S * f.e, f.d, f.d_ff)) return SMILE_ENOTSUP;
    c->ret_direct = false;
    c->out_direct = false;                   // training keeps ret1 (combine_bwd reads it)
    if (tc) set_ret_direct(c, f);
    cudaError_t e = launch_ffn_fwd_train(f, A1_ws, tc, S(stream));
    if (e == cudaErrorNotSupported) return SMILE_ENOTSUP;
    c->ret_direct = f.ret.bases != nullptr;
    return e == cudaSuccess ? post_launch() : SMILE_ECUDA;
}

extern "C" smile_status smile_combine_bwd(smile_ctx c, const void *gout, const void *back1, const float *logits,
                                          const smile_route *route, const smile_stats *stats, double alpha,
                                          double beta, double lam, void *dsend, float *dlogits, void *stream) {
    if (!c || !gout || !back1 || !logits || !route || !stats || !dsend || !dlogits) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    CombineBwdArgs a{};
    a.gout = gout; a.back1 = back1; a.logits = logits; a.route = *route; a.stats = *stats; a.dsend = dsend;
    a.dlogits = dlogits; a.V = c->sz.V; a.T = c->shape.T; a.d = c->shape.d; a.K1 = c->sz.K1; a.K2 = c->sz.K2;
    a.KW = c->sz.KW; a.C1 = c->sz.C1; a.alpha = alpha; a.beta = beta; a.lam = lam;
    a.flat = c->shape.mode == SMILE_FLAT; a.bf16 = c->shape.dtype == SMILE_BF16; a.peer = peer_of(c);
    a.topk = c->shape.topk > 1 ? c->shape.topk : 1;
    launch_combine_bwd(a, S(stream));
    return post_launch();
}

extern "C" smile_status smile_dispatch_grad(smile_ctx c, const void *drecv1, const int32_t *recv_meta,
                                            const int32_t *slot2, void *dsend2, void *stream) {
    if (!c || !drecv1 || !recv_meta || !slot2 || !dsend2) return SMILE_EINVAL;
    if (c->shape.mode != SMILE_BILEVEL) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    Dispatch2Args a{};
    a.recv1 = drecv1; a.recv_meta = recv_meta; a.slot2 = const_cast<int32_t *>(slot2); a.blk_off2 = nullptr;
    a.send2 = dsend2; a.V = c->sz.V; a.items = (int64_t)c->shape.n * c->sz.C1;
    a.rowbytes = (int64_t)c->shape.d * (c->shape.dtype == SMILE_BF16 ? 2 : 4); a.K2 = c->sz.K2; a.C2 = c->sz.C2;
    a.nblk = c->nblk2; a.peer = peer_of(c);
    launch_grad_dispatch2(a, S(stream));
    return post_launch();
}

extern "C" smile_status smile_expert_ffn_bwd(smile_ctx c, const void *X, const int32_t *counts, const void *A1,
                                             const void *H, const void *dY, const void *W1, const void *W2,
                                             void *dZ_ws, void *dX, float *dW1, float *db1, float *dW2, float *db2,
                                             void *stream) {
    if (!c || !X || !counts || !A1 || !H || !dY || !W1 || !W2 || !dZ_ws || !dX || !dW1 || !db1 || !dW2 || !db2)
        return SMILE_EINVAL;
    cudaSetDevice(c->shape.device);
    FfnBwdArgs b{};
    b.X = X; b.counts = counts; b.A1 = A1; b.H = H; b.dY = dY; b.W1 = W1; b.W2 = W2; b.dZ = dZ_ws; b.dX = dX;
    b.dW1 = dW1; b.db1 = db1; b.dW2 = dW2; b.db2 = db2; b.V = c->sz.V; b.S = c->sz.S; b.e = c->shape.e;
    b.Cseg = c->sz.Cseg; b.d = c->shape.d; b.d_ff = c->shape.d_ff; b.bf16 = c->shape.dtype == SMILE_BF16;
    b.num_sms = c->num_sms;
    b.colsum_ws = c->colsum_ws;
    const bool tc = ffn_use_tc(c);
    if (tc && !b.bf16) return SMILE_ENOTSUP;
    if (!ffn_simt_supported(b.V * b.S * b.e, b.d, b.d_ff)) return SMILE_ENOTSUP;
    cudaError_t e = launch_ffn_bwd(b, tc, S(stream));
    if (e == cudaErrorNotSupported) return SMILE_ENOTSUP;
    return e == cudaSuccess ? post_launch() : SMILE_ECUDA;
}

extern "C" smile_status smile_combine_grad(smile_ctx c, const void *ret_rows, const smile_route *route, void *dx,
                                           void *stream) {
    if (!c || !ret_rows || !route || !dx) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    Combine1Args a{};
    a.back1 = ret_rows; a.route = *route; a.out = dx; a.V = c->sz.V; a.T = c->shape.T; a.d = c->shape.d;
    a.K1 = c->sz.K1; a.C1 = c->sz.C1; a.bf16 = c->shape.dtype == SMILE_BF16; a.nogate = 1; a.peer = peer_of(c);
    a.topk = c->shape.topk > 1 ? c->shape.topk : 1;            // top-k: dx[t] = sum of the choices' rows
    launch_combine1(a, S(stream));
    return post_launch();
}

extern "C" smile_status smile_router_bwd(smile_ctx c, const void *x, const float *w_router, const float *dlogits,
                                         void *dx, float *dW, void *partial_ws, void *stream) {
    if (!c || !x || !w_router || !dlogits || !dx || !dW || !partial_ws) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c->shape.device);
    RouterBwdArgs a{};
    a.x = x; a.w = w_router; a.dlogits = dlogits; a.dx = dx; a.dW = dW; a.partial = (float *)partial_ws;
    a.rows = (int64_t)c->sz.V * c->shape.T; a.d = c->shape.d; a.KW = c->sz.KW; a.nchunk = 0;
    a.bf16 = c->shape.dtype == SMILE_BF16;
    launch_router_bwd(a, S(stream));
    return post_launch();
}

extern "C" smile_status smile_forward_ws(smile_ctx c, void *ws, smile_ws_view *view) {
    if (!c || !ws || !view) return SMILE_EINVAL;
    if (((uintptr_t)ws & 255) != 0) return SMILE_ESHAPE;
    ws_layout(&c->shape, &c->sz, nullptr, view, (char *)ws);
    return SMILE_OK;
}


extern "C" smile_status smile_set_fabric(smile_ctx c, const smile_fabric *f) {
    if (!c || !f) return SMILE_EINVAL;
    if (!(f->inter_gbps > 0.0)) {                       // disable
        c->fabric = smile_fabric{};
        return SMILE_OK;
    }
    if (!(f->inter_latency_us >= 0.0)) return SMILE_EINVAL;
    if (c->shape.nprocs != 1) return SMILE_ENOTSUP;     // an emulation of every rank on this GPU
    if (c->xchg == SMILE_XCHG_PEER) return SMILE_ENOTSUP;  // the emulated NICs carry the COPY exchange
    c->fabric = *f;
    return SMILE_OK;
}

extern "C" smile_status smile_set_output(smile_ctx c, void *out) {
    if (!c) return SMILE_EINVAL;
    c->out_bound = out;
    return SMILE_OK;
}

// The three stages of one forward (the order of smile_forward; SURVEY 8(f) row 2 runs
// them of consecutive chunks on two streams): a1-a8, a9, a10-a14.
static smile_status fwd_front(smile_ctx c, const smile_layer_io *io, const smile_ws_view &w, bool train, void *stream) {
    // gate then level-1 permute as two kernels: measured faster than the fused
    // smile_gate_dispatch_inter (C2: 0.166 vs 0.178 ms; C4: 0.77 vs 0.85 ms) -- the row moves
    // from the gate's epilogue warps reach less bandwidth than the dedicated movers
    STEP(smile_gate_inter(c, io->x, io->w_router, io->logits, (train && !io->logits) ? w.logits : nullptr, &w.route,
                          &w.stats, w.counts1, stream));
    STEP(smile_dispatch(c, 1, io->x, &w.route, nullptr, nullptr, w.send1, w.meta1, stream));
    if (c->shape.mode == SMILE_BILEVEL) {
        // the paper's "four sequential All2All operations"
        STEP(smile_all2all_inter(c, 0, w.send1, w.recv1, w.meta1, w.rmeta1, w.counts1, stream));
        STEP(smile_gate_intra(c, w.rmeta1, w.slot2, w.counts2, stream));
        STEP(smile_dispatch(c, 2, w.recv1, nullptr, w.rmeta1, w.slot2, w.send2, nullptr, stream));
        STEP(smile_all2all_intra(c, 0, w.send2, w.recv2, w.counts2, w.rcounts, w.counts2, stream));
    } else {
        STEP(smile_all2all(c, 0, 0, w.send1, w.recv1, w.counts1, w.rcounts, w.counts1, stream));
    }
    return SMILE_OK;
}

static smile_status fwd_ffn(smile_ctx c, const smile_layer_io *io, const smile_ws_view &w, bool train, void *stream) {
    void *X = c->shape.mode == SMILE_BILEVEL ? w.recv2 : w.recv1;
    if (train) return smile_expert_ffn_train(c, X, w.rcounts, io->W1t, io->b1, io->W2t, io->b2, w.A1, w.H, w.Y, stream);
    return smile_expert_ffn(c, X, w.rcounts, io->W1t, io->b1, io->W2t, io->b2, w.H, w.Y, stream);
}

static smile_status fwd_back(smile_ctx c, const smile_layer_io *io, const smile_ws_view &w, void *stream) {
    if (c->shape.mode == SMILE_BILEVEL) {
        STEP(smile_all2all_intra(c, 1, w.Y, w.ret2, nullptr, nullptr, w.counts2, stream));
        STEP(smile_combine(c, 2, w.ret2, nullptr, w.rmeta1, w.slot2, w.ret1, stream));
        STEP(smile_all2all_inter(c, 1, w.ret1, w.back1, nullptr, nullptr, w.counts1, stream));
    } else {
        STEP(smile_all2all(c, 0, 1, w.Y, w.back1, nullptr, nullptr, w.counts1, stream));
    }
    STEP(smile_combine(c, 1, w.back1, &w.route, nullptr, nullptr, io->out, stream));
    STEP(smile_aux_loss(c, &w.stats, io->alpha, io->beta, io->loss, stream));
    return SMILE_OK;
}

static smile_status fwd_check(smile_ctx c, const smile_layer_io *io) {
    if (!io->x || !io->out || !io->loss || !io->ws) return SMILE_EINVAL;
    if (!io->logits && !io->w_router) return SMILE_EINVAL;
    if (c->xchg == SMILE_XCHG_PEER && io->ws != c->reg_ws) return SMILE_ENOTSUP;
    return SMILE_OK;
}

extern "C" smile_status smile_forward(smile_ctx c, const smile_layer_io *io, void *stream) {
    if (!c || !io) return SMILE_EINVAL;
    if (c->shape.T == 0) return SMILE_OK;                 // no tokens: nothing to compute
    STEP(fwd_check(c, io));
    smile_ws_view w;
    STEP(smile_forward_ws(c, io->ws, &w));
    const bool train = io->train != 0;
    // inference binds io->out for this call (GEMM 2 may write in-process rows there)
    struct OutBinding {
        smile_ctx c; void *prev;
        ~OutBinding() { c->out_bound = prev; }
    } bind{c, c->out_bound};
    c->out_bound = train ? nullptr : io->out;
    STEP(fwd_front(c, io, w, train, stream));
    STEP(fwd_ffn(c, io, w, train, stream));
    STEP(fwd_back(c, io, w, stream));
    return SMILE_OK;
}

extern "C" smile_status smile_forward_chunked(smile_ctx const *ctxs, const smile_layer_io *ios, int32_t nchunks,
                                              void *stream, void *stream2) {
    if (!ctxs || !ios || nchunks < 1 || !stream2 || stream2 == stream) return SMILE_EINVAL;
    const smile_ctx c0 = ctxs[0];
    if (!c0) return SMILE_EINVAL;
    for (int k = 0; k < nchunks; ++k) {
        const smile_ctx c = ctxs[k];
        if (!c) return SMILE_EINVAL;
        for (int j = 0; j < k; ++j)
            if (ctxs[j] == c) return SMILE_EINVAL;                 // one context (and workspace) per chunk
        const smile_shape &a = c->shape, &b = c0->shape;
        if (a.n != b.n || a.m != b.m || a.e != b.e || a.mode != b.mode || a.dtype != b.dtype || a.d != b.d ||
            a.d_ff != b.d_ff || a.T != b.T || a.cf != b.cf || a.nprocs != b.nprocs || a.proc != b.proc ||
            a.device != b.device || a.ffn_impl != b.ffn_impl)
            return SMILE_ESHAPE;
        if (ios[k].train) return SMILE_ENOTSUP;                     // inference pipelining only
        if (c->shape.T > 0) STEP(fwd_check(c, &ios[k]));
    }
    if (c0->shape.T == 0) return SMILE_OK;
    cudaSetDevice(c0->shape.device);
    cudaStream_t s1 = S(stream), s2 = S(stream2);
    std::vector<smile_ws_view> w(nchunks);
    for (int k = 0; k < nchunks; ++k) STEP(smile_forward_ws(ctxs[k], ios[k].ws, &w[k]));
    // every chunk binds its own output for the GEMM 2 -> out fusion, restored on return
    struct Binds {
        smile_ctx const *c; int n; void *prev[64];
        ~Binds() { for (int k = 0; k < n && k < 64; ++k) c[k]->out_bound = prev[k]; }
    } binds{ctxs, 0, {}};
    if (nchunks > 64) return SMILE_ENOTSUP;
    for (int k = 0; k < nchunks; ++k) {
        binds.prev[k] = ctxs[k]->out_bound;
        ctxs[k]->out_bound = ios[k].out;
        binds.n = k + 1;
    }
    // stream 2 starts after the work already queued on stream 1
    CUDA_TRY(cudaEventRecord(ctxs[0]->ev_chunk_front, s1));
    CUDA_TRY(cudaStreamWaitEvent(s2, ctxs[0]->ev_chunk_front, 0));
    STEP(fwd_front(ctxs[0], &ios[0], w[0], false, stream));
    CUDA_TRY(cudaEventRecord(ctxs[0]->ev_chunk_front, s1));
    for (int k = 0; k < nchunks; ++k) {
        smile_ctx c = ctxs[k];
        // the FFN of chunk k (stream 2) overlaps the front of chunk k+1 and the back of k-1
        CUDA_TRY(cudaStreamWaitEvent(s2, c->ev_chunk_front, 0));
        STEP(fwd_ffn(c, &ios[k], w[k], false, stream2));
        CUDA_TRY(cudaEventRecord(c->ev_chunk_ffn, s2));
        if (k + 1 < nchunks) {
            STEP(fwd_front(ctxs[k + 1], &ios[k + 1], w[k + 1], false, stream));
            CUDA_TRY(cudaEventRecord(ctxs[k + 1]->ev_chunk_front, s1));
        }
        CUDA_TRY(cudaStreamWaitEvent(s1, c->ev_chunk_ffn, 0));
        STEP(fwd_back(c, &ios[k], w[k], stream));
    }
    return SMILE_OK;
}

extern "C" smile_status smile_forward_host_stream(smile_ctx c, const smile_layer_io *io, void *const *x_dev,
                                                  void *const *out_dev, int32_t nb, const void *const *host_x,
                                                  void *const *host_out, double *host_loss, void *stream) {
    if (!c || !io || !x_dev || !out_dev || !host_x || !host_out || !host_loss || nb < 0) return SMILE_EINVAL;
    if (io->logits || !x_dev[0] || !x_dev[1] || !out_dev[0] || !out_dev[1] || !io->loss) return SMILE_EINVAL;
    cudaSetDevice(c->shape.device);
    cudaStream_t st = S(stream);
    const size_t xb = (size_t)c->sz.V * c->shape.T * c->shape.d * (c->shape.dtype == SMILE_BF16 ? 2 : 4);
    const size_t lb = (size_t)c->sz.V * 8;
    // the copy streams start after the work already queued on the compute stream
    CUDA_TRY(cudaEventRecord(c->ev_d2h[0], st));
    CUDA_TRY(cudaStreamWaitEvent(c->s_h2d, c->ev_d2h[0], 0));
    CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->ev_d2h[0], 0));
    for (int b = 0; b < nb; ++b) {
        const int k = b & 1;
        // x_dev[k] is free once batch b-2's layer has read it
        if (b >= 2) CUDA_TRY(cudaStreamWaitEvent(c->s_h2d, c->ev_comp[k], 0));
        CUDA_TRY(cudaMemcpyAsync(x_dev[k], host_x[b], xb, cudaMemcpyHostToDevice, c->s_h2d));
        CUDA_TRY(cudaEventRecord(c->ev_h2d[k], c->s_h2d));
        // the layer: after its input landed and after out_dev[k]'s previous D2H
        CUDA_TRY(cudaStreamWaitEvent(st, c->ev_h2d[k], 0));
        if (b >= 2) CUDA_TRY(cudaStreamWaitEvent(st, c->ev_d2h[k], 0));
        smile_layer_io l = *io;
        l.x = x_dev[k];
        l.out = out_dev[k];
        STEP(smile_forward(c, &l, stream));
        CUDA_TRY(cudaMemcpyAsync(host_loss + (size_t)b * c->sz.V, io->loss, lb, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaEventRecord(c->ev_comp[k], st));
        CUDA_TRY(cudaStreamWaitEvent(c->s_d2h, c->ev_comp[k], 0));
        CUDA_TRY(cudaMemcpyAsync(host_out[b], out_dev[k], xb, cudaMemcpyDeviceToHost, c->s_d2h));
        CUDA_TRY(cudaEventRecord(c->ev_d2h[k], c->s_d2h));
    }
    CUDA_TRY(cudaStreamSynchronize(c->s_d2h));
    CUDA_TRY(cudaStreamSynchronize(st));
    return SMILE_OK;
}

extern "C" smile_status smile_backward(smile_ctx c, const smile_layer_io *io, const smile_grad_io *g, void *stream) {
    if (!c || !io || !g) return SMILE_EINVAL;
    if (c->shape.T == 0) {
        // the weight gradients are sums over no tokens
        if (!g->dW1 || !g->db1 || !g->dW2 || !g->db2) return SMILE_EINVAL;
        cudaSetDevice(c->shape.device);
        const size_t NEl = (size_t)c->sz.V * c->shape.e, d = c->shape.d, f = c->shape.d_ff;
        cudaStream_t st = S(stream);
        CUDA_TRY(cudaMemsetAsync(g->dW1, 0, NEl * d * f * 4, st));
        CUDA_TRY(cudaMemsetAsync(g->db1, 0, NEl * f * 4, st));
        CUDA_TRY(cudaMemsetAsync(g->dW2, 0, NEl * f * d * 4, st));
        CUDA_TRY(cudaMemsetAsync(g->db2, 0, NEl * d * 4, st));
        if (g->dW_router) CUDA_TRY(cudaMemsetAsync(g->dW_router, 0, (size_t)c->sz.KW * d * 4, st));
        return SMILE_OK;
    }
    if (!io->ws || !g->gout || !g->dx || !g->W1 || !g->W2 || !g->dW1 || !g->db1 || !g->dW2 ||
        !g->db2)
        return SMILE_EINVAL;
    if (io->w_router && !io->logits && !g->dW_router) return SMILE_EINVAL;
    const bool peer = c->xchg == SMILE_XCHG_PEER;
    if (peer && io->ws != c->reg_ws) return SMILE_ENOTSUP;
    // PEER: every exchange below is a barrier; the gradient rows are stored at / loaded
    // from their owners by combine_bwd, dispatch_grad, combine and combine_grad, and the
    // FFN backward writes dX over dY in the Y buffer (where the return path loads it)
    smile_ws_view w;
    STEP(smile_forward_ws(c, io->ws, &w));
    if (c->shape.T == 0) return SMILE_OK;
    const float *lg = io->logits ? io->logits : w.logits;
    // a16: gradient rows into the level-1 send layout (send1 is free after the forward)
    STEP(smile_combine_bwd(c, g->gout, w.back1, lg, &w.route, &w.stats, io->alpha, io->beta, g->lam, w.send1,
                           w.dlogits, stream));
    if (c->shape.mode == SMILE_BILEVEL) {
        STEP(smile_all2all_inter(c, 0, w.send1, w.recv1, nullptr, nullptr, w.counts1, stream));
        STEP(smile_dispatch_grad(c, w.recv1, w.rmeta1, w.slot2, w.send2, stream));
        // dY lands in the Y buffer (X = recv2 is still needed for dW1)
        STEP(smile_all2all_intra(c, 0, w.send2, w.Y, nullptr, nullptr, w.counts2, stream));
        STEP(smile_expert_ffn_bwd(c, w.recv2, w.rcounts, w.A1, w.H, w.Y, g->W1, g->W2, w.A1, peer ? w.Y : w.send2,
                                  g->dW1, g->db1, g->dW2, g->db2, stream));
        // a18: dX back along the return route
        STEP(smile_all2all_intra(c, 1, w.send2, w.ret2, nullptr, nullptr, w.counts2, stream));
        STEP(smile_combine(c, 2, w.ret2, nullptr, w.rmeta1, w.slot2, w.ret1, stream));
        STEP(smile_all2all_inter(c, 1, w.ret1, w.back1, nullptr, nullptr, w.counts1, stream));
    } else {
        STEP(smile_all2all(c, 0, 0, w.send1, w.Y, nullptr, nullptr, w.counts1, stream));
        STEP(smile_expert_ffn_bwd(c, w.recv1, w.rcounts, w.A1, w.H, w.Y, g->W1, g->W2, w.A1, peer ? w.Y : w.send1,
                                  g->dW1, g->db1, g->dW2, g->db2, stream));
        STEP(smile_all2all(c, 0, 1, w.send1, w.back1, nullptr, nullptr, w.counts1, stream));
    }
    STEP(smile_combine_grad(c, w.back1, &w.route, g->dx, stream));
    if (io->w_router && !io->logits)
        STEP(smile_router_bwd(c, io->x, io->w_router, w.dlogits, g->dx, g->dW_router, w.rpartial, stream));
    return SMILE_OK;
}

extern "C" smile_status smile_forward_host(smile_ctx c, const smile_layer_io *io, const void *host_x,
                                           const float *host_logits, void *host_out, double *host_loss, void *stream) {
    if (!c || !io || !host_x || !host_out || !host_loss) return SMILE_EINVAL;
    if (host_logits && !io->logits) return SMILE_EINVAL;
    cudaSetDevice(c->shape.device);
    cudaStream_t st = S(stream);
    const size_t xb = (size_t)c->sz.V * c->shape.T * c->shape.d * (c->shape.dtype == SMILE_BF16 ? 2 : 4);
    CUDA_TRY(cudaMemcpyAsync((void *)io->x, host_x, xb, cudaMemcpyHostToDevice, st));
    if (host_logits)
        CUDA_TRY(cudaMemcpyAsync((void *)io->logits, host_logits, (size_t)c->sz.V * c->shape.T * c->sz.KW * 4,
                                 cudaMemcpyHostToDevice, st));
    STEP(smile_forward(c, io, stream));
    CUDA_TRY(cudaMemcpyAsync(host_out, io->out, xb, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(host_loss, io->loss, (size_t)c->sz.V * 8, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return SMILE_OK;
}
