// TRPL+K engine: context creation (CSR -> SELL-32, halo plan, NCCL), Algorithm 1 driven on the
// device with one CUDA graph per outer cycle, and the C ABI of include/trplk.h /
// include/trplk_kernels.h.
//
// Host control flow mirrors Algorithm 1 with readings R1-R20;
// all vector work runs in the kernels of kernels.cu.  One host synchronisation per cycle
// (the soft-locking decision of steps 12-14 needs ||r_t||).
#include <cxxabi.h>
#include <nccl.h>

#include "comm.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "trplk.h"
#include "trplk_internal.cuh"
#include "trplk_kernels.h"

using namespace trplk;

namespace {

struct LogRec {
    int t;
    int64_t mv;
    double theta_t, res;
    int k, nprev;
    std::vector<double> thetas;
};

struct GraphRec {
    cudaGraphExec_t exec;
    double bytes;      // algorithmic bytes of one replay
    int64_t launches;  // kernels of one replay
};

struct Sizes {  // per-solve parameters that shape the captured graphs
    int p, q, l, ph, m;
    int prec;  // trplk_options.precond (0 Jacobi, 1 M = I)
    int blk;   // trplk_options.block (<= 1: Algorithm 1)
    bool operator<(const Sizes& o) const {
        return std::tie(p, q, l, ph, m, prec, blk) < std::tie(o.p, o.q, o.l, o.ph, o.m, o.prec, o.blk);
    }
    bool operator==(const Sizes& o) const { return !(*this < o) && !(o < *this); }
};

}  // namespace

struct trplk_ctx {
    int64_t n_global = 0, n_loc = 0, row_begin = 0, row_end = 0, n_ghost = 0, ld = 0;
    int rank = 0, nranks = 1;
    cudaStream_t stream = nullptr;       // internal non-blocking work stream (capturable)
    cudaStream_t user_stream = nullptr;  // the caller's stream; ordered with `stream` by events
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    trplk_allocator alloc{};
    bool has_alloc = false;
    std::vector<std::pair<void*, size_t>> allocs;
    bool hasB = false;
    double sigma = 0.0, mfloor = 0.0, normF = 0.0, amax = 0.0;
    double mfloor_solve = 0.0;  // the value kernels get: mfloor, or -1 for M = I (options.precond = 1)
    int pmode = 0;              // options.precond of the solve (2: per-cycle shifted Jacobi)
    Sell A, B;
    int64_t sellA_bytes = 0, sellB_bytes = 0, nnzA = 0, nnzB = 0;
    int64_t sellA_bytes_dc = 0;  // A's bytes as read by the DIA-C kernels (kern_reads_diac)
    // halo plan (nranks > 1): per peer, recv range in the ghost tail and send rows
    std::vector<int> peers;
    std::vector<int64_t> recv_off, recv_cnt, send_cnt, send_start;
    std::vector<int*> send_idx;
    double* sendbuf = nullptr;
    Comm* cm = nullptr;    // rank exchanges (NCCL, or the in-process loopback hub)
    int force3 = 0;        // debug: force the third CGS pass (trplk_set_debug / options.debug_checks & 2)
    int grid_on = -1;      // grid-wide inner loop: -1 = TRPLK_GRID env, else trplk_set_debug bit 1
    bool loopback = false;  // loopback hub / host callbacks: eager launches (exchanges are host rendezvous)
    // solve buffers
    int q_alloc = 0, ph_alloc = 0;
    double* U[2] = {nullptr, nullptr};
    double *w = nullptr, *w1 = nullptr, *w2 = nullptr, *u = nullptr, *u2 = nullptr, *xk = nullptr;
    double *T = nullptr, *Yg = nullptr, *part = nullptr, *gpart = nullptr, *red_local = nullptr, *red_all = nullptr;
    // block +K (block.cuh): control, the block being orthogonalised, the accepted vectors, reductions
    BlkCtl* blk = nullptr;
    double *wblk = nullptr, *xkb = nullptr, *sblk = nullptr, *bpart = nullptr, *bgpart = nullptr, *bred_local = nullptr,
           *bred_all = nullptr;
    unsigned* bcounter = nullptr;
    int blk_cols = 0;  // columns of wblk / xkb
    // IC(0) (options.precond = 3): factor, forward-solve scratch, chunk flags
    double *icL = nullptr, *ictmp = nullptr;
    int* icflags = nullptr;
    Ic0Args ic{};
    double* gridpart = nullptr;
    unsigned* rcnt = nullptr;  // fused K3 + K1 (fused.cuh): per-round completion counters
    int64_t rcnt_cap = 0;
    bool prof_fused = false;   // the live profile's slots are [K3 + K1 fused, K2, -]
    bool fuse_on = false;      // TRPLK_FUSE=1 at create: K3 + next K1 fused (fused.cuh)
    bool kplus_xd = true;      // +K first-pass dots on the preceding K1 (TRPLK_KPLUS_XD=0 at create: off)
    // halo overlap (nranks > 1, DIA, B = I): the exchange on hstream while K1 runs the interior
    // rows [hb0, hb1), then the boundary rows; TRPLK_HALO_OVERLAP=0 at create: exchange first
    cudaStream_t hstream = nullptr;
    cudaEvent_t hev_fork = nullptr, hev_done = nullptr;
    int64_t hb0 = 0, hb1 = 0;
    bool hov = false;
    unsigned long long* gtrace = nullptr;  // TRPLK_GRID_TRACE: per-step phase timestamps
    cudaEvent_t ctev[2] = {nullptr, nullptr};  // TRPLK_CYCLE_TRACE
    double ctrace_busy = 0.0;
    int ctrace_n = 0;  // all-reduce partials of the grid-wide inner loop (2 x GRID_MAXCTA x GRID_NVP)
    double* Wtmp = nullptr;
    unsigned* counter = nullptr;
    Ctl* ctl = nullptr;
    Ctl* ctl_h = nullptr;
    std::string err;
    std::vector<LogRec> log;
    int log_ph = 0;
    Sizes gsizes{0, 0, 0, 0, 0};
    std::map<uint64_t, GraphRec> graphs;
    // counters of the running solve
    int64_t a_mv = 0, b_mv = 0, prec = 0, inner = 0, verify = 0, draws = 0;
    double model_bytes = 0.0;
    int64_t launches = 0;
    // live profile of the middle inner step (trplk_profile)
    bool prof_on = false;
    cudaEvent_t pev[4] = {nullptr, nullptr, nullptr, nullptr};
    double prof_ms[3] = {0, 0, 0}, prof_bytes[3] = {0, 0, 0};
    int64_t prof_count = 0;
    const void* prof_kern[3] = {nullptr, nullptr, nullptr};  // kernels of the profiled groups K1, K2, K3
    // cycle phases (profile on): seed CGS2, inner steps, +K, Rayleigh-Ritz eig, rotation, residual
    cudaEvent_t phev[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    double phase_ms[6] = {0, 0, 0, 0, 0, 0};
    int64_t phase_count = 0;
    int prof_k = 0;
    // PL+1 quasi-optimality diagnostic (P7): capacity (0 = off) and the last solve's log
    int qopt_cap = 0;
    std::vector<double> qopt_star, qopt_rho;
    double qopt_last = 0.0;  // the solve's last rho_k (the default lambda1 of trplk_pl1_get_qopt)
    std::vector<int> qopt_dim;
};

namespace {

#define CK(call)                                                                       \
    do {                                                                               \
        cudaError_t e_ = (call);                                                       \
        if (e_ != cudaSuccess) {                                                       \
            ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);             \
            return TRPLK_ECUDA;                                                        \
        }                                                                              \
    } while (0)

#define NK(call)                                                                       \
    do {                                                                               \
        ncclResult_t r_ = (call);                                                      \
        if (r_ != ncclSuccess) {                                                       \
            ctx->err = std::string(#call) + ": " + ncclGetErrorString(r_);             \
            return TRPLK_ENCCL;                                                        \
        }                                                                              \
    } while (0)

#define CM(call)                                                                       \
    do {                                                                               \
        if (!(call)) {                                                                 \
            ctx->err = std::string(#call) + ": " + ctx->cm->what();                    \
            return TRPLK_ENCCL;                                                        \
        }                                                                              \
    } while (0)

#define ST(call)                                                                       \
    do {                                                                               \
        trplk_status s_ = (call);                                                      \
        if (s_ != TRPLK_OK) return s_;                                                 \
    } while (0)

// Order the internal work stream after / before the caller's stream.
void enter_stream(trplk_ctx* ctx) {
    if (ctx->user_stream != ctx->stream) {
        cudaEventRecord(ctx->ev_in, ctx->user_stream);
        cudaStreamWaitEvent(ctx->stream, ctx->ev_in, 0);
    }
}

void leave_stream(trplk_ctx* ctx) {
    if (ctx->user_stream != ctx->stream) {
        cudaEventRecord(ctx->ev_out, ctx->stream);
        cudaStreamWaitEvent(ctx->user_stream, ctx->ev_out, 0);
    }
}

// Device memory without a caller allocator comes from a process-wide stream-ordered pool per
// device (cudaMallocFromPoolAsync on the work stream): a create/solve/destroy sequence -- the
// e2e path -- re-uses the previous context's memory instead of paying cudaMalloc/cudaFree each
// time.  trplk_destroy trims the pool back to POOL_KEEP bytes (TRPLK_POOL_KEEP_MB, default 8 GB)
// so a finished large solve does not keep its footprint reserved.
static std::mutex g_pool_mu;
static std::map<int, cudaMemPool_t> g_pools;

static cudaMemPool_t device_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    auto it = g_pools.find(dev);
    if (it != g_pools.end()) return it->second;
    cudaMemPoolProps pr{};
    pr.allocType = cudaMemAllocationTypePinned;
    pr.handleTypes = cudaMemHandleTypeNone;
    pr.location.type = cudaMemLocationTypeDevice;
    pr.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &pr) != cudaSuccess) return nullptr;
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    g_pools[dev] = pool;
    return pool;
}

static void trim_pool() {
    cudaMemPool_t pool = device_pool();
    if (!pool) return;
    const char* e = getenv("TRPLK_POOL_KEEP_MB");
    const size_t keep = (e ? (size_t)atoll(e) : (size_t)8192) << 20;
    cudaMemPoolTrimTo(pool, keep);
}

// Pinned host blocks for the Ctl mirror, recycled across contexts (cudaMallocHost costs ~ms).
static std::vector<Ctl*> g_ctl_free;

static Ctl* ctl_host_alloc() {
    {
        std::lock_guard<std::mutex> lk(g_pool_mu);
        if (!g_ctl_free.empty()) {
            Ctl* c = g_ctl_free.back();
            g_ctl_free.pop_back();
            return c;
        }
    }
    Ctl* c = nullptr;
    if (cudaMallocHost(&c, sizeof(Ctl)) != cudaSuccess) return nullptr;
    return c;
}

static void ctl_host_free(Ctl* c) {
    if (!c) return;
    std::lock_guard<std::mutex> lk(g_pool_mu);
    g_ctl_free.push_back(c);
}

trplk_status dev_alloc(trplk_ctx* ctx, void** p, size_t bytes) {
    if (bytes == 0) bytes = 8;
    bytes = (bytes + 255) & ~(size_t)255;
    void* q = nullptr;
    if (ctx->has_alloc) {
        q = ctx->alloc.alloc(bytes, ctx->alloc.user);
        if (!q) {
            ctx->err = "allocator returned NULL for " + std::to_string(bytes) + " bytes";
            return TRPLK_ENOMEM;
        }
    } else {
        cudaMemPool_t pool = device_pool();
        cudaError_t e = pool ? cudaMallocFromPoolAsync(&q, bytes, pool, ctx->stream) : cudaMalloc(&q, bytes);
        if (e != cudaSuccess) {
            ctx->err = std::string("device allocation: ") + cudaGetErrorString(e);
            return e == cudaErrorMemoryAllocation ? TRPLK_ENOMEM : TRPLK_ECUDA;
        }
    }
    ctx->allocs.push_back({q, bytes});
    *p = q;
    return TRPLK_OK;
}

static void dev_release(trplk_ctx* ctx, void* p) {
    if (ctx->has_alloc) ctx->alloc.free(p, ctx->alloc.user);
    else if (device_pool()) cudaFreeAsync(p, ctx->stream);
    else cudaFree(p);
}

void dev_free(trplk_ctx* ctx, void* p) {
    if (!p) return;
    for (size_t i = 0; i < ctx->allocs.size(); ++i)
        if (ctx->allocs[i].first == p) {
            dev_release(ctx, p);
            ctx->allocs.erase(ctx->allocs.begin() + (long)i);
            return;
        }
}

template <typename T>
trplk_status dalloc(trplk_ctx* ctx, T** p, size_t count) {
    return dev_alloc(ctx, reinterpret_cast<void**>(p), count * sizeof(T));
}

// ----------------------------------------------------------------- CSR -> SELL-32
struct HostSell {
    std::vector<int64_t> sptr;
    std::vector<int> col;
    std::vector<double> val;
};

// Local column id of global column c (owned rows first, then the sorted ghost list).
inline int64_t local_col(int64_t c, int64_t rb, int64_t re, int64_t n_loc, const std::vector<int64_t>& ghosts) {
    if (c >= rb && c < re) return c - rb;
    auto it = std::lower_bound(ghosts.begin(), ghosts.end(), c);
    return n_loc + (int64_t)(it - ghosts.begin());
}

trplk_status build_sell(trplk_ctx* ctx, const int64_t* rp, const int64_t* ci, const double* va,
                        const std::vector<int64_t>& ghosts, HostSell& hs) {
    const int64_t n = ctx->n_loc, rb = ctx->row_begin, re = ctx->row_end;
    const int64_t ns = (n + 31) / 32;
    const int64_t base = rp[0];
    hs.sptr.assign(ns + 1, 0);
    std::vector<int> width(ns, 0);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < ns; ++s) {
        int w = 1;
        for (int64_t r = s * 32; r < std::min(n, s * 32 + 32); ++r) {
            int64_t cnt = rp[r + 1] - rp[r];
            bool has_diag = false;
            for (int64_t p = rp[r] - base; p < rp[r + 1] - base; ++p)
                if (ci[p] == rb + r) has_diag = true;
            int wr = (int)(has_diag ? cnt : cnt + 1);
            w = std::max(w, wr);
        }
        width[s] = w;
    }
    for (int64_t s = 0; s < ns; ++s) hs.sptr[s + 1] = hs.sptr[s] + 32 * (int64_t)width[s];
    const int64_t tot = hs.sptr[ns];
    hs.col.assign(tot, 0);
    hs.val.assign(tot, 0.0);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < ns; ++s) {
        for (int lane = 0; lane < 32; ++lane) {
            const int64_t r = s * 32 + lane;
            const int64_t b = hs.sptr[s] + lane;
            if (r >= n) {
                for (int j = 0; j < width[s]; ++j) hs.col[b + 32 * j] = 0;
                continue;
            }
            hs.col[b] = (int)r;  // slot 0: diagonal (explicit zero if not stored)
            hs.val[b] = 0.0;
            int j = 1;
            for (int64_t p = rp[r] - base; p < rp[r + 1] - base; ++p) {
                if (ci[p] == rb + r) {
                    hs.val[b] += va[p];
                } else {
                    hs.col[b + 32 * j] = (int)local_col(ci[p], rb, re, n, ghosts);
                    hs.val[b + 32 * j] = va[p];
                    ++j;
                }
            }
            for (; j < width[s]; ++j) hs.col[b + 32 * j] = (int)r;  // padding: val 0
        }
    }
    return TRPLK_OK;
}

trplk_status upload_sell(trplk_ctx* ctx, const HostSell& hs, Sell& S, int64_t& bytes) {
    int64_t* sptr;
    int* col;
    double* val;
    ST(dalloc(ctx, &sptr, hs.sptr.size()));
    ST(dalloc(ctx, &col, hs.col.size()));
    ST(dalloc(ctx, &val, hs.val.size()));
    CK(cudaMemcpyAsync(sptr, hs.sptr.data(), hs.sptr.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(col, hs.col.data(), hs.col.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(val, hs.val.data(), hs.val.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    S.nrows = ctx->n_loc;
    S.nslices = (int64_t)hs.sptr.size() - 1;
    S.sptr = sptr;
    S.col = col;
    S.val = val;
    bytes = (int64_t)(hs.sptr.size() * 8 + hs.col.size() * 4 + hs.val.size() * 8);
    return TRPLK_OK;
}

// Sorted unique global column ids outside [rb, re) referenced by the local rows of A (and B).
std::vector<int64_t> find_ghosts(int64_t n_loc, int64_t rb, int64_t re, const int64_t* a_rp, const int64_t* a_ci,
                                 const int64_t* b_rp, const int64_t* b_ci) {
    std::vector<int64_t> ghosts;
    for (int m = 0; m < 2; ++m) {
        const int64_t* rp = m == 0 ? a_rp : b_rp;
        const int64_t* ci = m == 0 ? a_ci : b_ci;
        if (!rp) continue;
        const int64_t nnz = rp[n_loc] - rp[0];
        for (int64_t p = 0; p < nnz; ++p)
            if (ci[p] < rb || ci[p] >= re) ghosts.push_back(ci[p]);
    }
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    return ghosts;
}

// Owner rank of each ghost id given all ranks' [begin, end) row ranges (rank order).
std::vector<int> ghost_owners(const std::vector<int64_t>& ghosts, const int64_t* ranges, int nranks) {
    std::vector<int> own(ghosts.size(), 0);
    for (size_t gi = 0; gi < ghosts.size(); ++gi) {
        int owner = 0;
        while (owner < nranks - 1 && ghosts[gi] >= ranges[2 * owner + 1]) ++owner;
        own[gi] = owner;
    }
    return own;
}

// One parallel pass over a local CSR block (rows [rb, re) of the global matrix): validation,
// the out-of-slab column ids (ghosts), the distinct diagonal offsets col - row (stops counting
// past DIA_MAX) and, when values are given, the squared Frobenius norm and max |A_jj|.  The
// sums are per 4096-row block, combined in block order: independent of the thread count.
struct CsrScan {
    std::vector<int64_t> ghosts;  // unsorted, may repeat
    std::vector<int64_t> offs;    // sorted distinct offsets (meaningful when !too_many)
    bool too_many = false;
    double fro2 = 0.0, amax = 0.0;
};

trplk_status scan_csr(trplk_ctx* ctx, const char* name, const int64_t* rp, const int64_t* ci, const double* va,
                      CsrScan& out) {
    if (!rp || !ci) {
        ctx->err = std::string(name) + ": NULL CSR array";
        return TRPLK_EINVAL;
    }
    const int64_t n = ctx->n_loc, rb = ctx->row_begin, re = ctx->row_end, ng = ctx->n_global, base = rp[0];
    constexpr int64_t BLK = 4096;
    const int64_t nb = (n + BLK - 1) / BLK;
    std::vector<double> bf((size_t)nb, 0.0), ba((size_t)nb, 0.0);
    std::vector<int64_t> bad((size_t)nb, -1);
    std::vector<int> badk((size_t)nb, 0);
#pragma omp parallel
    {
        std::vector<int64_t> gl, ol;
        bool over = false;
#pragma omp for schedule(static)
        for (int64_t b = 0; b < nb; ++b) {
            double f = 0.0, a = 0.0;
            const int64_t r1 = std::min(n, (b + 1) * BLK);
            for (int64_t r = b * BLK; r < r1 && bad[b] < 0; ++r) {
                if (rp[r + 1] < rp[r]) {
                    bad[b] = r, badk[b] = 1;
                    break;
                }
                int64_t prev = -1;
                size_t hint = 0;
                for (int64_t p = rp[r] - base; p < rp[r + 1] - base; ++p) {
                    const int64_t c = ci[p];
                    if (c < 0 || c >= ng) {
                        bad[b] = r, badk[b] = 2;
                        break;
                    }
                    if (c <= prev) {
                        bad[b] = r, badk[b] = 3;
                        break;
                    }
                    prev = c;
                    if (va) {
                        f += va[p] * va[p];
                        if (c == rb + r) a = std::max(a, std::fabs(va[p]));
                    }
                    if (c < rb || c >= re) gl.push_back(c);
                    if (!over) {
                        const int64_t off = c - (rb + r);
                        // offsets of consecutive entries of a row come in the same order row to row
                        if (hint < ol.size() && ol[hint] == off) {
                            ++hint;
                        } else {
                            auto it = std::find(ol.begin(), ol.end(), off);
                            if (it == ol.end()) {
                                ol.push_back(off);
                                hint = ol.size();
                                over = ol.size() > (size_t)DIA_MAX;
                            } else {
                                hint = (size_t)(it - ol.begin()) + 1;
                            }
                        }
                    }
                }
            }
            bf[b] = f;
            ba[b] = a;
        }
#pragma omp critical
        {
            out.ghosts.insert(out.ghosts.end(), gl.begin(), gl.end());
            out.too_many |= over;
            for (int64_t o : ol)
                if (std::find(out.offs.begin(), out.offs.end(), o) == out.offs.end()) out.offs.push_back(o);
        }
    }
    for (int64_t b = 0; b < nb; ++b)
        if (bad[b] >= 0) {
            static const char* what[] = {"", "row pointer decreases at row ", "column id out of range in row ",
                                         "columns not strictly increasing in row "};
            ctx->err = std::string(name) + ": " + what[badk[b]] + std::to_string(bad[b]);
            return TRPLK_EINVAL;
        }
    for (int64_t b = 0; b < nb; ++b) {
        out.fro2 += bf[b];
        out.amax = std::max(out.amax, ba[b]);
    }
    if (out.offs.size() > (size_t)DIA_MAX) out.too_many = true;
    std::sort(out.offs.begin(), out.offs.end());
    return TRPLK_OK;
}

static bool host_pinned(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// DIA-C (trplk_internal.cuh, Sell): diagonals whose stored entries all share one bit pattern
// are read as one presence bit per row plus the constant, instead of 8 bytes per row.  One
// device scan of the value arrays (min / max stored bit pattern per diagonal) decides; the
// decoded values are bit-identical to the stored ones, so the arithmetic does not change.
// Decoded only by the thread-per-row and fused K1 (lean_k1.cuh, fused.cuh): the shared SpMV row
// (mat_row) and the other K1 kernels ran slower with the decode in them, even when it was not
// taken (profiles/r02_variants.md); they read the value arrays, which stay populated.
// TRPLK_DIAC=0 at create: no presence bits.
trplk_status dia_compress(trplk_ctx* ctx, Sell& S, int64_t& bytes) {
    const char* e = getenv("TRPLK_DIAC");
    if ((e && e[0] == '0') || S.nrows == 0) return TRPLK_OK;  // TRPLK_DIAC=0: off
    const int nd = S.ndiag < 8 ? S.ndiag : 8;
    double* tmp;
    ST(dalloc(ctx, &tmp, (size_t)2 * nd));
    unsigned long long* mm = reinterpret_cast<unsigned long long*>(tmp);
    std::vector<unsigned long long> h(2 * (size_t)nd);
    for (int d = 0; d < nd; ++d) {
        h[2 * d] = ~0ull;
        h[2 * d + 1] = 0ull;
    }
    CK(cudaMemcpyAsync(mm, h.data(), 16 * (size_t)nd, cudaMemcpyHostToDevice, ctx->stream));
    launch_dia_const_scan(S.dval, S.nrows, S.ldv, nd, mm, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h.data(), mm, 16 * (size_t)nd, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    dev_free(ctx, tmp);
    unsigned cm = 0;
    double cv[8] = {};
    for (int d = 0; d < nd; ++d) {
        if (h[2 * d] == h[2 * d + 1] || (h[2 * d] == ~0ull && h[2 * d + 1] == 0ull)) {  // one pattern, or none
            cm |= 1u << d;
            const unsigned long long b = h[2 * d] == ~0ull ? 0ull : h[2 * d];
            std::memcpy(&cv[d], &b, 8);
        }
    }
    if (cm == 0) return TRPLK_OK;
    unsigned char* pm;
    ST(dalloc(ctx, &pm, (size_t)S.ldv));
    launch_dia_pmask(S.dval, S.nrows, S.ldv, nd, cm, pm, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    S.cmask = cm;
    S.pmask = pm;
    for (int d = 0; d < 8; ++d) S.cv[d] = cv[d];
    // `bytes` stays the value arrays' (what every other kernel reads); the DIA-C kernels' count:
    ctx->sellA_bytes_dc = (&S == &ctx->A) ? (int64_t)(S.ndiag - __builtin_popcount(cm)) * S.nrows * 8 + S.nrows
                                          : ctx->sellA_bytes_dc;
    (void)bytes;
    return TRPLK_OK;
}

// DIA conversion (values only; column = row + offset computed in the kernel).  Used when the
// local rows hold at most DIA_MAX distinct offsets col - row (from scan_csr), the padded
// diagonals store at most 1.25x the entries, and the ghost columns are the two contiguous
// ranges just below and above the owned rows (z-slab partitions of stencils).  ok = false
// otherwise.  Pinned host CSR arrays are copied to the device and scattered there
// (launch_csr_to_dia); pageable ones are scattered on the host and copied.
trplk_status try_dia(trplk_ctx* ctx, const int64_t* rp, const int64_t* ci, const double* va,
                     const std::vector<int64_t>& ghosts, const CsrScan& sc, Sell& S, int64_t& bytes, bool& ok) {
    ok = false;
    const int64_t n = ctx->n_loc, rb = ctx->row_begin, re = ctx->row_end, base = rp[0];
    int64_t glo = 0;
    for (int64_t g : ghosts) glo += g < rb ? 1 : 0;
    const int64_t ghi = (int64_t)ghosts.size() - glo;
    if (glo > 0 && (ghosts[0] != rb - glo || ghosts[glo - 1] != rb - 1)) return TRPLK_OK;
    if (ghi > 0 && (ghosts[glo] != re || ghosts.back() != re + ghi - 1)) return TRPLK_OK;
    if (sc.too_many) return TRPLK_OK;
    std::vector<int64_t> offs = sc.offs;
    if (std::find(offs.begin(), offs.end(), (int64_t)0) == offs.end()) offs.push_back(0);
    if ((int)offs.size() > DIA_MAX) return TRPLK_OK;
    std::sort(offs.begin(), offs.end());
    const int nd = (int)offs.size();
    const int64_t nnz = rp[n] - base;
    if ((double)n * nd > 1.25 * (double)nnz + 64.0 * nd) return TRPLK_OK;
    for (int64_t o : offs)
        if (o > INT32_MAX || o < INT32_MIN) return TRPLK_OK;
    const int64_t ldv = ((n + 31) / 32) * 32;
    double* dd;
    ST(dalloc(ctx, &dd, (size_t)nd * ldv));
    S = Sell();
    for (int d = 0; d < nd; ++d) S.offs[d] = (int)offs[d];
    if (host_pinned(rp) && host_pinned(ci) && host_pinned(va)) {
        int64_t *rpd, *cid;
        double* vad;
        ST(dalloc(ctx, &rpd, (size_t)n + 1));
        ST(dalloc(ctx, &cid, (size_t)std::max<int64_t>(nnz, 1)));
        ST(dalloc(ctx, &vad, (size_t)std::max<int64_t>(nnz, 1)));
        CK(cudaMemcpyAsync(rpd, rp, 8 * ((size_t)n + 1), cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(cid, ci, 8 * (size_t)nnz, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemcpyAsync(vad, va, 8 * (size_t)nnz, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaMemsetAsync(dd, 0, 8 * (size_t)nd * ldv, ctx->stream));
        launch_csr_to_dia(rpd, cid, vad, n, rb, S.offs, nd, ldv, dd, ctx->stream);
        CK(cudaGetLastError());
        dev_free(ctx, rpd);
        dev_free(ctx, cid);
        dev_free(ctx, vad);
    } else {
        std::unique_ptr<double[]> dv(new double[(size_t)nd * ldv]);
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < ldv; ++r) {
            for (int d = 0; d < nd; ++d) dv[(size_t)d * ldv + r] = 0.0;
            if (r >= n) continue;
            for (int64_t p = rp[r] - base; p < rp[r + 1] - base; ++p) {
                const int64_t off = ci[p] - (rb + r);
                const int d = (int)(std::lower_bound(offs.begin(), offs.end(), off) - offs.begin());
                dv[(size_t)d * ldv + r] = va[p];
            }
        }
        CK(cudaMemcpyAsync(dd, dv.get(), 8 * (size_t)nd * ldv, cudaMemcpyHostToDevice, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
    }
    S.fmt = 1;
    S.nrows = n;
    S.nslices = (n + 31) / 32;
    S.ndiag = nd;
    S.ldv = ldv;
    S.glo = glo;
    S.nghost = (int64_t)ghosts.size();
    S.dval = dd;
    for (int d = 0; d < nd; ++d)
        if (offs[d] == 0) S.diag_slot = d;
    bytes = (int64_t)nd * n * 8;
    ok = true;
    return dia_compress(ctx, S, bytes);
}

// ----------------------------------------------------------------- halo exchange
trplk_status halo(trplk_ctx* ctx, const double* xconst, cudaStream_t hs = nullptr) {
    if (ctx->nranks == 1 || ctx->peers.empty()) return TRPLK_OK;
    cudaStream_t st = hs ? hs : ctx->stream;
    double* x = const_cast<double*>(xconst);
    int64_t off = 0;
    for (size_t i = 0; i < ctx->peers.size(); ++i) {
        if (ctx->send_cnt[i] > 0 && ctx->send_start[i] < 0) {
            launch_gather(x, ctx->send_idx[i], ctx->send_cnt[i], ctx->sendbuf + off, st);
        }
        off += ctx->send_cnt[i];
    }
    std::vector<Xfer> sends, recvs;
    off = 0;
    for (size_t i = 0; i < ctx->peers.size(); ++i) {
        const int pr = ctx->peers[i];
        if (ctx->recv_cnt[i] > 0) recvs.push_back({pr, x + ctx->n_loc + ctx->recv_off[i], (size_t)ctx->recv_cnt[i]});
        if (ctx->send_cnt[i] > 0) {
            double* src = ctx->send_start[i] >= 0 ? x + ctx->send_start[i] : ctx->sendbuf + off;
            sends.push_back({pr, src, (size_t)ctx->send_cnt[i]});
        }
        off += ctx->send_cnt[i];
    }
    CM(ctx->cm->sendrecv(sends, recvs, 8, st));
    return TRPLK_OK;
}

// ----------------------------------------------------------------- kernel wrappers
SdotsArgs sd_base(trplk_ctx* ctx) {
    SdotsArgs a{};
    a.nrows = ctx->n_loc;
    a.theta_idx = -1;
    a.tcol_fixed = -1;
    a.sigma = ctx->sigma;
    a.mfloor = ctx->mfloor_solve;
    a.pmode = ctx->pmode;
    a.ctl = ctx->ctl;
    a.T = ctx->T;
    a.ldT = QMAX;
    a.part = ctx->part;
    a.gpart = ctx->gpart;
    a.counter = ctx->counter;
    a.maxcta = MAXCTA;
    a.ldu = ctx->ld;
    a.x_ld = ctx->ld;
    return a;
}

UpdArgs up_base(trplk_ctx* ctx) {
    UpdArgs a{};
    a.nrows = ctx->n_loc;
    a.ldu = ctx->ld;
    a.x_ld = ctx->ld;
    a.ctl = ctx->ctl;
    a.part = ctx->part;
    a.gpart = ctx->gpart;
    a.counter = ctx->counter;
    a.maxcta = MAXCTA;
    a.dest_ld = ctx->ld;
    return a;
}

double vec_bytes(trplk_ctx* ctx) { return 8.0 * (double)ctx->n_loc; }

double mat_bytes(trplk_ctx* ctx, bool b) {
    return (double)(b ? ctx->sellB_bytes : ctx->sellA_bytes);
}

// kbytes_cols: nominal number of basis columns the launch reads (>= the device-side k); it
// selects the register-row template and feeds the byte model.
trplk_status run_sdots(trplk_ctx* ctx, SdotsArgs a, int kbytes_cols, bool count_bytes = true) {
    const int kmax = (a.set1 || a.set2) ? kmax_bucket(std::max(kbytes_cols, 1)) : 0;
    // algorithmic bytes of this launch (DESIGN.md byte model)
    double by = 0.0;
    if (a.A.nrows && a.out_mode != 4) by += mat_bytes(ctx, false) + vec_bytes(ctx);
    if (a.B.nrows) by += mat_bytes(ctx, true);
    if (!a.A.nrows) by += vec_bytes(ctx);
    if (a.out) by += vec_bytes(ctx);
    if (a.uout) by += vec_bytes(ctx);
    if (a.wext) by += vec_bytes(ctx);
    if (a.set2 == 4) by += vec_bytes(ctx);  // the external dot vector x2
    if (a.set1 || a.set2) by += vec_bytes(ctx) * kbytes_cols;
    if (count_bytes) ctx->model_bytes += by;
    ctx->launches += ctx->nranks > 1 ? 2 : 1;
    if (ctx->nranks > 1) {
        a.red_local = ctx->red_local;
        launch_sdots(a, kmax, ctx->stream);
        CM(ctx->cm->allgather(ctx->red_local, ctx->red_all, NV_MAX, 8, ctx->stream));
        launch_finalize_sdots_multi(a, ctx->red_all, ctx->nranks, NV_MAX, ctx->stream);
    } else {
        launch_sdots(a, kmax, ctx->stream);
    }
    if (count_bytes && a.A.nrows && a.out_mode != 4 && kern_reads_diac(g_last_kern))
        ctx->model_bytes -= (double)(ctx->sellA_bytes - ctx->sellA_bytes_dc);
    CK(cudaGetLastError());
    return TRPLK_OK;
}

// Inner-step K1 of a row slab with the halo exchange overlapped: the exchange of
// g's boundary rows runs on hstream while K1 covers the interior rows [hb0, hb1), which read no
// ghost; then K1 covers [0, hb0) and [hb1, n).  The three launches are partial slots of ONE
// deterministic grid reduction (fixed slot order), finished by the last launch's last CTA.
bool k1_overlap_ok(const trplk_ctx* ctx, const SdotsArgs& a, int k) {
    return ctx->hov && a.A.nrows && !a.B.nrows && a.out_mode <= 2 && a.set1 == 1 && a.norm2 == 0 && a.x_dyn == 0 &&
           kmax_bucket(std::max(k, 1)) <= 48;
}

trplk_status run_k1_overlap(trplk_ctx* ctx, SdotsArgs a, int k) {
    const int kmax = kmax_bucket(std::max(k, 1));
    CK(cudaEventRecord(ctx->hev_fork, ctx->stream));
    CK(cudaStreamWaitEvent(ctx->hstream, ctx->hev_fork, 0));
    const int64_t n = ctx->n_loc;
    const int64_t rr[3][2] = {{ctx->hb0, ctx->hb1}, {0, ctx->hb0}, {ctx->hb1, n}};
    int g[3], tot = 0;
    for (int i = 0; i < 3; ++i) {  // one tile pair per warp, 2 CTAs per SM at most
        const int64_t tiles = (rr[i][1] - rr[i][0] + 31) / 32;
        int64_t need = (tiles + 2 * WARPS - 1) / (2 * WARPS);
        const int64_t cap = 2 * 148;
        g[i] = (int)std::max<int64_t>(1, std::min(need, cap));
        tot += g[i];
    }
    ctx->model_bytes += mat_bytes(ctx, false) + vec_bytes(ctx) * (k + 2 + (a.out ? 1 : 0));
    ctx->launches += 5;
    a.red_local = ctx->red_local;
    a.cta_tot = tot;
    int off = 0;
    for (int i = 0; i < 3; ++i) {
        SdotsArgs b = a;
        b.row0 = rr[i][0];
        b.nrows = rr[i][1];
        b.cta_off = off;
        b.grid_force = g[i];
        off += g[i];
        if (i == 1) {  // boundary rows: after the exchange
            CK(cudaEventRecord(ctx->hev_done, ctx->hstream));
            CK(cudaStreamWaitEvent(ctx->stream, ctx->hev_done, 0));
        }
        launch_sdots(b, kmax, ctx->stream);
        CK(cudaGetLastError());
        if (i == 0) ST(halo(ctx, a.x, ctx->hstream));  // enqueued after the interior launch
    }
    CM(ctx->cm->allgather(ctx->red_local, ctx->red_all, NV_MAX, 8, ctx->stream));
    launch_finalize_sdots_multi(a, ctx->red_all, ctx->nranks, NV_MAX, ctx->stream);
    CK(cudaGetLastError());
    return TRPLK_OK;
}

trplk_status run_upd(trplk_ctx* ctx, UpdArgs a, int k_nominal) {
    const int kmax = kmax_bucket(std::max(k_nominal, 1));
    if (a.mode != 3) ctx->model_bytes += vec_bytes(ctx) * (k_nominal + 2);
    const bool dots = a.dots && (a.mode == 1 || a.mode == 2);
    ctx->launches += (ctx->nranks > 1 && dots) ? 2 : 1;
    if (ctx->nranks > 1 && dots) {
        a.red_local = ctx->red_local;
        launch_upd(a, kmax, ctx->stream);
        CM(ctx->cm->allgather(ctx->red_local, ctx->red_all, NV_MAX, 8, ctx->stream));
        launch_finalize_upd_multi(a, ctx->red_all, ctx->nranks, NV_MAX, ctx->stream);
    } else {
        launch_upd(a, kmax, ctx->stream);
    }
    CK(cudaGetLastError());
    return TRPLK_OK;
}

// Small-n latency path: one CTA runs the whole inner loop (small.cuh) when the local problem
// is a few rows per thread, one rank, B = I and q <= 24.  TRPLK_NO_SMALL=1 disables it.
bool small_path(const trplk_ctx* ctx, const Sizes& S) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TRPLK_NO_SMALL");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1 && ctx->nranks == 1 && !ctx->hasB && ctx->n_loc <= SMALL_NMAX && S.q <= 24 && S.prec != 3;
}

// Mid-size latency path: one cooperative grid-wide kernel runs all m steps (inner_grid.cuh) for
// one rank, B = I, q <= 32 and n above the single-CTA range.  Opt-in (TRPLK_GRID=1 or
// trplk_set_debug bit 1): at C2 it measured 40 us per inner step against ~37 us for the
// multi-kernel step, whose launches overlap in the graph (profiles/r01_variants.md).
bool grid_path(const trplk_ctx* ctx, const Sizes& S) {
    static int env = -1;
    if (env < 0) {
        const char* e = getenv("TRPLK_GRID");
        env = (e && e[0] == '1') ? 1 : 0;
    }
    const bool on = ctx->grid_on < 0 ? env == 1 : ctx->grid_on == 1;
    return on && !small_path(ctx, S) && ctx->nranks == 1 && !ctx->hasB && S.q <= 32 && ctx->gridpart != nullptr &&
           S.prec != 3;
}

// One rank and B = I: the FINAL kernel is launched cooperatively and runs a third pass itself
// (grid barrier), so the two gated pass-3 launches (~2.5 us each, normally no-ops) disappear
// from every CGS2.  TRPLK_NO_COOP3=1 keeps the gated launches.
// The debug switch changes the captured kernels' arguments: drop the cached graphs.
void set_force3(trplk_ctx* ctx, int v) {
    if (ctx->force3 == v) return;
    ctx->force3 = v;
    for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.second.exec);
    ctx->graphs.clear();
}

bool coop3(const trplk_ctx* ctx) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TRPLK_NO_COOP3");
        v = (e && e[0] == '1') ? 0 : 1;
    }
    return v == 1 && ctx->nranks == 1 && !ctx->hasB;
}

// profile events inside a cycle: external event nodes under stream capture, plain records when
// the cycle is issued eagerly (loopback / host-exchange contexts, use_graphs = 0)
static cudaError_t record_event(trplk_ctx* ctx, cudaEvent_t ev) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(ctx->stream, &cs);
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, ctx->stream, cudaEventRecordExternal)
                                               : cudaEventRecord(ev, ctx->stream);
}

// K3 of inner step j + K1 of step j+1 as one kernel (fused.cuh): one rank, B = I, a DIA matrix
// of <= 8 diagonals, Jacobi / none / shifted preconditioner, the multi-kernel inner step (not the
// latency paths).  Opt-in (TRPLK_FUSE=1, read at create); TRPLK_FUSE_SLACK = rounds of slack
// between a tile's stencil reach and its K1 (default 1).
bool fuse_path(const trplk_ctx* ctx, const Sizes& S) {
    return ctx->fuse_on && ctx->nranks == 1 && !ctx->hasB && ctx->A.fmt == 1 && ctx->A.ndiag <= 8 && ctx->rcnt &&
           S.prec != 3 && S.q <= 48 && !small_path(ctx, S) && !grid_path(ctx, S);
}

bool run_fused(trplk_ctx* ctx, const UpdArgs& u, const SdotsArgs& a, int kn, int k_next) {
    static int slack = -1;
    if (slack < 0) {
        const char* sl = getenv("TRPLK_FUSE_SLACK");
        slack = sl ? std::max(0, atoi(sl)) : 1;
    }
    if (u.dest2 || !u.dest_dyn || u.mode != 2) return false;
    FusedArgs f{};
    f.u = u;
    f.a = a;
    f.rcnt = ctx->rcnt;
    f.rcnt_cap = ctx->rcnt_cap;
    int maxoff = 0;
    for (int d = 0; d < ctx->A.ndiag; ++d) maxoff = std::max(maxoff, std::abs(ctx->A.offs[d]));
    if (!launch_fin_step1(f, kmax_bucket(std::max(k_next, 1)), maxoff, slack, ctx->stream)) return false;
    // bytes: FINAL (U(:, 1:kn), w', g) + the K1 without its U / g re-reads (L2): A, w
    ctx->model_bytes += vec_bytes(ctx) * (kn + 2) + (double)ctx->sellA_bytes_dc + (a.out ? vec_bytes(ctx) : 0.0);
    ctx->launches += 1;
    return true;
}

// CGS2 in the B-inner product (R3) of x against V = Ubase(:, 0:kv) (kv = -1: ctl->k), result
// normalised into Ubase(:, ctl->k) (dest_dyn) or `dest`, ctl->k += 1 on success.
struct CgsSpec {
    const double* x;
    int x_dyn = 0, x_off = 0;
    const double* V;
    int64_t ldv = 0;  // 0 => ctx->ld
    int kv;          // fixed width or -1 (ctl->k)
    int k_nominal;   // upper bound for the kernel bucket
    bool first_done; // B = I: h0 / N_IN2 already computed by the fused K1
    unsigned gate1 = 0;  // extra gate bits of the first-pass launch (F_XD0 << j: not yet done elsewhere)
    double* dest;
    int dest_dyn;
    double* dest2;
    unsigned gate, clear;
    int inc_k;
    cudaEvent_t mark_final = nullptr;  // profiling: recorded just before the FINAL update
    const SdotsArgs* fuse_next = nullptr;  // FINAL fused with this K1 of the next inner step (fused.cuh)
    int k_next = 0;                        // its nominal basis width
};

trplk_status cgs2(trplk_ctx* ctx, const CgsSpec& c) {
    const int kn = std::max(c.k_nominal, 1);
    const int64_t ldv = c.ldv > 0 ? c.ldv : ctx->ld;
    // pass 1 coefficients: h0 = V^T B x, N_IN2 = x^T B x
    if (!c.first_done) {
        SdotsArgs a = sd_base(ctx);
        a.x = c.x;
        a.x_dyn = c.x_dyn;
        a.x_off = c.x_off;
        if (ctx->hasB) {
            a.A = ctx->B;  // z = B x
            a.set1 = 1;
            a.norm1 = 2;   // x.z
            ST(halo(ctx, c.x));
        } else {
            a.set1 = 3;    // x
            a.norm1 = 3;   // x.x
        }
        a.U = c.V;
        a.ldu = ldv;
        a.k1 = c.kv;
        a.k_from_ctl = c.kv < 0;
        a.dest1 = D_H0 + 0;
        a.nslot1 = N_IN2;
        a.gate = c.gate | c.gate1;
        ST(run_sdots(ctx, a, kn, c.gate1 == 0));  // normally skipped when gated on F_XD0 << j
    }
    // pass 2: w1 = x - V h0 (+ B = I: h1 = V^T w1, N_1SQ)
    {
        UpdArgs u = up_base(ctx);
        u.x = c.x;
        u.x_dyn = c.x_dyn;
        u.x_off = c.x_off;
        u.U = c.V;
        u.ldu = ldv;
        u.kv = c.kv;
        u.hslot = 0;
        u.mode = ctx->hasB ? 0 : 1;
        u.dots = ctx->hasB ? 0 : 1;
        u.out = ctx->w1;
        u.hout = 1;
        u.gate = c.gate;
        ST(run_upd(ctx, u, kn));
        if (c.mark_final) ctx->prof_kern[1] = g_last_kern;
    }
    if (ctx->hasB) {
        SdotsArgs a = sd_base(ctx);
        ST(halo(ctx, ctx->w1));
        a.x = ctx->w1;
        a.A = ctx->B;
        a.set1 = 1;
        a.norm1 = 2;
        a.U = c.V;
        a.ldu = ldv;
        a.k1 = c.kv;
        a.k_from_ctl = c.kv < 0;
        a.dest1 = D_H0 + 1;
        a.nslot1 = N_1SQ;
        a.gate = c.gate;
        ST(run_sdots(ctx, a, kn));
    }
    // final: y = w1 - V h1, beta from Pythagoras; pass 3 into w2 if the norm dropped > 1/sqrt2
    if (c.mark_final) CK(record_event(ctx, c.mark_final));
    {
        UpdArgs u = up_base(ctx);
        u.x = ctx->w1;
        u.U = c.V;
        u.ldu = ldv;
        u.kv = c.kv;
        u.hslot = 1;
        u.mode = 2;
        u.dots = 0;
        u.out = ctx->w2;
        u.hout = 2;
        u.dest = c.dest;
        u.dest_dyn = c.dest_dyn;
        u.dest2 = c.dest2;
        u.inc_k = c.inc_k;
        u.gate = c.gate;
        u.clear_on_brk = c.clear;
        u.force3 = ctx->force3;
        u.coop = coop3(ctx);
        if (c.fuse_next && run_fused(ctx, u, *c.fuse_next, kn, c.k_next)) {
            if (c.mark_final) ctx->prof_kern[0] = g_last_kern;
            return TRPLK_OK;
        }
        ST(run_upd(ctx, u, kn));
        if (c.mark_final) ctx->prof_kern[2] = g_last_kern;
        if (u.coop) return TRPLK_OK;  // the third pass, when needed, ran inside the FINAL kernel
    }
    {  // third-pass dots h3 = V^T B w2, N_2SQ_EXP = w2^T B w2 (gated on ctl->pass3, normally a no-op)
        SdotsArgs a = sd_base(ctx);
        a.x = ctx->w2;
        if (ctx->hasB) {
            ST(halo(ctx, ctx->w2));
            a.A = ctx->B;
            a.set1 = 1;
            a.norm1 = 2;
        } else {
            a.set1 = 3;
            a.norm1 = 3;
        }
        a.U = c.V;
        a.ldu = ldv;
        a.k1 = c.kv;
        a.k_from_ctl = c.kv < 0;
        a.dest1 = D_H0 + 2;
        a.nslot1 = N_2SQ_EXP;
        a.gate = c.gate;
        a.gate_pass3 = 1;
        ST(run_sdots(ctx, a, kn, false));  // rare path, not in the byte model
    }
    {
        UpdArgs u = up_base(ctx);
        u.x = ctx->w2;
        u.U = c.V;
        u.ldu = ldv;
        u.kv = c.kv;
        u.hslot = 2;
        u.mode = 3;
        u.dest = c.dest;
        u.dest_dyn = c.dest_dyn;
        u.dest2 = c.dest2;
        u.inc_k = c.inc_k;
        u.gate = c.gate;
        u.clear_on_brk = c.clear;
        ST(run_upd(ctx, u, kn));
    }
    return TRPLK_OK;
}

// IC(0) (reading P2a): v <- (L L^T)^-1 v by the forward and the backward sync-free solve
trplk_status ic0_apply(trplk_ctx* ctx, double* v, unsigned gate) {
    Ic0Args f = ctx->ic;
    f.v = v;
    f.y = ctx->ictmp;
    f.trans = 0;
    f.ctl = ctx->ctl;
    f.gate = gate;
    launch_ic0_solve(f, ctx->stream);
    Ic0Args b = f;
    b.v = ctx->ictmp;
    b.y = v;
    b.trans = 1;
    launch_ic0_solve(b, ctx->stream);
    ctx->launches += 2;
    ctx->model_bytes += 2.0 * (8.0 * ctx->n_loc * (ctx->ic.nlow + 1) + 2 * vec_bytes(ctx));
    CK(cudaGetLastError());
    return TRPLK_OK;
}

// the IC(0) factor of A - sigma I for this solve (buffers on first use)
trplk_status ic0_setup(trplk_ctx* ctx) {
    if (ctx->A.fmt != 1 || ctx->hasB || ctx->nranks > 1) {
        ctx->err = "options.precond = 3 (IC(0)): DIA matrix, B = I and one rank on the device";
        return TRPLK_EINVAL;
    }
    Ic0Args& a = ctx->ic;
    a = Ic0Args{};
    a.A = ctx->A;
    a.sigma = ctx->sigma;
    a.floor = ctx->mfloor;
    a.n = ctx->n_loc;
    a.ldl = ctx->ld;
    int lo[DIA_MAX], ls[DIA_MAX], nl = 0;
    for (int d = 0; d < ctx->A.ndiag; ++d)
        if (ctx->A.offs[d] < 0) {
            lo[nl] = ctx->A.offs[d];
            ls[nl] = d;
            ++nl;
        }
    for (int x = 1; x < nl; ++x)  // ascending offsets (the oracle's column order)
        for (int y = x; y > 0 && lo[y - 1] > lo[y]; --y) {
            std::swap(lo[y - 1], lo[y]);
            std::swap(ls[y - 1], ls[y]);
        }
    a.nlow = nl;
    for (int d = 0; d < nl; ++d) {
        a.loff[d] = lo[d];
        a.lslot[d] = ls[d];
        for (int b = 0; b < DIA_MAX; ++b) a.pair[d][b] = -1;
        for (int b = 0; b < d; ++b)
            for (int e2 = 0; e2 < nl; ++e2)
                if (lo[e2] == lo[b] - lo[d]) a.pair[d][b] = e2;
    }
    if (!ctx->icL) {
        ST(dalloc(ctx, &ctx->icL, (size_t)ctx->ld * (DIA_MAX + 1)));
        ST(dalloc(ctx, &ctx->ictmp, (size_t)ctx->ld));
        ST(dalloc(ctx, &ctx->icflags, (size_t)(ctx->n_loc + 31) / 32 + 8));
    }
    a.L = ctx->icL;
    a.flags = ctx->icflags;
    a.ctl = nullptr;
    launch_ic0_factor(a, ctx->stream);
    ctx->launches += 1;
    CK(cudaGetLastError());
    return TRPLK_OK;
}

// r = A x - theta B x, u = M r, N_RES2 = ||r||^2  (Alg.1 steps 12/15)
trplk_status residual(trplk_ctx* ctx, const double* x, int x_dyn, int theta_idx, double* uout, unsigned gate) {
    if (x_dyn == 0) ST(halo(ctx, x));
    SdotsArgs a = sd_base(ctx);
    a.A = ctx->A;
    if (ctx->hasB) a.B = ctx->B;
    a.x = x;
    a.x_dyn = x_dyn;
    a.out_mode = 3;
    a.uout = uout;
    a.norm1 = 1;
    a.nslot1 = N_RES2;
    a.theta_idx = theta_idx;
    a.gate = gate;
    ST(run_sdots(ctx, a, 0));
    if (ctx->pmode == 3 && uout) ST(ic0_apply(ctx, uout, gate));  // u = (L L^T)^-1 r
    return TRPLK_OK;
}

trplk_status ensure_block_buffers(trplk_ctx* ctx, int c) {
    if (ctx->blk_cols >= c) return TRPLK_OK;
    dev_free(ctx, ctx->wblk);
    dev_free(ctx, ctx->xkb);
    dev_free(ctx, ctx->sblk);
    ctx->wblk = ctx->xkb = ctx->sblk = nullptr;
    const size_t ld = (size_t)ctx->ld;
    ST(dalloc(ctx, &ctx->wblk, ld * c));
    ST(dalloc(ctx, &ctx->xkb, ld * c));
    ST(dalloc(ctx, &ctx->sblk, ld * c));
    CK(cudaMemsetAsync(ctx->wblk, 0, ld * c * 8, ctx->stream));
    CK(cudaMemsetAsync(ctx->xkb, 0, ld * c * 8, ctx->stream));
    CK(cudaMemsetAsync(ctx->sblk, 0, ld * c * 8, ctx->stream));
    ctx->blk_cols = c;
    for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.second.exec);
    ctx->graphs.clear();
    return TRPLK_OK;
}

trplk_status ensure_buffers(trplk_ctx* ctx, int q, int ph) {
    if (ctx->q_alloc >= q && ctx->ph_alloc >= ph) return TRPLK_OK;
    // release previous solve buffers
    for (double** b : {&ctx->U[0], &ctx->U[1], &ctx->Wtmp}) {
        dev_free(ctx, *b);
        *b = nullptr;
    }
    const size_t ld = (size_t)ctx->ld;
    ST(dalloc(ctx, &ctx->U[0], ld * q));
    ST(dalloc(ctx, &ctx->U[1], ld * q));
    ST(dalloc(ctx, &ctx->Wtmp, ld * ph));
    CK(cudaMemsetAsync(ctx->U[0], 0, ld * q * 8, ctx->stream));
    CK(cudaMemsetAsync(ctx->U[1], 0, ld * q * 8, ctx->stream));
    ctx->q_alloc = q;
    ctx->ph_alloc = ph;
    for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.second.exec);
    ctx->graphs.clear();
    return TRPLK_OK;
}

trplk_status ctl_push(trplk_ctx* ctx) {
    CK(cudaMemcpyAsync(ctx->ctl, ctx->ctl_h, offsetof(Ctl, k_rr), cudaMemcpyHostToDevice, ctx->stream));
    return TRPLK_OK;
}

trplk_status ctl_pull(trplk_ctx* ctx) {
    CK(cudaMemcpyAsync(ctx->ctl_h, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TRPLK_OK;
}

// One block-kernel launch (block.cuh); several ranks: local sums, allgather, rank-ordered finalize.
trplk_status run_block(trplk_ctx* ctx, BlkArgs a, int kmax, double bytes) {
    a.part = ctx->bpart;
    a.gpart = ctx->bgpart;
    a.counter = ctx->bcounter;
    a.maxcta = MAXCTA;
    a.ctl = ctx->ctl;
    ctx->model_bytes += bytes;
    ctx->launches += ctx->nranks > 1 ? 2 : 1;
    if (ctx->nranks > 1) {
        a.red_local = ctx->bred_local;
        if (!launch_block(a, kmax, ctx->stream)) {
            ctx->err = "block kernel: unsupported width";
            return TRPLK_EINVAL;
        }
        CM(ctx->cm->allgather(ctx->bred_local, ctx->bred_all, BLK_NV, 8, ctx->stream));
        launch_blk_finalize_multi(a, ctx->bred_all, ctx->nranks, BLK_NV, ctx->stream);
    } else if (!launch_block(a, kmax, ctx->stream)) {
        ctx->err = "block kernel: unsupported width";
        return TRPLK_EINVAL;
    }
    CK(cudaGetLastError());
    return TRPLK_OK;
}

// +K as one block (B = I): block CGS2 of the c = nprev X^prev columns against U with Cholesky-QR
// inside the block (BCGS2, third pass gated by R3's rule, dependent columns dropped by R16's
// threshold), the accepted vectors appended, then one SpMM for their T columns (eq 3.1).  Four
// passes over U for the whole block instead of four per column.  Default for c >= 3 (measured:
// C3, l = 3: +K 1.45 -> 1.23 ms per cycle, solve 3.59 -> 3.47 s); at c = 2 the per-column path is
// as fast at C5 (29.9 vs 30.5 ms per cycle) and faster at C2 (0.100 vs 0.161 ms: fewer, shorter
// launches).  TRPLK_KPLUS=col / =block force one of them.
bool block_kplus(const trplk_ctx* ctx, int nprev) {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TRPLK_KPLUS");
        v = (e && !strcmp(e, "col")) ? 0 : ((e && !strcmp(e, "block")) ? 2 : 1);
    }
    if (v == 0 || ctx->hasB || nprev < 1 || nprev > BC) return false;
    return v == 2 || nprev >= 3;
}

// The first CGS pass of +K column j (U^T x^prev_j, ||x^prev_j||^2; reading R3) as the second dot
// set of a K1 launch that streams U anyway: the last inner step's K1 (j = 0) or the T-column K1 of
// +K column j - 1.  The column's own first-pass launch is gated on F_XD0 << j, which that K1's
// finalize clears, so it still runs when the K1 did not (inner breakdown, a dropped column, the
// latency paths).  TRPLK_KPLUS_XD=0 at create: off.
static bool kplus_xd_on(const trplk_ctx* ctx, int nprev) {
    return ctx->kplus_xd && nprev > 0 && nprev <= 8 && !ctx->hasB && !block_kplus(ctx, nprev);
}
static void set_kplus_xd(SdotsArgs& a, const double* Uo, int64_t ld, int xprev_static, int j) {
    a.set2 = 4;
    if (xprev_static >= 0) {
        a.x2 = Uo + ld * (xprev_static + j);
    } else {
        a.x2 = Uo;
        a.x2_dyn = 2;
        a.x2_off = j;
        a.x2_ld = ld;
    }
    a.dest2 = D_H0 + 0;
    a.norm2 = 5;
    a.nslot2 = N_IN2;
    a.clear_done = F_XD0 << j;
}

// Block CGS2 (BCGS2 with Cholesky-QR inside the block) of the c vectors Y against the current basis
// Uc(:, 0:ctl->k): two projections (a third gated by R3's rule), dependent vectors dropped (R16),
// the accepted ones appended at Uc(:, ctl->k ..) and copied to the static block xkb; ctl->k grows.
// first_done: the first pass (U^T Y, Y^T Y) is already in blk->HV[0] / blk->G[0] (the fused SpMM).
// c_dyn: the vector count lives on the device (static c is the upper bound for the byte model).
trplk_status bcgs2_blk(trplk_ctx* ctx, double* Uc, int kn, const double* Y, int y_dyn, int c, const int* c_dyn,
                       bool first_done, int seed) {
    const int64_t ld = ctx->ld;
    const double vb = vec_bytes(ctx);
    BlkArgs b{};
    b.nrows = ctx->n_loc;
    b.U = Uc;
    b.ldu = ld;
    b.k_from_ctl = 1;
    b.c = c;
    b.c_dyn = c_dyn;
    b.gate = F_CYCLE;
    if (!first_done) {  // pass 1: H0 = U^T Y, G0 = Y^T Y
        BlkArgs g = b;
        g.mode = BM_GRAM;
        g.Y = Y;
        g.y_dyn = y_dyn;
        g.ldy = ld;
        g.HV = ctx->blk->HV[0];
        g.G = ctx->blk->G[0];
        ST(run_block(ctx, g, kn, vb * (kn + c)));
    }
    // pass 2: W1 = Y - U H0, U^T W1, W1^T W1
    BlkArgs u1 = b;
    u1.mode = BM_UPD;
    u1.Y = Y;
    u1.y_dyn = y_dyn;
    u1.ldy = ld;
    u1.H = ctx->blk->HV[0];
    u1.Yout = ctx->wblk;
    u1.ldyo = ld;
    u1.HV = ctx->blk->HV[1];
    u1.G = ctx->blk->G[1];
    ST(run_block(ctx, u1, kn, vb * (kn + 2 * c)));
    launch_blk_ctl(ctx->blk, ctx->ctl, 1, c, c_dyn, seed, F_CYCLE, ctx->stream);
    // pass 3: W2 = W1 R1^-1 - U (U^T W1 R1^-1) in place, U^T W2, W2^T W2
    BlkArgs u2 = b;
    u2.mode = BM_UPD;
    u2.Y = ctx->wblk;
    u2.ldy = ld;
    u2.Rinv = ctx->blk->Rinv;
    u2.H = ctx->blk->Hs;
    u2.Yout = ctx->wblk;
    u2.ldyo = ld;
    u2.HV = ctx->blk->HV[2];
    u2.G = ctx->blk->G[2];
    ST(run_block(ctx, u2, kn, vb * (kn + 2 * c)));
    launch_blk_ctl(ctx->blk, ctx->ctl, 2, c, c_dyn, seed, F_CYCLE, ctx->stream);
    // gated third pass (R3)
    BlkArgs u3 = u2;
    u3.gate = F_CYCLE | F_BPASS3;
    u3.HV = ctx->blk->HV[3];
    u3.G = ctx->blk->G[3];
    ST(run_block(ctx, u3, kn, 0.0));
    launch_blk_ctl(ctx->blk, ctx->ctl, 3, c, c_dyn, seed, F_CYCLE | F_BPASS3, ctx->stream);
    // accepted vectors Q = W R^-1 into U(:, k0 ..) and the scratch block; ctl->k += accepted
    launch_blk_place(ctx->wblk, ld, ctx->blk, ctx->ctl, Uc, ld, ctx->xkb, ld, ctx->n_loc, 0, F_CYCLE, ctx->stream);
    ctx->launches += 4;
    ctx->model_bytes += vb * 3 * c;
    return TRPLK_OK;
}

// T columns of the block just appended (xkb, blk->acc vectors at blk->k0): T(1:k, k0 + j) = U^T A x~_j
// (eq 3.1), one SpMM.  With W: also W = M (A x~ - rho x~) -> wblk and U^T W, W^T W (the first
// pass of the next block CGS2), SpMM-with-preconditioner of the block inner step (reading B1).
trplk_status block_spmm(trplk_ctx* ctx, double* Uc, int kn, int cmax, bool with_w) {
    const int64_t ld = ctx->ld;
    for (int j = 0; j < cmax; ++j) ST(halo(ctx, ctx->xkb + ld * j));
    BlkArgs sp{};
    sp.nrows = ctx->n_loc;
    sp.U = Uc;
    sp.ldu = ld;
    sp.k_from_ctl = 1;
    sp.mode = with_w ? BM_SPMW : BM_SPMM;
    sp.A = ctx->A;
    sp.sigma = ctx->sigma;
    sp.mfloor = ctx->mfloor_solve;
    sp.Y = ctx->xkb;
    sp.ldy = ld;
    sp.c = cmax;
    sp.c_dyn = &ctx->blk->acc;
    sp.T = ctx->T;
    sp.ldT = QMAX;
    sp.k0p = &ctx->blk->k0;
    sp.gate = F_CYCLE;
    if (with_w) {
        sp.Yout = ctx->wblk;
        sp.ldyo = ld;
        sp.HV = ctx->blk->HV[0];
        sp.G = ctx->blk->G[0];
    }
    const double vb = vec_bytes(ctx);
    return run_block(ctx, sp, kn, mat_bytes(ctx, false) + vb * (kn + (with_w ? 3 : 1) * cmax));
}

trplk_status kplus_block(trplk_ctx* ctx, const Sizes& S, double* Uc, const double* Uo, int nprev, int xprev_static) {
    const int64_t ld = ctx->ld;
    const int kn = S.ph + S.m + nprev;  // widest basis of the cycle
    const double* Y = xprev_static >= 0 ? Uo + ld * xprev_static : Uo;
    ST(bcgs2_blk(ctx, Uc, kn, Y, xprev_static >= 0 ? 0 : 2, nprev, nullptr, false, 0));
    return block_spmm(ctx, Uc, kn, nprev, false);
}

// Block inner loop (trplk_options.block = b > 1, reading B1): seeds M r_{t+i}, i < be, block CGS2
// against X; then per group G_j of the block Krylov space of eq 3.2's C: one SpMM with the
// preconditioner (T columns of G_j and W = M (A - rho B) G_j with its first-pass dots), a block
// CGS2 of the images that still fit the basis (p^ + m columns), appended as G_{j+1}.
trplk_status inner_block(trplk_ctx* ctx, const Sizes& S, double* Uc, int be, int extras) {
    const int64_t ld = ctx->ld;
    const int kn = S.ph + S.m;
    if (extras)  // residuals of the next targets (the cycle's first is ctx->u): one A-matvec each
        for (int i = 1; i < be; ++i) {
            SdotsArgs a = sd_base(ctx);
            a.A = ctx->A;
            a.x = Uc;
            a.x_dyn = 1;
            a.x_off = i;
            a.out_mode = 3;
            a.uout = ctx->sblk + ld * i;
            a.norm1 = 1;
            a.nslot1 = N_AUX;
            a.theta_idx = -1;
            a.gate = F_CYCLE;
            if (ctx->nranks > 1) {
                ctx->err = "block inner loop: one rank only";
                return TRPLK_EINVAL;
            }
            ST(run_sdots(ctx, a, 0));
        }
    launch_copy_cols(ctx->u, ld, ctx->sblk, ld, ctx->n_loc, 1, ctx->stream);
    ctx->launches += 1;
    ST(bcgs2_blk(ctx, Uc, kn, ctx->sblk, 0, be, nullptr, false, 1));
    const int steps = (S.m + be - 1) / be;
    for (int s = 1; s <= steps; ++s) {
        if (s < steps) {
            ST(block_spmm(ctx, Uc, kn, be, true));
            launch_blk_room(ctx->blk, ctx->ctl, S.ph + S.m, F_CYCLE, ctx->stream);
            ctx->launches += 1;
            ST(bcgs2_blk(ctx, Uc, kn, ctx->wblk, 0, be, &ctx->blk->cin, true, 0));
        } else {
            ST(block_spmm(ctx, Uc, kn, be, false));
        }
    }
    return TRPLK_OK;
}

// phase boundary event of the live cycle profile (trplk_profile_phases)
static trplk_status phase_mark(trplk_ctx* ctx, int i) {
    if (ctx->prof_on) CK(record_event(ctx, ctx->phev[i]));
    return TRPLK_OK;
}

// One outer cycle after the seed vector u is in place: eq 3.1 inner steps, +K, RR, rotation,
// residual of the target.  Issued eagerly or under stream capture.
trplk_status issue_cycle(trplk_ctx* ctx, const Sizes& S, int cur, int nprev, int t_static, int xprev_static,
                         int be, int extras) {
    const int oth = 1 - cur;
    double* Uc = ctx->U[cur];
    double* Uo = ctx->U[oth];
    const int64_t ld = ctx->ld;
    // seed: g_1 = (I - X X^T B) u / beta  (eq 3.2 u1 = C x_t, R4), written to column p^
    ST(phase_mark(ctx, 0));
    if (be > 1) {  // block TRPL+K (reading B1): seeds, block inner loop
        ST(phase_mark(ctx, 1));
        ST(inner_block(ctx, S, Uc, be, extras));
    } else {
        CgsSpec c{};
        c.x = ctx->u;
        c.V = Uc;
        c.kv = S.ph;
        c.k_nominal = S.ph;
        c.first_done = false;
        c.dest = Uc;
        c.dest_dyn = 1;
        c.gate = F_CYCLE;
        c.clear = F_CYCLE;
        c.inc_k = 1;
        ST(cgs2(ctx, c));
    // inner steps, eq 3.1
    ST(phase_mark(ctx, 1));
    const int jmid = std::max(1, std::min(S.m - 1, S.m / 2));
    const bool fused = small_path(ctx, S) || grid_path(ctx, S);
    if (fused) {  // one kernel runs all m steps (latency paths, small.cuh / inner_grid.cuh)
        SmallArgs sa{};
        sa.A = ctx->A;
        sa.nrows = ctx->n_loc;
        sa.U = Uc;
        sa.ldu = ld;
        sa.w = ctx->w;
        sa.w1 = ctx->w1;
        sa.w2 = ctx->w2;
        sa.ctl = ctx->ctl;
        sa.T = ctx->T;
        sa.ldT = QMAX;
        sa.m = S.m;
        sa.sigma = ctx->sigma;
        sa.mfloor = ctx->mfloor_solve;
        sa.pmode = ctx->pmode;
        sa.gate = F_CYCLE | F_INNER;
        sa.clear = F_INNER;
        sa.force3 = ctx->force3;
        if (ctx->prof_on) CK(record_event(ctx, ctx->pev[0]));
        if (small_path(ctx, S)) {
            launch_inner_small(sa, S.q, ctx->stream);
            ctx->prof_kern[0] = g_last_kern;
        } else {
            GridArgs ga{sa, ctx->gridpart, nullptr};
            static const bool trace = getenv("TRPLK_GRID_TRACE") != nullptr;
            if (trace) {
                if (!ctx->gtrace) ST(dalloc(ctx, &ctx->gtrace, 8 * 64));
                ga.trace = ctx->gtrace;
            }
            if (!launch_inner_grid(ga, S.q, ctx->stream)) {
                ctx->err = "cooperative launch of the grid-wide inner loop failed";
                return TRPLK_ECUDA;
            }
            ctx->prof_kern[0] = g_last_kern;
        }
        CK(cudaGetLastError());
        if (ctx->prof_on)
            for (int e = 1; e < 4; ++e) CK(record_event(ctx, ctx->pev[e]));
        ctx->launches += 1;
        for (int j = 1; j <= S.m; ++j) {  // byte model of the m steps (as the multi-kernel path)
            const int k = S.ph + j;
            ctx->model_bytes += mat_bytes(ctx, false) + vec_bytes(ctx) * (k + 2);
            if (j < S.m) ctx->model_bytes += 2 * vec_bytes(ctx) * (k + 2);
        }
    }
    // K1 arguments of inner step j (eq 3.1: z = A g_j, T(1:k,k) = U^T z, w = M (z - rho B g_j),
    // h0 = U^T w, ||w||^2)
    bool xd = false;
    auto k1_args = [&](int j) {
        const int k = S.ph + j;
        SdotsArgs a = sd_base(ctx);
        a.A = ctx->A;
        a.x = Uc + ld * (k - 1);
        a.U = Uc;
        a.k_from_ctl = 1;
        a.set1 = 1;  // T(1:k,k) = U^T z
        a.dest1 = D_TCOL;
        a.gate = F_CYCLE | F_INNER;
        if (j < S.m) {
            a.out_mode = 2;  // w = M (z - rho B g)
            a.out = ctx->w;
            if (ctx->hasB) {
                a.B = ctx->B;
            } else if (ctx->pmode != 3) {
                a.set2 = 2;  // h0 = U^T w
                a.dest2 = D_H0 + 0;
                a.norm1 = 1;  // ||w||^2
                a.nslot1 = N_IN2;
            }
        } else if (xd) {
            set_kplus_xd(a, Uo, ld, xprev_static, 0);  // +K column 0's first CGS pass rides along
        }
        return a;
    };
    // fz: the FINAL of step j and the K1 of step j+1 run as one kernel (fused.cuh)
    const bool fz = !fused && fuse_path(ctx, S);
    xd = !fz && kplus_xd_on(ctx, nprev);
    ctx->prof_fused = fz;
    for (int j = 1; j <= S.m && !fused; ++j) {
        const int k = S.ph + j;  // nominal width incl. g_j
        const bool prof = ctx->prof_on && j == jmid && j < S.m;
        const double* g = Uc + ld * (k - 1);
        SdotsArgs a = k1_args(j);
        const bool k1_done = fz && j > 1;  // ran inside the previous step's fused kernel
        const bool ov = !k1_done && k1_overlap_ok(ctx, a, k);
        if (!ov) ST(halo(ctx, g));
        if (j < S.m) {
            const bool ic0 = ctx->pmode == 3;
            if (prof && !fz) CK(record_event(ctx, ctx->pev[0]));
            if (!k1_done) ST(ov ? run_k1_overlap(ctx, a, k) : run_sdots(ctx, a, k));
            if (prof && !fz) ctx->prof_kern[0] = g_last_kern;
            if (ic0) ST(ic0_apply(ctx, ctx->w, F_CYCLE | F_INNER));  // w = (L L^T)^-1 (z - rho g)
            if (prof) CK(record_event(ctx, ctx->pev[fz ? 0 : 1]));
            CgsSpec c{};
            SdotsArgs an{};
            if (fz) {
                an = k1_args(j + 1);
                c.fuse_next = &an;
                c.k_next = k + 1;
            }
            if (prof) c.mark_final = ctx->pev[fz ? 1 : 2];
            c.x = ctx->w;
            c.V = Uc;
            c.kv = -1;
            c.k_nominal = k;
            c.first_done = !ctx->hasB && ctx->pmode != 3;
            c.dest = Uc;
            c.dest_dyn = 1;
            c.gate = F_CYCLE | F_INNER;
            c.clear = F_INNER;
            c.inc_k = 1;
            ST(cgs2(ctx, c));
            if (prof) {
                CK(record_event(ctx, ctx->pev[fz ? 2 : 3]));
                if (fz) CK(record_event(ctx, ctx->pev[3]));
            }
        } else if (!k1_done) {
            ST(ov ? run_k1_overlap(ctx, a, k) : run_sdots(ctx, a, k));
        }
    }
    }  // seed + inner loop of Algorithm 1
    // +K: X^prev appended after G, explicitly orthogonalised, one matvec each
    ST(phase_mark(ctx, 2));
    if (block_kplus(ctx, nprev)) ST(kplus_block(ctx, S, Uc, Uo, nprev, xprev_static));
    const bool fz = fuse_path(ctx, S);
    const bool xdk = !fz && kplus_xd_on(ctx, nprev);
    for (int jj = 0; jj < nprev && !block_kplus(ctx, nprev); ++jj) {
        const unsigned kb = F_KCOL0 << jj;
        CgsSpec c{};
        if (xprev_static >= 0) {
            c.x = Uo + ld * (xprev_static + jj);
        } else {
            c.x = Uo;
            c.x_dyn = 2;
            c.x_off = jj;
        }
        c.V = Uc;
        c.kv = -1;
        c.k_nominal = S.ph + S.m + jj;
        c.dest = Uc;
        c.dest_dyn = 1;
        c.dest2 = fz ? nullptr : ctx->xk;
        c.gate = F_CYCLE | kb;
        if (xdk) c.gate1 = F_XD0 << jj;  // unless the preceding K1 computed this first pass
        c.clear = kb;
        c.inc_k = 1;
        // the column's one matvec and T column: z = A x, T(1:k,k) = U^T z (fused with the FINAL
        // update when the inner steps are, reading x from its basis column)
        SdotsArgs a = sd_base(ctx);
        a.A = ctx->A;
        a.x = ctx->xk;
        a.U = Uc;
        a.k_from_ctl = 1;
        a.set1 = 1;
        a.dest1 = D_TCOL;
        a.gate = F_CYCLE | kb;
        if (xdk && jj + 1 < nprev) set_kplus_xd(a, Uo, ld, xprev_static, jj + 1);  // next column's first pass
        if (fz) {
            c.fuse_next = &a;
            c.k_next = S.ph + S.m + jj + 1;
        }
        ST(cgs2(ctx, c));
        if (fz) continue;
        ST(halo(ctx, ctx->xk));
        ST(run_sdots(ctx, a, S.ph + S.m + jj + 1));
    }
    // Rayleigh-Ritz (step 11) and rotation X = U Y(:,1:p^) into the other buffer
    ST(phase_mark(ctx, 3));
    launch_eig(ctx->ctl, ctx->T, QMAX, ctx->Yg, QMAX, S.ph, 0, F_CYCLE, ctx->stream);
    CK(cudaGetLastError());
    ST(phase_mark(ctx, 4));
    launch_rotate(Uc, ld, ctx->n_loc, ctx->ctl, 0, ctx->Yg, QMAX, S.ph, Uo, ld, F_CYCLE, ctx->stream, S.q);
    ctx->launches += 2;
    CK(cudaGetLastError());
    ctx->model_bytes += vec_bytes(ctx) * (S.q + S.ph);
    // residual of the target, u = M r (steps 12, 15)
    ST(phase_mark(ctx, 5));
    if (t_static > 0) ST(residual(ctx, Uo + ld * (t_static - 1), 0, -1, ctx->u, F_CYCLE));
    else ST(residual(ctx, Uo, 1, -1, ctx->u, F_CYCLE));
    ST(phase_mark(ctx, 6));
    return TRPLK_OK;
}

// Process-wide cache of instantiated cycle graphs, keyed by everything a captured kernel
// argument can depend on: the cycle key, the solve sizes, every device allocation of the
// context (address and size, in allocation order), the matrix descriptors and the scalar
// arguments.  A context created right after another one of the same problem (the e2e path:
// create -> solve -> destroy, again and again) usually gets the same device addresses back from
// the allocator, so its graphs are reused instead of captured and instantiated again.
static std::mutex g_graph_mu;
static std::map<std::string, GraphRec> g_graph_cache;
static std::vector<std::string> g_graph_order;
constexpr size_t GRAPH_CACHE_MAX = 64;

static std::string graph_fingerprint(const trplk_ctx* ctx, uint64_t key, const Sizes& S) {
    std::string f;
    auto put = [&f](const void* p, size_t n) { f.append(static_cast<const char*>(p), n); };
    put(&key, sizeof(key));
    put(&S, sizeof(S));
    for (const auto& a : ctx->allocs) {
        put(&a.first, sizeof(a.first));
        put(&a.second, sizeof(a.second));
    }
    for (const Sell* M : {&ctx->A, &ctx->B}) {  // field by field (no padding bytes)
        const int64_t v[11] = {M->fmt, M->nrows, M->nslices, (int64_t)(uintptr_t)M->sptr, (int64_t)(uintptr_t)M->col,
                               (int64_t)(uintptr_t)M->val, M->ndiag, M->diag_slot, M->ldv, M->glo, M->nghost};
        put(v, sizeof(v));
        put(&M->dval, sizeof(M->dval));
        put(M->offs, sizeof(M->offs));
        const int64_t c[2] = {(int64_t)M->cmask, (int64_t)(uintptr_t)M->pmask};
        put(c, sizeof(c));
        put(M->cv, sizeof(M->cv));
    }
    const double sc[5] = {ctx->sigma, ctx->mfloor, ctx->normF, ctx->mfloor_solve, (double)ctx->pmode};
    put(sc, sizeof(sc));
    const int64_t iv[6] = {ctx->n_loc, ctx->ld, ctx->row_begin, ctx->n_global, (int64_t)ctx->force3,
                           (int64_t)ctx->grid_on};
    put(iv, sizeof(iv));
    put(&ctx->ctl_h, sizeof(ctx->ctl_h));
    return f;
}

// hand a context's graphs to the cache (destroy) / take matching ones back (run_cycle)
static void graphs_to_cache(trplk_ctx* ctx) {
    if (ctx->nranks > 1 || ctx->prof_on) {
        for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.second.exec);
        ctx->graphs.clear();
        return;
    }
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto& g : ctx->graphs) {
        const std::string f = graph_fingerprint(ctx, g.first, ctx->gsizes);
        auto it = g_graph_cache.find(f);
        if (it != g_graph_cache.end()) {
            cudaGraphExecDestroy(g.second.exec);
            continue;
        }
        g_graph_cache.emplace(f, g.second);
        g_graph_order.push_back(f);
        if (g_graph_order.size() > GRAPH_CACHE_MAX) {
            auto old = g_graph_cache.find(g_graph_order.front());
            if (old != g_graph_cache.end()) {
                cudaGraphExecDestroy(old->second.exec);
                g_graph_cache.erase(old);
            }
            g_graph_order.erase(g_graph_order.begin());
        }
    }
    ctx->graphs.clear();
}

static bool graph_from_cache(trplk_ctx* ctx, uint64_t key, const Sizes& S, GraphRec& rec) {
    if (ctx->nranks > 1 || ctx->prof_on) return false;
    const std::string f = graph_fingerprint(ctx, key, S);
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = g_graph_cache.find(f);
    if (it == g_graph_cache.end()) return false;
    rec = it->second;
    g_graph_cache.erase(it);
    g_graph_order.erase(std::find(g_graph_order.begin(), g_graph_order.end(), f));
    return true;
}

trplk_status run_cycle(trplk_ctx* ctx, const Sizes& S, int cur, int nprev, int t, int xprev, bool use_graph, int be,
                       int extras) {
    if (ctx->loopback) use_graph = false;  // loopback exchanges are host rendezvous: eager only
    const bool multi = ctx->nranks > 1;
    const int ts = multi ? t : -1;  // static addresses are needed for the halo exchange
    const int xs = multi ? xprev : -1;
    if (!use_graph) return issue_cycle(ctx, S, cur, nprev, ts, xs, be, extras);
    if (!(ctx->gsizes == S)) {
        for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.second.exec);
        ctx->graphs.clear();
        ctx->gsizes = S;
    }
    const uint64_t key = ((uint64_t)cur) | ((uint64_t)nprev << 1) | ((uint64_t)(ts + 1) << 8) |
                         ((uint64_t)(xs + 1) << 24) | ((uint64_t)(ctx->prof_on ? 1 : 0) << 40) |
                         ((uint64_t)be << 44) | ((uint64_t)(extras ? 1 : 0) << 52);
    auto it = ctx->graphs.find(key);
    if (it == ctx->graphs.end()) {
        GraphRec cached;
        if (graph_from_cache(ctx, key, S, cached)) it = ctx->graphs.emplace(key, cached).first;
    }
    if (it == ctx->graphs.end()) {
        const double mb0 = ctx->model_bytes;
        const int64_t l0 = ctx->launches;
        cudaGraph_t graph;
        CK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
        trplk_status st = issue_cycle(ctx, S, cur, nprev, ts, xs, be, extras);
        cudaError_t e = cudaStreamEndCapture(ctx->stream, &graph);
        if (st != TRPLK_OK) return st;
        if (e != cudaSuccess) {
            ctx->err = std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e);
            return TRPLK_ECUDA;
        }
        GraphRec rec;
        rec.bytes = ctx->model_bytes - mb0;
        ctx->model_bytes = mb0;
        rec.launches = ctx->launches - l0;
        ctx->launches = l0;
        CK(cudaGraphInstantiate(&rec.exec, graph, 0));
        cudaGraphDestroy(graph);
        it = ctx->graphs.emplace(key, rec).first;
    }
    CK(cudaGraphLaunch(it->second.exec, ctx->stream));
    ctx->model_bytes += it->second.bytes;
    ctx->launches += it->second.launches;
    return TRPLK_OK;
}

}  // namespace

// ======================================================================= ABI
extern "C" {

void trplk_options_default(trplk_options* opt) {
    if (!opt) return;
    opt->seed = 12;
    opt->max_cycles = 5000;
    opt->tol_mode = 0;
    opt->restart_size = 0;
    opt->lock_mode = 0;
    opt->debug_checks = 0;
    opt->use_graphs = 1;
    opt->precond = 0;
    opt->block = 1;
}

trplk_status trplk_nccl_unique_id(void* out, size_t out_bytes) {
    if (!out || out_bytes < sizeof(ncclUniqueId)) return TRPLK_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return TRPLK_ENCCL;
    memcpy(out, &id, sizeof(id));
    return TRPLK_OK;
}

const char* trplk_last_error(const trplk_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

// TRPLK_TIMING=1: host wall time of the create phases on stderr (tools/e2e_breakdown.py).
struct PhaseTimer {
    const char* what;
    bool on;
    std::chrono::steady_clock::time_point t;
    explicit PhaseTimer(const char* w) : what(w), on(getenv("TRPLK_TIMING") != nullptr), t(std::chrono::steady_clock::now()) {}
    void mark(const char* phase) {
        if (!on) return;
        auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "[trplk %s] %-10s %8.3f ms\n", what, phase,
                std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

static trplk_status create_impl(trplk_ctx* ctx, int64_t n_global, const int64_t* a_rowptr, const int64_t* a_col,
                                const double* a_val, const int64_t* b_rowptr, const int64_t* b_col,
                                const double* b_val, double sigma, const trplk_dist* dist, void* hubp,
                                const trplk_host_comm* hc) {
    ctx->n_global = n_global;
    ctx->sigma = sigma;
    PhaseTimer pt("create");
    if (n_global < 1) {
        ctx->err = "n_global < 1";
        return TRPLK_EINVAL;
    }
    if (dist) {
        ctx->rank = dist->rank;
        ctx->nranks = dist->nranks;
        ctx->row_begin = dist->row_begin;
        ctx->row_end = dist->row_end;
        if (ctx->nranks < 1 || ctx->rank < 0 || ctx->rank >= ctx->nranks || ctx->row_begin < 0 ||
            ctx->row_end > n_global || ctx->row_end <= ctx->row_begin) {
            ctx->err = "bad trplk_dist (rank/nranks/row range)";
            return TRPLK_EINVAL;
        }
        if (ctx->nranks > 1 && !dist->nccl_unique_id && !hubp && !hc) {
            ctx->err = "nranks > 1 needs nccl_unique_id (trplk_create_ex: a loopback hub or host callbacks)";
            return TRPLK_EINVAL;
        }
    } else {
        ctx->row_begin = 0;
        ctx->row_end = n_global;
    }
    ctx->n_loc = ctx->row_end - ctx->row_begin;
    ctx->hasB = b_rowptr != nullptr;
    if ((b_rowptr == nullptr) != (b_col == nullptr) || (b_rowptr == nullptr) != (b_val == nullptr)) {
        ctx->err = "B: give all three CSR arrays or none";
        return TRPLK_EINVAL;
    }
    if (!a_val) {
        ctx->err = "A: NULL values";
        return TRPLK_EINVAL;
    }
    // validation, ghosts, DIA offsets and norms in one parallel pass per matrix
    CsrScan scA, scB;
    ST(scan_csr(ctx, "A", a_rowptr, a_col, a_val, scA));
    if (ctx->hasB) ST(scan_csr(ctx, "B", b_rowptr, b_col, nullptr, scB));
    pt.mark("scan");

    if (ctx->nranks > 1) {
        if (hubp) {
            LoopHub* hub = static_cast<LoopHub*>(hubp);
            if (hub->n != ctx->nranks) {
                ctx->err = "loopback hub size != nranks";
                return TRPLK_EINVAL;
            }
            ctx->cm = new LoopComm(hub, ctx->rank);
            ctx->loopback = true;
        } else if (hc) {
            if (!hc->allgather || !hc->sendrecv || !hc->allreduce) {
                ctx->err = "trplk_host_comm: NULL callback";
                return TRPLK_EINVAL;
            }
            HostComm* h = new HostComm(*hc);
            h->nranks = ctx->nranks;
            ctx->cm = h;
            ctx->loopback = true;  // host rendezvous: eager launches
        } else {
            NcclComm* c = new NcclComm();
            ctx->cm = c;
            ncclUniqueId id;
            memcpy(&id, dist->nccl_unique_id, sizeof(id));
            NK(ncclCommInitRank(&c->comm, ctx->nranks, id, ctx->rank));
        }
    }
    // ghost columns (global ids outside the owned range), sorted
    std::vector<int64_t> ghosts = std::move(scA.ghosts);
    ghosts.insert(ghosts.end(), scB.ghosts.begin(), scB.ghosts.end());
    std::sort(ghosts.begin(), ghosts.end());
    ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
    ctx->n_ghost = (int64_t)ghosts.size();
    if (ctx->n_loc + ctx->n_ghost >= (int64_t)1 << 31) {
        ctx->err = "local rows + ghosts exceed int32 column ids";
        return TRPLK_EINVAL;
    }
    ctx->ld = ((ctx->n_loc + ctx->n_ghost + 31) / 32) * 32;
    ctx->nnzA = a_rowptr[ctx->n_loc] - a_rowptr[0];
    ctx->nnzB = ctx->hasB ? b_rowptr[ctx->n_loc] - b_rowptr[0] : 0;

    // ||A||_F and max |A_jj| (local, then across ranks)
    double fro2 = scA.fro2, amax = scA.amax;

    // device format: DIA when the matrix is a few full diagonals (stencils), else SELL-32
    const bool force_sell = getenv("TRPLK_FORCE_SELL") != nullptr;
    bool diaA = false, diaB = false;
    if (!force_sell) ST(try_dia(ctx, a_rowptr, a_col, a_val, ghosts, scA, ctx->A, ctx->sellA_bytes, diaA));
    if (!diaA) {
        HostSell hs;
        ST(build_sell(ctx, a_rowptr, a_col, a_val, ghosts, hs));
        ST(upload_sell(ctx, hs, ctx->A, ctx->sellA_bytes));
    }
    if (ctx->hasB) {
        if (!force_sell) ST(try_dia(ctx, b_rowptr, b_col, b_val, ghosts, scB, ctx->B, ctx->sellB_bytes, diaB));
        if (!diaB) {
            HostSell hb;
            ST(build_sell(ctx, b_rowptr, b_col, b_val, ghosts, hb));
            ST(upload_sell(ctx, hb, ctx->B, ctx->sellB_bytes));
        }
    }

    if (ctx->A.cmask == 0) ctx->sellA_bytes_dc = ctx->sellA_bytes;
    pt.mark("format");
    // fixed device buffers
    const size_t ld = (size_t)ctx->ld;
    ST(dalloc(ctx, &ctx->w, ld));
    ST(dalloc(ctx, &ctx->w1, ld));
    ST(dalloc(ctx, &ctx->w2, ld));
    ST(dalloc(ctx, &ctx->u, ld));
    ST(dalloc(ctx, &ctx->u2, ld));
    ST(dalloc(ctx, &ctx->xk, ld));
    ST(dalloc(ctx, &ctx->T, (size_t)QMAX * QMAX));
    ST(dalloc(ctx, &ctx->Yg, (size_t)QMAX * QMAX));
    ST(dalloc(ctx, &ctx->part, (size_t)NV_MAX * MAXCTA));
    ST(dalloc(ctx, &ctx->gpart, (size_t)NV_MAX * MAXG));
    ST(dalloc(ctx, &ctx->red_local, (size_t)NV_MAX));
    ST(dalloc(ctx, &ctx->red_all, (size_t)NV_MAX * ctx->nranks));
    ST(dalloc(ctx, &ctx->counter, NCOUNTERS));
    ST(dalloc(ctx, &ctx->blk, 1));
    ST(dalloc(ctx, &ctx->bpart, (size_t)BLK_NV * MAXCTA));
    ST(dalloc(ctx, &ctx->bgpart, (size_t)BLK_NV * MAXG));
    ST(dalloc(ctx, &ctx->bcounter, NCOUNTERS));
    ST(dalloc(ctx, &ctx->bred_local, (size_t)BLK_NV));
    ST(dalloc(ctx, &ctx->bred_all, (size_t)BLK_NV * ctx->nranks));
    CK(cudaMemsetAsync(ctx->bcounter, 0, sizeof(unsigned) * NCOUNTERS, ctx->stream));
    CK(cudaMemsetAsync(ctx->blk, 0, sizeof(BlkCtl), ctx->stream));
    if (ctx->nranks == 1 && !ctx->hasB) ST(dalloc(ctx, &ctx->gridpart, (size_t)2 * GRID_MAXCTA * GRID_NVP));
    {  // opt-in: measured slower than the three-kernel step (fused K3 + K1)
        const char* e = getenv("TRPLK_FUSE");
        ctx->fuse_on = e && e[0] == '1';
        const char* x = getenv("TRPLK_KPLUS_XD");
        ctx->kplus_xd = !(x && x[0] == '0');
    }
    if (ctx->nranks > 1 && !ctx->hasB && ctx->A.fmt == 1) {  // halo overlap: interior rows of the slab
        const char* e = getenv("TRPLK_HALO_OVERLAP");
        int lo = 0, hi = 0;
        for (int d = 0; d < ctx->A.ndiag; ++d) {
            lo = std::max(lo, -ctx->A.offs[d]);
            hi = std::max(hi, ctx->A.offs[d]);
        }
        ctx->hb0 = ((int64_t)lo + 31) / 32 * 32;
        ctx->hb1 = (ctx->n_loc - hi) / 32 * 32;
        ctx->hov = !(e && e[0] == '0') && ctx->hb1 - ctx->hb0 >= 64;
        if (ctx->hov && !ctx->hstream) {
            CK(cudaStreamCreateWithFlags(&ctx->hstream, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ctx->hev_fork, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->hev_done, cudaEventDisableTiming));
        }
    }
    if (ctx->nranks == 1 && !ctx->hasB && ctx->A.fmt == 1) {
        ctx->rcnt_cap = (ctx->n_loc + 31) / 32 / (148 * WARPS) + 64;
        ST(dalloc(ctx, &ctx->rcnt, (size_t)ctx->rcnt_cap));
        CK(cudaMemsetAsync(ctx->rcnt, 0, sizeof(unsigned) * ctx->rcnt_cap, ctx->stream));
    }
    ST(dalloc(ctx, &ctx->ctl, 1));
    CK(cudaMemsetAsync(ctx->counter, 0, sizeof(unsigned) * NCOUNTERS, ctx->stream));
    CK(cudaMemsetAsync(ctx->ctl, 0, sizeof(Ctl), ctx->stream));
    CK(cudaMemsetAsync(ctx->T, 0, sizeof(double) * QMAX * QMAX, ctx->stream));
    for (double* v : {ctx->w, ctx->w1, ctx->w2, ctx->u, ctx->u2, ctx->xk})
        CK(cudaMemsetAsync(v, 0, ld * 8, ctx->stream));
    ctx->ctl_h = ctl_host_alloc();
    if (!ctx->ctl_h) {
        ctx->err = "cudaMallocHost (control block)";
        return TRPLK_ENOMEM;
    }
    memset(ctx->ctl_h, 0, sizeof(Ctl));
    pt.mark("buffers");

    if (ctx->nranks > 1) {
        // global ||A||_F^2 and max |A_jj|
        double* tmp;
        ST(dalloc(ctx, &tmp, 2 + 2 * (size_t)ctx->nranks));
        CM(ctx->cm->allreduce_host(&fro2, 1, 0, ctx->stream, tmp));
        CM(ctx->cm->allreduce_host(&amax, 1, 1, ctx->stream, tmp));
        // all row ranges
        int64_t* ranges;
        ST(dalloc(ctx, &ranges, 2 * (size_t)ctx->nranks + 2));
        int64_t mine[2] = {ctx->row_begin, ctx->row_end};
        CK(cudaMemcpyAsync(ranges + 2 * ctx->nranks, mine, 16, cudaMemcpyHostToDevice, ctx->stream));
        CM(ctx->cm->allgather(ranges + 2 * ctx->nranks, ranges, 2, 8, ctx->stream));
        std::vector<int64_t> rg(2 * (size_t)ctx->nranks);
        CK(cudaMemcpyAsync(rg.data(), ranges, 16 * (size_t)ctx->nranks, cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        int64_t tot = 0;
        for (int r = 0; r < ctx->nranks; ++r) {
            tot += rg[2 * r + 1] - rg[2 * r];
            if (r > 0 && rg[2 * r] != rg[2 * r - 1]) {
                ctx->err = "row ranges do not tile [0, n) in rank order";
                return TRPLK_EINVAL;
            }
        }
        if (tot != n_global || rg[0] != 0) {
            ctx->err = "row ranges do not tile [0, n)";
            return TRPLK_EINVAL;
        }
        // recv plan: ghosts grouped by owner (contiguous, since sorted)
        std::vector<int64_t> need_cnt(ctx->nranks, 0), need_off(ctx->nranks, 0);
        const std::vector<int> owners = ghost_owners(ghosts, rg.data(), ctx->nranks);
        for (size_t gi = 0; gi < ghosts.size(); ++gi) {
            const int owner = owners[gi];
            if (need_cnt[owner] == 0) need_off[owner] = (int64_t)gi;
            need_cnt[owner]++;
        }
        // exchange counts (all-to-all through allgather of the count matrix)
        int64_t* cnts;
        ST(dalloc(ctx, &cnts, (size_t)ctx->nranks * ctx->nranks + ctx->nranks));
        CK(cudaMemcpyAsync(cnts + (size_t)ctx->nranks * ctx->nranks, need_cnt.data(), 8 * (size_t)ctx->nranks,
                           cudaMemcpyHostToDevice, ctx->stream));
        CM(ctx->cm->allgather(cnts + (size_t)ctx->nranks * ctx->nranks, cnts, ctx->nranks, 8, ctx->stream));
        std::vector<int64_t> cm((size_t)ctx->nranks * ctx->nranks);
        CK(cudaMemcpyAsync(cm.data(), cnts, 8 * cm.size(), cudaMemcpyDeviceToHost, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        // exchange the requested global ids
        int64_t* gdev;
        ST(dalloc(ctx, &gdev, ghosts.size() + 1));
        if (!ghosts.empty())
            CK(cudaMemcpyAsync(gdev, ghosts.data(), 8 * ghosts.size(), cudaMemcpyHostToDevice, ctx->stream));
        std::vector<int64_t*> req(ctx->nranks, nullptr);
        std::vector<Xfer> sends, recvs;
        for (int s = 0; s < ctx->nranks; ++s) {
            if (s == ctx->rank) continue;
            const int64_t they_need = cm[(size_t)s * ctx->nranks + ctx->rank];
            if (they_need > 0) {
                ST(dalloc(ctx, &req[s], (size_t)they_need));
                recvs.push_back({s, req[s], (size_t)they_need});
            }
            if (need_cnt[s] > 0) sends.push_back({s, gdev + need_off[s], (size_t)need_cnt[s]});
        }
        CM(ctx->cm->sendrecv(sends, recvs, 8, ctx->stream));
        CK(cudaStreamSynchronize(ctx->stream));
        int64_t sendtot = 0;
        for (int s = 0; s < ctx->nranks; ++s) {
            if (s == ctx->rank) continue;
            const int64_t they_need = cm[(size_t)s * ctx->nranks + ctx->rank];
            if (they_need == 0 && need_cnt[s] == 0) continue;
            ctx->peers.push_back(s);
            ctx->recv_off.push_back(need_off[s]);
            ctx->recv_cnt.push_back(need_cnt[s]);
            ctx->send_cnt.push_back(they_need);
            std::vector<int64_t> ids(they_need);
            if (they_need) CK(cudaMemcpy(ids.data(), req[s], 8 * they_need, cudaMemcpyDeviceToHost));
            bool contig = true;
            for (int64_t i = 1; i < they_need; ++i) contig &= ids[i] == ids[i - 1] + 1;
            if (they_need > 0 && contig) {
                ctx->send_start.push_back(ids[0] - ctx->row_begin);
                ctx->send_idx.push_back(nullptr);
            } else {
                ctx->send_start.push_back(-1);
                std::vector<int> loc(they_need);
                for (int64_t i = 0; i < they_need; ++i) loc[i] = (int)(ids[i] - ctx->row_begin);
                int* d = nullptr;
                ST(dalloc(ctx, &d, (size_t)std::max<int64_t>(they_need, 1)));
                if (they_need) {
                    CK(cudaMemcpyAsync(d, loc.data(), 4 * they_need, cudaMemcpyHostToDevice, ctx->stream));
                    CK(cudaStreamSynchronize(ctx->stream));  // loc is a local
                }
                ctx->send_idx.push_back(d);
            }
            sendtot += they_need;
        }
        ST(dalloc(ctx, &ctx->sendbuf, (size_t)std::max<int64_t>(sendtot, 1)));
    }
    ctx->normF = std::sqrt(fro2);
    ctx->amax = amax;
    ctx->mfloor = 1e-8 * amax;  // S:192 floor eps_d * max_j |A_jj| (R12)
    CK(cudaStreamSynchronize(ctx->stream));
    pt.mark("halo+sync");
    return TRPLK_OK;
}

trplk_status trplk_create(trplk_ctx** out, int64_t n_global, const int64_t* a_rowptr, const int64_t* a_col,
                          const double* a_val, const int64_t* b_rowptr, const int64_t* b_col, const double* b_val,
                          double sigma, const trplk_dist* dist, const trplk_allocator* alloc, void* stream) {
    return trplk_create_ex(out, n_global, a_rowptr, a_col, a_val, b_rowptr, b_col, b_val, sigma, dist, nullptr,
                           nullptr, alloc, stream);
}

trplk_status trplk_create_ex(trplk_ctx** out, int64_t n_global, const int64_t* a_rowptr, const int64_t* a_col,
                             const double* a_val, const int64_t* b_rowptr, const int64_t* b_col, const double* b_val,
                             double sigma, const trplk_dist* dist, void* loopback_hub,
                             const trplk_host_comm* host_comm, const trplk_allocator* alloc, void* stream) {
    if (!out) return TRPLK_EINVAL;
    if ((loopback_hub || host_comm) && (!dist || (loopback_hub && host_comm))) {
        *out = nullptr;
        return TRPLK_EINVAL;
    }
    trplk_ctx* ctx = new trplk_ctx();
    *out = ctx;
    ctx->user_stream = (cudaStream_t)stream;
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming) != cudaSuccess) {
        ctx->err = "cannot create the work stream";
        return TRPLK_ECUDA;
    }
    enter_stream(ctx);
    if (alloc && alloc->alloc && alloc->free) {
        ctx->alloc = *alloc;
        ctx->has_alloc = true;
    }
    return create_impl(ctx, n_global, a_rowptr, a_col, a_val, b_rowptr, b_col, b_val, sigma, dist, loopback_hub,
                       host_comm);
}

void trplk_destroy(trplk_ctx* ctx) {
    if (!ctx) return;
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->user_stream) cudaStreamSynchronize(ctx->user_stream);
    graphs_to_cache(ctx);  // before the allocations go: the fingerprint lists them
    for (auto& a : ctx->allocs) dev_release(ctx, a.first);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (!ctx->has_alloc) trim_pool();
    ctl_host_free(ctx->ctl_h);
    if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
    if (ctx->hev_fork) cudaEventDestroy(ctx->hev_fork);
    if (ctx->hev_done) cudaEventDestroy(ctx->hev_done);
    if (ctx->hstream) cudaStreamDestroy(ctx->hstream);
    for (auto& e : ctx->pev)
        if (e) cudaEventDestroy(e);
    for (auto& e : ctx->phev)
        if (e) cudaEventDestroy(e);
    if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx->cm;
    delete ctx;
}

trplk_status trplk_info(const trplk_ctx* ctx, int64_t* n_local, int64_t* n_ghost, int* rank, int* nranks,
                        double* frob_a, int64_t* sell_bytes_a, int64_t* sell_bytes_b) {
    if (!ctx) return TRPLK_EINVAL;
    if (n_local) *n_local = ctx->n_loc;
    if (n_ghost) *n_ghost = ctx->n_ghost;
    if (rank) *rank = ctx->rank;
    if (nranks) *nranks = ctx->nranks;
    if (frob_a) *frob_a = ctx->normF;
    if (sell_bytes_a) *sell_bytes_a = ctx->sellA_bytes;
    if (sell_bytes_b) *sell_bytes_b = ctx->sellB_bytes;
    return TRPLK_OK;
}

int trplk_get_log(const trplk_ctx* ctx, int cap, int* t, int64_t* mv, double* theta_t, double* res, int* k,
                  int* nprev, double* thetas) {
    if (!ctx) return 0;
    const int n = std::min<int>(cap, (int)ctx->log.size());
    for (int i = 0; i < n; ++i) {
        const LogRec& L = ctx->log[i];
        if (t) t[i] = L.t;
        if (mv) mv[i] = L.mv;
        if (theta_t) theta_t[i] = L.theta_t;
        if (res) res[i] = L.res;
        if (k) k[i] = L.k;
        if (nprev) nprev[i] = L.nprev;
        if (thetas)
            for (int j = 0; j < ctx->log_ph; ++j) thetas[(size_t)i * ctx->log_ph + j] = L.thetas[j];
    }
    return n;
}

static trplk_status solve_impl(trplk_ctx* ctx, int p, int q, int l, double tol, double* evals, double* evecs,
                               double* resid, const trplk_options* optin, trplk_stats* stats) {
    trplk_options opt;
    trplk_options_default(&opt);
    if (optin) opt = *optin;
    const int ph = opt.restart_size > 0 ? opt.restart_size : p;
    const int m = q - ph - l;
    if (p < 1 || l < 0 || ph < p || m < 1 || !(tol > 0.0) || q > QMAX || ph + 1 > ctx->n_global ||
        opt.max_cycles < 1 || l > 16 || ph > 24) {
        ctx->err = "invalid solve arguments (need p>=1, l>=0, p<=p^<=24, m=q-p^-l>=1, q<=" +
                   std::to_string(QMAX) + ", tol>0, l<=16)";
        return TRPLK_EINVAL;
    }
    if (!evals || !resid) {
        ctx->err = "NULL output";
        return TRPLK_EINVAL;
    }
    if (opt.precond < 0 || opt.precond > 3 || (opt.precond >= 2 && opt.block > 1)) {
        ctx->err = "options.precond must be 0 (Jacobi), 1 (none), 2 (Jacobi of A - rho_i B) or 3 (IC(0)); "
                   "2 and 3 with block = 1";
        return TRPLK_EINVAL;
    }
    ctx->mfloor_solve = (opt.precond == 1 || opt.precond == 3) ? -1.0 : ctx->mfloor;  // IC(0): kernels apply I
    ctx->pmode = opt.precond;
    const int blk = opt.block > 1 ? opt.block : 1;
    if (blk > 1 && (blk > BC || ctx->hasB || ctx->nranks > 1)) {
        ctx->err = "options.block: 1..8, B = I and one rank on the device";
        return TRPLK_EINVAL;
    }
    const Sizes S{p, q, l, ph, m, opt.precond, blk};
    PhaseTimer pt("solve");
    ST(ensure_buffers(ctx, q, ph));
    if (ctx->pmode == 3) ST(ic0_setup(ctx));
    if (!ctx->hasB && std::max(l <= BC ? l : 0, blk > 1 ? blk : 0) > 0)
        ST(ensure_block_buffers(ctx, std::max(l <= BC ? l : 0, blk > 1 ? blk : 0)));
    pt.mark("buffers");
    ctx->log.clear();
    ctx->log_ph = ph;
    ctx->a_mv = ctx->b_mv = ctx->prec = ctx->inner = ctx->verify = ctx->draws = 0;
    ctx->model_bytes = 0.0;
    ctx->launches = 0;  // per-solve count (stats->kernel_launches)

    const double tau = opt.tol_mode == 1 ? tol * ctx->normF : tol;  // eq 5.1 vs Alg.1 step 12 (R8)
    const int64_t ld = ctx->ld;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, ctx->stream));

    Ctl& H = *ctx->ctl_h;
    ST(ctl_pull(ctx));
    const int p3_start = H.pass3_count;
    int cur = 0;
    trplk_status status = TRPLK_NOT_CONVERGED;
    // ---------------- Alg.1 steps 1-2: X = B-orthonormalised rand(n, p^) (R13)
    H.k = 0;
    H.flags = ~0u;
    H.t = 1;
    H.pass3 = 0;
    H.rho = 0.0;
    H.xprev_col = 0;
    for (int c = 0; c < ph; ++c) {
        double* xc = ctx->U[cur] + ld * c;
        launch_random(xc, ctx->n_loc, ctx->row_begin, ctx->n_global, opt.seed, 0, (uint64_t)c, ctx->stream);
        int tries = 0;
        for (;;) {
            H.k = c;
            H.flags = ~0u;
            H.pass3 = 0;
            ST(ctl_push(ctx));
            CgsSpec cs{};
            cs.x = xc;
            cs.V = ctx->U[cur];
            cs.kv = c;
            cs.k_nominal = c;
            cs.dest = ctx->U[cur];
            cs.dest_dyn = 1;
            cs.gate = F_CYCLE;
            cs.clear = F_CYCLE;
            cs.inc_k = 1;
            // orthogonalise a copy: dest column == source column, so route through w
            launch_copy_cols(xc, ld, ctx->w, ld, ctx->n_loc, 1, ctx->stream);
            cs.x = ctx->w;
            ST(cgs2(ctx, cs));
            ST(ctl_pull(ctx));
            if (ctx->hasB) ctx->b_mv += 2;
            if (H.flags & F_CYCLE) break;
            if (tries++ >= 3) {
                ctx->err = "start block: dependent columns after 3 random replacements";
                status = TRPLK_BREAKDOWN;
                goto finish;
            }
            launch_random(xc, ctx->n_loc, ctx->row_begin, ctx->n_global, opt.seed, 2, (uint64_t)ctx->draws++,
                          ctx->stream);
        }
    }
    {
        H.k = ph;
        H.flags = ~0u;
        H.pass3 = 0;
        ST(ctl_push(ctx));
        // W = A X (p^ matvecs), T0 = X^T W (full, symmetrised inside the eig), eig, rotate X and W
        for (int c = 0; c < ph; ++c) {
            ST(halo(ctx, ctx->U[cur] + ld * c));
            SdotsArgs a = sd_base(ctx);
            a.A = ctx->A;
            a.x = ctx->U[cur] + ld * c;
            a.out_mode = 1;
            a.out = ctx->Wtmp + ld * c;
            ST(run_sdots(ctx, a, 0));
            ctx->a_mv++;
        }
        for (int c = 0; c < ph; ++c) {
            SdotsArgs a = sd_base(ctx);
            a.x = ctx->Wtmp + ld * c;
            a.set1 = 3;
            a.U = ctx->U[cur];
            a.k1 = ph;
            a.dest1 = D_TCOL;
            a.tcol_fixed = c;
            ST(run_sdots(ctx, a, ph));
        }
        launch_eig(ctx->ctl, ctx->T, QMAX, ctx->Yg, QMAX, ph, ph, 0, ctx->stream);
        launch_rotate(ctx->U[cur], ld, ctx->n_loc, ctx->ctl, ph, ctx->Yg, QMAX, ph, ctx->U[1 - cur], ld, 0,
                      ctx->stream, ph);
        launch_rotate(ctx->Wtmp, ld, ctx->n_loc, ctx->ctl, ph, ctx->Yg, QMAX, ph, ctx->U[cur], ld, 0, ctx->stream, ph);
        CK(cudaGetLastError());
        cur = 1 - cur;  // X in U[cur], A X in U[1-cur]
        // r = A x_1 - theta_1 B x_1 from W (no matvec), u = M r
        ST(halo(ctx, ctx->U[cur]));
        SdotsArgs a = sd_base(ctx);
        a.A = ctx->A;
        if (ctx->hasB) a.B = ctx->B;
        a.x = ctx->U[cur];
        a.wext = ctx->U[1 - cur];
        a.out_mode = 4;
        a.uout = ctx->u;
        a.norm1 = 1;
        a.nslot1 = N_RES2;
        a.theta_idx = 0;
        ST(run_sdots(ctx, a, 0));
        if (ctx->pmode == 3) ST(ic0_apply(ctx, ctx->u, 0));
        if (ctx->hasB) ctx->b_mv++;
        ctx->prec++;
        // block (B1): seeds of targets 2 .. b_e from A X as well (no matvec)
        const int be0 = std::min(blk, std::min(ph, m));
        for (int i = 1; i < be0; ++i) {
            SdotsArgs e2 = a;
            e2.x = ctx->U[cur] + ld * i;
            e2.wext = ctx->U[1 - cur] + ld * i;
            e2.uout = ctx->sblk + ld * i;
            e2.nslot1 = N_AUX;
            e2.theta_idx = i;
            ST(run_sdots(ctx, e2, 0));
            ctx->prec++;
        }
        ST(ctl_pull(ctx));
        ctx->b_mv += ctx->hasB ? H.pass3_count - p3_start : 0;
        pt.mark("start block");
    }
    {
        int t = 1, nprev = 0, xprev = 0;
        double rho = H.theta[0];
        bool all_conv = false;
        int cyc = 0;
        int seed_tries = 0;
        std::vector<double> theta(q);
        int p3_prev = H.pass3_count;
        while (cyc < opt.max_cycles) {
            // -------- one outer cycle on the device
            H.k = ph;
            H.flags = ~0u;
            H.t = t;
            H.pass3 = 0;
            H.rho = rho;
            H.xprev_col = xprev;
            ST(ctl_push(ctx));
            static const bool ctrace = getenv("TRPLK_CYCLE_TRACE") != nullptr;  // GPU busy vs idle per cycle
            if (ctrace) {
                if (!ctx->ctev[0]) {
                    CK(cudaEventCreate(&ctx->ctev[0]));
                    CK(cudaEventCreate(&ctx->ctev[1]));
                }
                CK(cudaEventRecord(ctx->ctev[0], ctx->stream));
            }
            const int be = blk > 1 ? std::min(blk, std::min(ph - t + 1, m)) : 1;
            const int extras = (be > 1 && cyc > 0) ? 1 : 0;  // cycle 1's came from A X at start-up
            ST(run_cycle(ctx, S, cur, nprev, t, xprev, opt.use_graphs != 0, be, extras));
            if (extras) {
                ctx->a_mv += be - 1;
                ctx->prec += be - 1;
            }
            if (ctrace) CK(cudaEventRecord(ctx->ctev[1], ctx->stream));
            ST(ctl_pull(ctx));
            if (ctrace) {
                float cms = 0.f;
                CK(cudaEventElapsedTime(&cms, ctx->ctev[0], ctx->ctev[1]));
                ctx->ctrace_busy += cms;
                ctx->ctrace_n++;
            }
            if (!(H.flags & F_CYCLE)) {  // seed in span(X): inject a stream-2 random vector (R16)
                if (seed_tries++ >= 3) {
                    ctx->err = "seed vector dependent after 3 random replacements";
                    status = TRPLK_BREAKDOWN;
                    break;
                }
                launch_random(ctx->u, ctx->n_loc, ctx->row_begin, ctx->n_global, opt.seed, 2, (uint64_t)ctx->draws++,
                              ctx->stream);
                continue;
            }
            seed_tries = 0;
            ++cyc;
            const int kr = H.k_rr;
            int appended = 0;
            for (int jj = 0; jj < nprev; ++jj) appended += (H.flags & (F_KCOL0 << jj)) ? 1 : 0;
            const int G = kr - ph - appended;  // inner Lanczos columns built (R16: may stop early)
            const int ncgs = (H.flags & F_INNER) ? G - 1 : G;
            ctx->a_mv += G + appended + 1;      // m + |X^prev| + residual
            ctx->inner += G;
            ctx->prec += ncgs + 1;
            if (ctx->hasB) ctx->b_mv += 2 + 3 * ncgs + 2 * nprev + 1 + (H.pass3_count - p3_prev);
            p3_prev = H.pass3_count;
            if (ctx->prof_on) {  // live cycle-phase profile
                for (int i = 0; i < 6; ++i) {
                    float pm = 0.f;
                    CK(cudaEventElapsedTime(&pm, ctx->phev[i], ctx->phev[i + 1]));
                    ctx->phase_ms[i] += pm;
                }
                ctx->phase_count++;
            }
            if (ctx->prof_on && !(blk > 1)) {  // live inner-step profile (events inside the cycle; Alg. 1 path)
                const int jmid = std::max(1, std::min(m - 1, m / 2));
                if (m >= 2 && G > jmid) {
                    float e[3];
                    CK(cudaEventElapsedTime(&e[0], ctx->pev[0], ctx->pev[1]));
                    CK(cudaEventElapsedTime(&e[1], ctx->pev[1], ctx->pev[2]));
                    CK(cudaEventElapsedTime(&e[2], ctx->pev[2], ctx->pev[3]));
                    const bool fused = small_path(ctx, S) || grid_path(ctx, S);
                    const double n = (double)ctx->n_loc, k = (double)(ph + jmid);
                    // matrix bytes of the device format (DIA: 8 ndiag n; SELL: 12 per slot + slice ptrs)
                    const double spA = (double)ctx->sellA_bytes, spB = (double)ctx->sellB_bytes;
                    double b1, b2;
                    const double spA1 = kern_reads_diac(ctx->prof_kern[0]) ? (double)ctx->sellA_bytes_dc : spA;
                    if (ctx->hasB) {
                        b1 = spA + spB + 8.0 * n * (k + 2);
                        b2 = 2 * (spB + 8.0 * n * (k + 1)) + 8.0 * n * (k + 2);
                    } else {
                        b1 = spA1 + 8.0 * n * (k + 2);  // A (as the launched K1 reads it), g, U(:,1:k), w
                        b2 = 8.0 * n * (k + 2);        // U, w, w'
                    }
                    const double b3 = 8.0 * n * (k + 2);  // U, w', g_{j+1}
                    double bb[3] = {b1, b2, b3};
                    if (ctx->prof_fused) {
                        // slots [K3 of step jmid + K1 of step jmid+1, K2, -]: the fused kernel moves the
                        // FINAL's bytes and the K1's A and w (its U and g re-reads come from L2)
                        const float ek2 = e[0];
                        e[0] = e[1];
                        e[1] = ek2;
                        e[2] = 0.0f;
                        bb[0] = b3 + (double)ctx->sellA_bytes_dc + 8.0 * n;
                        bb[1] = b2;
                        bb[2] = 0.0;
                    }
                    if (fused) {  // one launch for all G steps: its time, the bytes of all G steps
                        double tot = 0.0;
                        for (int j = 1; j <= G; ++j) {
                            const double kj = (double)(ph + j);
                            tot += (double)ctx->sellA_bytes + 8.0 * n * (kj + 2);
                            if (j < m) tot += 2 * 8.0 * n * (kj + 2);
                        }
                        bb[0] = tot;
                        bb[1] = bb[2] = 0.0;
                        e[1] = e[2] = 0.0f;
                    }
                    for (int i = 0; i < 3; ++i) {
                        ctx->prof_ms[i] += e[i];
                        ctx->prof_bytes[i] += bb[i];
                    }
                    ctx->prof_count++;
                }
            }
            for (int i = 0; i < kr; ++i) theta[i] = H.theta[i];
            double res = std::sqrt(H.nrm[N_RES2]);
            LogRec L;
            L.t = t;
            L.theta_t = theta[t - 1];
            L.res = res;
            L.k = kr;
            L.nprev = appended;
            L.thetas.assign(theta.begin(), theta.begin() + ph);
            // Alg.1 step 10 (before the RR): X^prev <- X(:, t : min(t+l-1, p)) of this cycle's basis
            int xcol = t - 1;
            int nnew = std::max(0, std::min(t + l - 1, p) - t + 1);
            // steps 12-14: soft locking (R7)
            while (res <= tau) {
                t += 1;
                if (nnew > 0) {
                    xcol++;
                    nnew--;
                }
                if (t > p) {
                    all_conv = true;
                    break;
                }
                H.t = t;
                ST(ctl_push(ctx));
                ST(residual(ctx, ctx->U[1 - cur] + ld * (t - 1), 0, t - 1, ctx->u, 0));
                ctx->a_mv++;
                ctx->prec++;
                if (ctx->hasB) ctx->b_mv++;
                ST(ctl_pull(ctx));
                res = std::sqrt(H.nrm[N_RES2]);
                if (opt.lock_mode == 0) break;
            }
            L.mv = ctx->a_mv;
            ctx->log.push_back(L);
            cur = 1 - cur;
            nprev = nnew;
            xprev = xcol;
            if (all_conv) {
                // final verification of all p pairs (R9)
                int first_fail = -1;
                for (int i = 0; i < p; ++i) {
                    ST(residual(ctx, ctx->U[cur] + ld * i, 0, i, ctx->u2, 0));
                    ctx->verify++;
                    ctx->a_mv++;
                    if (ctx->hasB) ctx->b_mv++;
                    ST(ctl_pull(ctx));
                    resid[i] = std::sqrt(H.nrm[N_RES2]);
                    if (resid[i] > tau && first_fail < 0) {
                        first_fail = i;
                        CK(cudaMemcpyAsync(ctx->u, ctx->u2, 8 * ctx->n_loc, cudaMemcpyDeviceToDevice, ctx->stream));
                    }
                }
                if (first_fail < 0) {
                    status = TRPLK_OK;
                    break;
                }
                t = first_fail + 1;
                all_conv = false;
            }
            rho = theta[t - 1];
            H.t = t;
        }
        if (status != TRPLK_OK) {
            for (int i = 0; i < p; ++i) {
                ST(residual(ctx, ctx->U[cur] + ld * i, 0, i, nullptr, 0));
                ctx->verify++;
                ctx->a_mv++;
                if (ctx->hasB) ctx->b_mv++;
                ST(ctl_pull(ctx));
                resid[i] = std::sqrt(H.nrm[N_RES2]);
            }
        }
        if (stats) stats->cycles = cyc;
    }
finish:
    pt.mark("cycles");
    if (ctx->ctrace_n) {
        fprintf(stderr, "[cycle trace] %d cycles, graph time %.3f ms (%.1f us per cycle)\n", ctx->ctrace_n,
                ctx->ctrace_busy, 1e3 * ctx->ctrace_busy / ctx->ctrace_n);
        ctx->ctrace_busy = 0.0;
        ctx->ctrace_n = 0;
    }
    if (ctx->gtrace) {  // TRPLK_GRID_TRACE: phase durations (us) of the last grid-path cycle, per step
        unsigned long long tr[64];
        cudaStreamSynchronize(ctx->stream);
        cudaMemcpy(tr, ctx->gtrace, sizeof(tr), cudaMemcpyDeviceToHost);
        for (int j = 0; j < 8 && tr[j * 8 + 6] > tr[j * 8]; ++j)
            fprintf(stderr, "[grid step %d] p1 %.2f red %.2f p2 %.2f red %.2f fin %.2f sync %.2f total %.2f\n", j + 1,
                    (tr[j * 8 + 1] - tr[j * 8]) * 1e-3, (tr[j * 8 + 2] - tr[j * 8 + 1]) * 1e-3,
                    (tr[j * 8 + 3] - tr[j * 8 + 2]) * 1e-3, (tr[j * 8 + 4] - tr[j * 8 + 3]) * 1e-3,
                    (tr[j * 8 + 5] - tr[j * 8 + 4]) * 1e-3, (tr[j * 8 + 6] - tr[j * 8 + 5]) * 1e-3,
                    (tr[j * 8 + 6] - tr[j * 8]) * 1e-3);
    }
    for (int i = 0; i < p; ++i) evals[i] = H.theta[i];
    if (evecs) {
        CK(cudaMemcpy2DAsync(evecs, 8 * ctx->n_loc, ctx->U[cur], 8 * ld, 8 * ctx->n_loc, p, cudaMemcpyDefault,
                             ctx->stream));
    }
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    pt.mark("d2h");
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (stats) {
        stats->a_matvecs = ctx->a_mv;
        stats->b_matvecs = ctx->b_mv;
        stats->precond_applies = ctx->prec;
        stats->inner_steps = ctx->inner;
        stats->verify_matvecs = ctx->verify;
        stats->random_draws = ctx->draws;
        stats->status = status;
        stats->solve_seconds = ms * 1e-3;
        stats->model_bytes = ctx->model_bytes;
        stats->kernel_launches = ctx->launches;
    }
    return status;
}

trplk_status trplk_solve(trplk_ctx* ctx, int p, int max_basis, int k_plus, double tol, double* eigenvalues,
                         double* eigenvectors, double* residual_norms, const trplk_options* opt, trplk_stats* stats) {
    if (!ctx) return TRPLK_EINVAL;
    const int f3 = ctx->force3;
    const int f3_solve = f3 | ((opt && (opt->debug_checks & 2)) ? 1 : 0);
    if (f3_solve != f3) set_force3(ctx, f3_solve);
    enter_stream(ctx);
    const trplk_status st =
        solve_impl(ctx, p, max_basis, k_plus, tol, eigenvalues, eigenvectors, residual_norms, opt, stats);
    leave_stream(ctx);
    if (f3_solve != f3) set_force3(ctx, f3);
    return st;
}

trplk_status trplk_set_debug(trplk_ctx* ctx, int flags) {
    if (!ctx) return TRPLK_EINVAL;
    set_force3(ctx, flags & 1);
    const int g = (flags & 2) ? 1 : -1;
    if (g != ctx->grid_on) {  // the captured cycle graphs hold the other inner-loop kernels
        ctx->grid_on = g;
        for (auto& e : ctx->graphs) cudaGraphExecDestroy(e.second.exec);
        ctx->graphs.clear();
    }
    return TRPLK_OK;
}

// ------------------------------------------------------------ PL+1 (Algorithm 2, NEXT-1)
// Readings P1-P6; the oracle's orc_pl1_solve follows the same steps.
// Q = [x, g_1..g_m, p] lives in one block of m+2 columns (ld = ctx->ld) so that the Gram
// columns Q^T (A q_j), Q^T (B q_j) come from the fused dot kernel (set1 = x, D_TCOL) and the
// combination G w from the DMMA rotation; A Q and B Q are kept as blocks of the same shape.
static trplk_status pl1_impl(trplk_ctx* ctx, int m, double tol, int variant, int use_precond, int max_iter,
                             uint64_t seed, const double* x0, double* rho_out, double* resid_out, double* x_out,
                             int log_cap, double* log_rho, double* log_res, double* log_conj, int* log_len,
                             trplk_stats* stats) {
    const int64_t n = ctx->n_loc, ld = ctx->ld;
    const int nc = m + 2;
    cudaStream_t st = ctx->stream;
    double *Q, *AQ, *BQ, *r, *xt, *g, *pt, *v, *tmp, *Hq, *Sq, *part;
    Pl1Dev* dv;
    ST(dalloc(ctx, &Q, (size_t)ld * nc));
    ST(dalloc(ctx, &AQ, (size_t)ld * nc));
    BQ = Q;
    if (ctx->hasB) ST(dalloc(ctx, &BQ, (size_t)ld * nc));
    for (double** b : {&r, &xt, &g, &pt, &v, &tmp}) ST(dalloc(ctx, b, (size_t)ld));
    ST(dalloc(ctx, &Hq, (size_t)nc * nc));
    ST(dalloc(ctx, &Sq, (size_t)nc * nc));
    ST(dalloc(ctx, &part, (size_t)PL1_PART));
    ST(dalloc(ctx, &dv, 1));
    CK(cudaMemsetAsync(Q, 0, 8 * (size_t)ld * nc, st));
    CK(cudaMemsetAsync(AQ, 0, 8 * (size_t)ld * nc, st));
    if (ctx->hasB) CK(cudaMemsetAsync(BQ, 0, 8 * (size_t)ld * nc, st));
    for (double* b : {r, xt, g, pt, v, tmp}) CK(cudaMemsetAsync(b, 0, 8 * (size_t)ld, st));
    CK(cudaMemsetAsync(dv, 0, sizeof(Pl1Dev), st));
    double* x = Q;
    double* G = Q + ld;
    double* p = Q + ld * (m + 1);
    double *Ax = AQ, *AG = AQ + ld, *Ap = AQ + ld * (m + 1);
    double *Bx = BQ, *BG = BQ + ld, *Bp = BQ + ld * (m + 1);
    double* sc = dv->sc;
    int64_t amv = 0, bmv = 0;
    ctx->launches = 0;
    ctx->model_bytes = 0.0;
    const double vb = 8.0 * (double)n;  // bytes of one n-vector (DESIGN.md byte model)
    auto spmv = [&](bool useB, const double* xin, double* out) -> trplk_status {
        ST(halo(ctx, xin));
        SdotsArgs a = sd_base(ctx);
        a.A = useB ? ctx->B : ctx->A;
        a.x = xin;
        a.out_mode = 1;
        a.out = out;
        ST(run_sdots(ctx, a, 0));
        if (useB) bmv++;
        else amv++;
        return TRPLK_OK;
    };
    // several ranks: local sums into red_local (same slots), allgather, rank-ordered sums into sc
    auto dots = [&](std::initializer_list<std::pair<std::pair<const double*, const double*>, int>> L)
        -> trplk_status {
        Pl1Pairs P{};
        for (auto& e : L) {
            P.a[P.np] = e.first.first;
            P.b[P.np] = e.first.second;
            P.slot[P.np] = e.second;
            P.np++;
        }
        ctx->launches += 2;
        ctx->model_bytes += 2.0 * vb * P.np;
        if (ctx->nranks == 1) {
            pl1_dots(P, n, part, sc, st);
            return TRPLK_OK;
        }
        pl1_dots(P, n, part, ctx->red_local, st);
        CM(ctx->cm->allgather(ctx->red_local, ctx->red_all, 16, 8, st));
        pl1_dots_ranks(P, ctx->red_all, ctx->nranks, 16, sc, st);
        ctx->launches += 1;
        return TRPLK_OK;
    };
    double h[16];
    auto read_sc = [&]() -> trplk_status {
        CK(cudaMemcpyAsync(h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return TRPLK_OK;
    };
    Ctl& H = *ctx->ctl_h;
    ST(ctl_pull(ctx));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, st));
    // step 2: x_0 (P6), ||x_0||_B = 1, rho_0, r_0
    if (x0) CK(cudaMemcpyAsync(x, x0, 8 * (size_t)n, cudaMemcpyDefault, st));
    else launch_random(x, n, ctx->row_begin, ctx->n_global, seed, 3, 0, st);
    const double* Bxin = x;
    if (ctx->hasB) {
        ST(spmv(true, x, tmp));
        Bxin = tmp;
    }
    ST(dots({{{x, Bxin}, 0}}));
    pl1_scale(n, x, sc + 0, x, st);
    ST(spmv(false, x, Ax));
    if (ctx->hasB) ST(spmv(true, x, Bx));
    ST(dots({{{x, Ax}, 1}, {{x, Bx}, 2}}));
    pl1_res(n, Ax, Bx, sc + 1, sc + 2, r, st);
    ST(dots({{{r, r}, 3}}));
    pl1_shift_rho(dv, sc, st);  // rho_cur = rho_0
    // quasi-optimality diagnostic (P7, Def. defnglbopt): B-orthonormal basis Z
    // of U_k = span{x_0} + span{g_0..g_{k-1}} and Hz = Z^T A Z, extended between iterations
    // (eager launches outside the iteration graphs; matvecs, launches and bytes not counted)
    const int qcap = std::min(ctx->qopt_cap, QMAX);
    double *Z = nullptr, *Hz = nullptr, *Azq = nullptr, *qstar = nullptr;
    int dq = 0;
    ctx->qopt_star.clear();
    ctx->qopt_rho.clear();
    ctx->qopt_dim.clear();
    auto gram_col = [&](const double* Az, int col) -> trplk_status {  // Hz(0:col, col) = Z^T (A z_col)
        SdotsArgs a = sd_base(ctx);
        a.x = Az;
        a.set1 = 3;
        a.U = Z;
        a.k1 = col + 1;
        a.dest1 = D_TCOL;
        a.tcol_fixed = col;
        a.T = Hz;
        a.ldT = QMAX;
        return run_sdots(ctx, a, col + 1, false);
    };
    if (qcap > 0) {
        ST(dalloc(ctx, &Z, (size_t)ld * qcap));
        ST(dalloc(ctx, &Hz, (size_t)QMAX * QMAX));
        ST(dalloc(ctx, &Azq, (size_t)ld));
        ST(dalloc(ctx, &qstar, (size_t)qcap));
        CK(cudaMemsetAsync(Z, 0, 8 * (size_t)ld * qcap, st));
        CK(cudaMemsetAsync(Hz, 0, 8 * (size_t)QMAX * QMAX, st));
        CK(cudaMemsetAsync(Azq, 0, 8 * (size_t)ld, st));
        CK(cudaMemcpyAsync(Z, x, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));  // U_0 = span{x_0}
        const double mb = ctx->model_bytes;
        const int64_t la = ctx->launches;
        ST(gram_col(Ax, 0));
        ctx->model_bytes = mb;
        ctx->launches = la;
        dq = 1;
        ctx->qopt_dim.push_back(1);
    }
    ST(read_sc());
    double rho = h[1] / h[2], res = std::sqrt(h[3]);
    double rho_prev = rho, conj_next = 0.0;
    int has_p = 0, k = 0;
    trplk_status status = TRPLK_NOT_CONVERGED;
    int nlog = 0;
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    double gbytes[2] = {0.0, 0.0};
    int64_t glaunch[2] = {0, 0}, gamv[2] = {0, 0}, gbmv[2] = {0, 0};
    for (k = 0;; ++k) {
        if (k < qcap) ctx->qopt_rho.push_back(rho);
        ctx->qopt_last = rho;
        if (k < log_cap) {
            if (log_rho) log_rho[k] = rho;
            if (log_res) log_res[k] = res;
            if (log_conj) log_conj[k] = conj_next;
            nlog = k + 1;
        }
        if (res <= tol) {  // step 3
            status = TRPLK_OK;
            break;
        }
        if (k >= max_iter) break;
        auto issue_iter = [&](int has_p) -> trplk_status {
        // step 4 (P1): G_k, each new vector CGS2-orthogonalised against the previous ones.  The
        // CGS2 kernels append at column ctl->k and clear F_CYCLE on a breakdown (R16), which
        // gates the remaining CGS2 launches of the block: no host round trip inside step 4.
        pl1_begin(ctx->ctl, st);
        for (int j = 0; j < m; ++j) {
            if (j == 0) pl1_prec(ctx->A, ctx->B, n, ctx->sigma, ctx->mfloor, r, r, nullptr, v, use_precond, st);
            else pl1_prec(ctx->A, ctx->B, n, ctx->sigma, ctx->mfloor, AG + ld * (j - 1), BG + ld * (j - 1), &dv->rho_cur, v,
                          use_precond, st);
            ctx->launches++;
            ctx->model_bytes += (j == 0 ? 2.0 : 3.0) * vb + (double)ctx->sellA_bytes / 8.0;  // z, s, v + diag
            CgsSpec cs{};
            cs.x = v;
            cs.V = G;
            cs.kv = -1;
            cs.k_nominal = j;
            cs.dest = G;
            cs.dest_dyn = 1;
            cs.gate = F_CYCLE;
            cs.clear = F_CYCLE;
            cs.inc_k = 1;
            ST(cgs2(ctx, cs));
            ST(spmv(false, G + ld * j, AG + ld * j));  // counted for the columns actually built below
            if (ctx->hasB) ST(spmv(true, G + ld * j, BG + ld * j));
        }
        // step 5 (P2, P3): Gram columns of Q_k = [x_k, G_k, p_{k-1}], reduced pencil, eig.  Columns
        // past a breakdown hold finite stale data; the reduction ignores them, w weighs them 0.
        if (has_p) {
            ST(spmv(false, p, Ap));
            if (ctx->hasB) ST(spmv(true, p, Bp));
        }
        const bool gram1 = ctx->nranks == 1 && pl1_gram(nc, Q, AQ, ctx->hasB ? BQ : nullptr, ld, n, part, Hq, Sq, st);
        if (gram1) {
            ctx->launches += 2;
            ctx->model_bytes += vb * nc * (ctx->hasB ? 3.0 : 2.0);
        }
        for (int j = 0; j < nc && !gram1; ++j) {
            if (j == m + 1 && !has_p) continue;
            for (int which = 0; which < 2; ++which) {
                SdotsArgs a = sd_base(ctx);
                a.x = (which == 0 ? AQ : BQ) + ld * j;
                a.set1 = 3;
                a.U = Q;
                a.k1 = nc;
                a.dest1 = D_TCOL;
                a.tcol_fixed = j;
                a.T = which == 0 ? Hq : Sq;
                a.ldT = nc;
                ST(run_sdots(ctx, a, nc));
            }
        }
        pl1_reduce(Hq, Sq, nc, m, ctx->ctl, has_p, ctx->T, QMAX, dv, st);
        launch_eig(ctx->ctl, ctx->T, QMAX, ctx->Yg, QMAX, 0, 0, 0, st);  // k = ctl->k = nq
        pl1_back(ctx->Yg, QMAX, m, dv, st);
        ctx->launches += 3;
        // step 6 (P5): g_k = G w(2:m+1), x~ = w(1) x + g + w(m+2) p, x_{k+1}, rho_{k+1}, r_{k+1}
        launch_rotate(G, ld, n, ctx->ctl, m, dv->w + 1, PL1_QP, 1, g, ld, 0, st, m);
        pl1_xt(n, x, g, p, dv, m, xt, st);
        ctx->model_bytes += vb * (m + 1) + 4.0 * vb + 2.0 * vb + 3.0 * vb;  // rotation, xt, scale, res
        const double* Bxt = xt;
        if (ctx->hasB) {
            ST(spmv(true, xt, tmp));
            Bxt = tmp;
        }
        ST(dots({{{xt, Bxt}, 0}}));
        pl1_scale(n, xt, sc + 0, x, st);
        ST(spmv(false, x, Ax));
        if (ctx->hasB) ST(spmv(true, x, Bx));
        ST(dots({{{x, Ax}, 1}, {{x, Bx}, 2}}));
        pl1_res(n, Ax, Bx, sc + 1, sc + 2, r, st);
        ST(dots({{{r, r}, 3}}));
        ctx->launches += 5;
        // step 7 (P4): p~_k and p_k
        const bool conj = has_p && variant == 0;
        (void)conj;
        if (!has_p) {
            CK(cudaMemcpyAsync(pt, g, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
        } else if (variant == 1) {
            pl1_pt(n, g, p, sc + 4, sc + 5, 0.0, 1, dv, m, pt, st);
        } else {
            pl1_dvec(n, Ap, Bp, dv, v, st);  // d = (A - rho_{k-1} B) p_{k-1}
            ctx->model_bytes += 3.0 * vb;
            ST(dots({{{v, g}, 4}, {{v, p}, 5}}));
            pl1_pt(n, g, p, sc + 4, sc + 5, 1e-14 * ctx->normF, 0, dv, m, pt, st);
        }
        const double* Bpt = pt;
        ctx->model_bytes += 3.0 * vb + 2.0 * vb;  // p~, scale
        if (ctx->hasB) {
            ST(spmv(true, pt, tmp));
            Bpt = tmp;
        }
        ST(dots({{{pt, Bpt}, 6}}));
        pl1_scale_p(n, pt, sc + 6, p, dv, st);
        if (conj) ST(dots({{{v, p}, 7}}));
        pl1_shift_rho(dv, sc, st);
        ctx->launches += 1;
            return TRPLK_OK;
        };
        // one CUDA graph per has_p (the only host-side branch of an iteration); counters and
        // byte model recorded at capture and re-added per launch
        const int gi = has_p ? 1 : 0;
        if (ctx->loopback) {  // loopback exchanges are host rendezvous: eager only
            ST(issue_iter(has_p));
        } else if (!gexec[gi]) {
            const double mb0 = ctx->model_bytes;
            const int64_t l0 = ctx->launches, a0 = amv, b0 = bmv;
            cudaGraph_t graph;
            CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            trplk_status cs_ = issue_iter(has_p);
            cudaError_t e = cudaStreamEndCapture(st, &graph);
            if (cs_ != TRPLK_OK) return cs_;
            if (e != cudaSuccess) {
                ctx->err = std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e);
                return TRPLK_ECUDA;
            }
            CK(cudaGraphInstantiate(&gexec[gi], graph, 0));
            cudaGraphDestroy(graph);
            gbytes[gi] = ctx->model_bytes - mb0;
            glaunch[gi] = ctx->launches - l0;
            gamv[gi] = amv - a0;
            gbmv[gi] = bmv - b0;
            ctx->model_bytes = mb0;
            ctx->launches = l0;
            amv = a0;
            bmv = b0;
        }
        if (!ctx->loopback) {
            CK(cudaGraphLaunch(gexec[gi], st));
            ctx->model_bytes += gbytes[gi];
            ctx->launches += glaunch[gi];
            amv += gamv[gi];
            bmv += gbmv[gi];
        }
        // the one host round trip of the iteration: scalars, step-5 status, G_k width, CGS2 passes
        int info[4];
        CK(cudaMemcpyAsync(h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(info, &dv->nq, sizeof(info), cudaMemcpyDeviceToHost, st));
        const int p3 = H.pass3_count;
        ST(ctl_pull(ctx));
        const int mg = info[2];
        if (ctx->hasB) bmv += 2 * std::min(mg + 1, m) + (H.pass3_count - p3) - (m - mg);  // B SpMVs of unbuilt columns
        amv -= (m - mg);  // SpMVs of columns past a breakdown are not the algorithm's
        if (info[1] >= 0) {
            amv -= 1;  // the step-6 product of the discarded iterate
            ctx->err = "PL+1: Q_k^T B Q_k not positive definite on [x_k, G_k] (P3)";
            status = TRPLK_BREAKDOWN;
            break;
        }
        conj_next = (has_p && variant == 0 && info[3]) ? h[7] / ctx->normF : 0.0;
        has_p = info[3];
        rho_prev = rho;
        rho = h[1] / h[2];
        res = std::sqrt(h[3]);
        if (k + 1 < qcap) {  // P7: U_{k+1} = U_k + span{g_k}; g_k dropped on a CGS2 breakdown (R16)
            const double mb = ctx->model_bytes;
            const int64_t la = ctx->launches;
            const int brk0 = H.brk;
            CgsSpec cs{};
            cs.x = g;
            cs.V = Z;
            cs.kv = dq;
            cs.k_nominal = dq;
            cs.dest = Z + ld * dq;
            cs.dest_dyn = 0;
            cs.gate = 0;
            cs.clear = 0;
            cs.inc_k = 0;
            ST(cgs2(ctx, cs));
            ST(ctl_pull(ctx));
            if (H.brk == brk0) {
                ST(halo(ctx, Z + ld * dq));
                SdotsArgs a = sd_base(ctx);
                a.A = ctx->A;
                a.x = Z + ld * dq;
                a.out_mode = 1;
                a.out = Azq;
                ST(run_sdots(ctx, a, 0, false));
                ST(gram_col(Azq, dq));
                ++dq;
            }
            ctx->qopt_dim.push_back(dq);
            ctx->model_bytes = mb;
            ctx->launches = la;
        }
    }
    if (qcap > 0) {  // rho(y*_k) = lowest eigenvalue of the leading dim(U_k) block of Hz (P7)
        const int nq = (int)ctx->qopt_dim.size();
        pl1_qmirror(Hz, QMAX, dq, st);
        for (int j = 0; j < nq; ++j) {
            const int d = ctx->qopt_dim[j];
            if (j > 0 && d == ctx->qopt_dim[j - 1]) {
                CK(cudaMemcpyAsync(qstar + j, qstar + j - 1, 8, cudaMemcpyDeviceToDevice, st));
            } else if (d == 1) {
                CK(cudaMemcpyAsync(qstar + j, Hz, 8, cudaMemcpyDeviceToDevice, st));
            } else {
                launch_eig(ctx->ctl, Hz, QMAX, ctx->Yg, QMAX, 0, d, 0, st);
                CK(cudaMemcpyAsync(qstar + j, &ctx->ctl->theta[0], 8, cudaMemcpyDeviceToDevice, st));
            }
        }
        ctx->qopt_star.resize(nq);
        CK(cudaMemcpyAsync(ctx->qopt_star.data(), qstar, 8 * (size_t)nq, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        ctx->qopt_rho.resize(std::min(ctx->qopt_rho.size(), (size_t)nq));
        for (void* b : {(void*)Z, (void*)Hz, (void*)Azq, (void*)qstar}) dev_free(ctx, b);
    }
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (auto& ge : gexec)
        if (ge) cudaGraphExecDestroy(ge);
    if (x_out) CK(cudaMemcpyAsync(x_out, x, 8 * (size_t)n, cudaMemcpyDefault, st));
    CK(cudaStreamSynchronize(st));
    ctx->qopt_last = rho;
    if (rho_out) *rho_out = rho;
    if (resid_out) *resid_out = res;
    if (log_len) *log_len = nlog;
    if (stats) {
        memset(stats, 0, sizeof(*stats));
        stats->a_matvecs = amv;
        stats->b_matvecs = bmv;
        stats->cycles = k;
        stats->status = status;
        stats->solve_seconds = ms * 1e-3;
        stats->kernel_launches = ctx->launches;
        stats->model_bytes = ctx->model_bytes;
    }
    for (void* b : {(void*)Q, (void*)AQ, (void*)r, (void*)xt, (void*)g, (void*)pt, (void*)v, (void*)tmp, (void*)Hq,
                    (void*)Sq, (void*)part, (void*)dv})
        dev_free(ctx, b);
    if (ctx->hasB) dev_free(ctx, BQ);
    return status;
}

trplk_status trplk_pl1_solve(trplk_ctx* ctx, int m, double tol, int variant, int use_precond, int max_iter,
                             uint64_t seed, const double* x0, double* rho, double* resid, double* x_out,
                             int log_cap, double* log_rho, double* log_res, double* log_conj, int* log_len,
                             trplk_stats* stats) {
    if (!ctx) return TRPLK_EINVAL;
    if (m < 1 || m > 32 || !(tol > 0.0) || max_iter < 0 || (variant != 0 && variant != 1)) {
        ctx->err = "PL+1: needs 1 <= m <= 32, tol > 0, max_iter >= 0, variant 0/1";
        return TRPLK_EINVAL;
    }
    enter_stream(ctx);
    const trplk_status s = pl1_impl(ctx, m, tol, variant, use_precond, max_iter, seed, x0, rho, resid, x_out,
                                    log_cap, log_rho, log_res, log_conj, log_len, stats);
    leave_stream(ctx);
    return s;
}

trplk_status trplk_pl1_set_qopt(trplk_ctx* ctx, int cap) {
    if (!ctx) return TRPLK_EINVAL;
    if (cap < 0 || cap > QMAX) {
        ctx->err = "PL+1 quasi-optimality diagnostic: needs 0 <= cap <= 64";
        return TRPLK_EINVAL;
    }
    ctx->qopt_cap = cap;
    return TRPLK_OK;
}

int trplk_pl1_get_qopt(const trplk_ctx* ctx, int cap, double lambda1, double* rho_star, int* dim, double* ratio) {
    if (!ctx) return 0;
    const int n = std::min<int>(cap, (int)std::min(ctx->qopt_star.size(), ctx->qopt_rho.size()));
    if (n <= 0) return 0;
    const double lam = std::isnan(lambda1) ? ctx->qopt_last : lambda1;
    for (int j = 0; j < n; ++j) {
        if (rho_star) rho_star[j] = ctx->qopt_star[j];
        if (dim) dim[j] = ctx->qopt_dim[j];
        if (ratio) {
            const double den = ctx->qopt_rho[j] - lam;
            ratio[j] = den > 0.0 ? (ctx->qopt_rho[j] - ctx->qopt_star[j]) / den : NAN;
        }
    }
    return n;
}

// ------------------------------------------------------------ kernel-level entry points
static trplk_status kprep(trplk_ctx* ctx, int k) {
    if (!ctx) return TRPLK_EINVAL;
    if (k < 0 || k > QMAX) {
        ctx->err = "k out of range";
        return TRPLK_EINVAL;
    }
    enter_stream(ctx);
    Ctl& H = *ctx->ctl_h;
    H.k = k;
    H.flags = ~0u;
    H.t = 1;
    H.pass3 = 0;
    H.xprev_col = 0;
    return ctl_push(ctx);
}

trplk_status trplk_k_spmv(trplk_ctx* ctx, int which, const double* x, double* y) {
    ST(kprep(ctx, 0));
    if (which == 1 && !ctx->hasB) {
        ctx->err = "no B matrix";
        return TRPLK_EINVAL;
    }
    SdotsArgs a = sd_base(ctx);
    a.A = which == 1 ? ctx->B : ctx->A;
    a.x = x;
    a.out_mode = 1;
    a.out = y;
    ST(run_sdots(ctx, a, 0));
    CK(cudaStreamSynchronize(ctx->stream));
    return TRPLK_OK;
}

trplk_status trplk_k_step1(trplk_ctx* ctx, const double* U, int64_t ldu, int k, const double* g, double rho,
                           double* w, double* tcol, double* h1, double* wnorm2) {
    ST(kprep(ctx, k));
    if (ldu < ctx->n_loc || k < 1) {
        ctx->err = "bad ldu or k";
        return TRPLK_EINVAL;
    }
    ctx->ctl_h->rho = rho;
    ST(ctl_push(ctx));
    SdotsArgs a = sd_base(ctx);
    a.A = ctx->A;
    a.x = g;
    a.U = U;
    a.ldu = ldu;
    a.k_from_ctl = 1;
    a.set1 = 1;
    a.dest1 = D_TCOL;
    a.out_mode = 2;
    a.out = w;
    if (ctx->hasB) {
        a.B = ctx->B;
    } else {
        a.set2 = 2;
        a.dest2 = D_H0 + 0;
        a.norm1 = 1;
        a.nslot1 = N_IN2;
    }
    ST(run_sdots(ctx, a, k));
    if (ctx->hasB) {
        ST(halo(ctx, w));
        SdotsArgs b = sd_base(ctx);
        b.A = ctx->B;
        b.x = w;
        b.U = U;
        b.ldu = ldu;
        b.k1 = k;
        b.set1 = 1;
        b.norm1 = 2;
        b.dest1 = D_H0 + 0;
        b.nslot1 = N_IN2;
        ST(run_sdots(ctx, b, k));
    }
    ST(ctl_pull(ctx));
    if (tcol) CK(cudaMemcpy(tcol, ctx->T + (size_t)(k - 1) * QMAX, 8 * (size_t)k, cudaMemcpyDeviceToHost));
    if (h1) memcpy(h1, ctx->ctl_h->h[0], 8 * (size_t)k);
    if (wnorm2) *wnorm2 = ctx->ctl_h->nrm[N_IN2];
    return TRPLK_OK;
}

trplk_status trplk_k_cgs2(trplk_ctx* ctx, const double* U, int64_t ldu, int k, const double* w, double* out,
                          double* h, double* beta, int* breakdown, int* passes) {
    ST(kprep(ctx, k));
    if (ldu < ctx->n_loc) {
        ctx->err = "bad ldu";
        return TRPLK_EINVAL;
    }
    ST(ctl_pull(ctx));
    const int p3 = ctx->ctl_h->pass3_count;
    CgsSpec c{};
    c.x = w;
    c.V = U;
    c.ldv = ldu;
    c.kv = k;
    c.k_nominal = k;
    c.dest = out;
    c.dest_dyn = 0;
    c.gate = F_CYCLE;
    c.clear = F_CYCLE;
    c.inc_k = 0;
    ST(cgs2(ctx, c));
    ST(ctl_pull(ctx));
    const Ctl& H = *ctx->ctl_h;
    const bool third = H.pass3_count > p3;
    double hn = 0.0;
    const int last = third ? 2 : 1;
    for (int i = 0; i < k; ++i) hn += H.h[last][i] * H.h[last][i];
    const double b2 = (third ? H.nrm[N_2SQ_EXP] : H.nrm[N_1SQ]) - hn;
    if (beta) *beta = std::sqrt(b2 > 0 ? b2 : 0.0);
    if (breakdown) *breakdown = (H.flags & F_CYCLE) ? 0 : 1;
    if (passes) *passes = third ? 3 : 2;
    if (h)
        for (int i = 0; i < k; ++i) h[i] = H.h[0][i] + H.h[1][i] + (third ? H.h[2][i] : 0.0);
    return TRPLK_OK;
}

trplk_status trplk_k_block(trplk_ctx* ctx, int mode, const double* U, int64_t ldu, int k, const double* Y,
                           int64_t ldy, int c, const double* Rinv, const double* H, double* Yout, int64_t ldyo,
                           double* HV, double* G) {
    ST(kprep(ctx, k));
    if (c < 1 || c > BC || mode < BM_GRAM || mode > BM_SPMM || ldu < ctx->n_loc || ldy < ctx->n_loc ||
        (mode == BM_UPD && (!H || !Yout || ldyo < ctx->n_loc))) {
        ctx->err = "trplk_k_block: bad arguments";
        return TRPLK_EINVAL;
    }
    std::vector<double> hb((size_t)QMAX * BC, 0.0), rb((size_t)BC * BC, 0.0);
    if (H)
        for (int j = 0; j < c; ++j)
            for (int i = 0; i < k; ++i) hb[i + (size_t)QMAX * j] = H[i + (size_t)k * j];
    if (Rinv)
        for (int j = 0; j < c; ++j)
            for (int i = 0; i < c; ++i) rb[i + (size_t)BC * j] = Rinv[i + (size_t)c * j];
    CK(cudaMemcpyAsync(ctx->blk->Hs, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemcpyAsync(ctx->blk->Rinv, rb.data(), rb.size() * 8, cudaMemcpyHostToDevice, ctx->stream));
    if (mode == BM_SPMM) {
        for (int j = 0; j < c; ++j) ST(halo(ctx, Y + ldy * j));
    }
    BlkArgs a{};
    a.nrows = ctx->n_loc;
    a.U = U;
    a.ldu = ldu;
    a.k = k;
    a.Y = Y;
    a.ldy = ldy;
    a.c = c;
    a.mode = mode;
    a.A = ctx->A;
    a.Rinv = Rinv ? ctx->blk->Rinv : nullptr;
    a.H = ctx->blk->Hs;
    a.Yout = Yout;
    a.ldyo = ldyo;
    a.HV = ctx->blk->HV[0];
    a.G = ctx->blk->G[0];
    a.gate = F_CYCLE;
    ST(run_block(ctx, a, std::max(k, 1), 0.0));
    std::vector<double> hv((size_t)QMAX * BC), g((size_t)BC * BC);
    CK(cudaMemcpyAsync(hv.data(), ctx->blk->HV[0], hv.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaMemcpyAsync(g.data(), ctx->blk->G[0], g.size() * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (HV)
        for (int j = 0; j < c; ++j)
            for (int i = 0; i < k; ++i) HV[i + (size_t)k * j] = hv[i + (size_t)QMAX * j];
    if (G && mode != BM_SPMM)
        for (int j = 0; j < c; ++j)
            for (int i = 0; i < c; ++i) G[i + (size_t)c * j] = g[i + (size_t)BC * j];
    return TRPLK_OK;
}

trplk_status trplk_k_rotate(trplk_ctx* ctx, const double* U, int64_t ldu, int k, const double* Y, int ncol,
                            double* X, int64_t ldx) {
    ST(kprep(ctx, k));
    if (k < 1 || ncol < 1 || ncol > 24 || ldu < ctx->n_loc || ldx < ctx->n_loc) {
        ctx->err = "bad rotate sizes";
        return TRPLK_EINVAL;
    }
    CK(cudaMemcpy2DAsync(ctx->Yg, 8 * QMAX, Y, 8 * (size_t)k, 8 * (size_t)k, ncol, cudaMemcpyHostToDevice,
                         ctx->stream));
    launch_rotate(U, ldu, ctx->n_loc, ctx->ctl, k, ctx->Yg, QMAX, ncol, X, ldx, 0, ctx->stream, k);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return TRPLK_OK;
}

trplk_status trplk_k_sym_eig(trplk_ctx* ctx, int k, const double* T, double* theta, double* Y) {
    ST(kprep(ctx, k));
    if (k < 1) {
        ctx->err = "k < 1";
        return TRPLK_EINVAL;
    }
    double* Td;
    ST(dalloc(ctx, &Td, (size_t)QMAX * QMAX));
    CK(cudaMemcpy2DAsync(Td, 8 * QMAX, T, 8 * (size_t)k, 8 * (size_t)k, k, cudaMemcpyHostToDevice, ctx->stream));
    launch_eig(ctx->ctl, Td, QMAX, ctx->Yg, QMAX, 0, k, 0, ctx->stream);
    CK(cudaGetLastError());
    ST(ctl_pull(ctx));
    if (theta) memcpy(theta, ctx->ctl_h->theta, 8 * (size_t)k);
    if (Y) CK(cudaMemcpy2D(Y, 8 * (size_t)k, ctx->Yg, 8 * QMAX, 8 * (size_t)k, k, cudaMemcpyDeviceToHost));
    dev_free(ctx, Td);
    return TRPLK_OK;
}

trplk_status trplk_k_sym_eig_time(trplk_ctx* ctx, int k, const double* T, int reps, double* ms, int* sweeps) {
    ST(kprep(ctx, k));
    if (k < 1 || reps < 1) {
        ctx->err = "k < 1 or reps < 1";
        return TRPLK_EINVAL;
    }
    double* Td;
    ST(dalloc(ctx, &Td, (size_t)QMAX * QMAX));
    CK(cudaMemcpy2DAsync(Td, 8 * QMAX, T, 8 * (size_t)k, 8 * (size_t)k, k, cudaMemcpyHostToDevice, ctx->stream));
    launch_eig(ctx->ctl, Td, QMAX, ctx->Yg, QMAX, 0, k, 0, ctx->stream);  // warm-up
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, ctx->stream));
    for (int i = 0; i < reps; ++i) launch_eig(ctx->ctl, Td, QMAX, ctx->Yg, QMAX, 0, k, 0, ctx->stream);
    CK(cudaEventRecord(e1, ctx->stream));
    CK(cudaEventSynchronize(e1));
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(cudaGetLastError());
    ST(ctl_pull(ctx));
    if (ms) *ms = (double)t / reps;
    if (sweeps) *sweeps = ctx->ctl_h->eig_sweeps;
    dev_free(ctx, Td);
    return TRPLK_OK;
}

trplk_status trplk_loopback_create(int nranks, void** hub) {
    if (nranks < 1 || !hub) return TRPLK_EINVAL;
    *hub = new LoopHub(nranks);
    return TRPLK_OK;
}

void trplk_loopback_destroy(void* hub) { delete static_cast<LoopHub*>(hub); }

trplk_status trplk_k_residual(trplk_ctx* ctx, const double* x, double theta, double* r, double* u, double* rnorm2) {
    ST(kprep(ctx, 0));
    SdotsArgs a = sd_base(ctx);
    a.A = ctx->A;
    if (ctx->hasB) a.B = ctx->B;
    a.x = x;
    a.out_mode = 3;
    a.out = r;
    a.uout = u;
    a.norm1 = 1;
    a.nslot1 = N_RES2;
    a.theta_idx = -2;
    a.theta_val = theta;
    ST(run_sdots(ctx, a, 0));
    ST(ctl_pull(ctx));
    if (rnorm2) *rnorm2 = ctx->ctl_h->nrm[N_RES2];
    return TRPLK_OK;
}

trplk_status trplk_k_random(trplk_ctx* ctx, uint64_t seed, uint64_t stream, uint64_t col, double* x) {
    if (!ctx) return TRPLK_EINVAL;
    enter_stream(ctx);
    launch_random(x, ctx->n_loc, ctx->row_begin, ctx->n_global, seed, stream, col, ctx->stream);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(ctx->stream));
    return TRPLK_OK;
}

trplk_status trplk_plan_ghosts(int64_t row_begin, int64_t row_end, const int64_t* a_rowptr, const int64_t* a_col,
                               const int64_t* b_rowptr, const int64_t* b_col, const int64_t* ranges, int nranks,
                               int64_t* ghosts_out, int* owners_out, int64_t cap, int64_t* n_ghost) {
    if (!a_rowptr || !a_col || row_end < row_begin || !n_ghost || nranks < 1) return TRPLK_EINVAL;
    const std::vector<int64_t> g =
        find_ghosts(row_end - row_begin, row_begin, row_end, a_rowptr, a_col, b_rowptr, b_col);
    *n_ghost = (int64_t)g.size();
    if ((int64_t)g.size() > cap) return TRPLK_EINVAL;
    const std::vector<int> own = ranges ? ghost_owners(g, ranges, nranks) : std::vector<int>(g.size(), 0);
    for (size_t i = 0; i < g.size(); ++i) {
        if (ghosts_out) ghosts_out[i] = g[i];
        if (owners_out) owners_out[i] = own[i];
    }
    return TRPLK_OK;
}

trplk_status trplk_profile(trplk_ctx* ctx, int enable) {
    if (!ctx) return TRPLK_EINVAL;
    if (enable && !ctx->pev[0]) {
        for (auto& e : ctx->pev) CK(cudaEventCreate(&e));
        for (auto& e : ctx->phev) CK(cudaEventCreate(&e));
    }
    ctx->prof_on = enable != 0;
    for (int i = 0; i < 3; ++i) ctx->prof_ms[i] = ctx->prof_bytes[i] = 0.0;
    ctx->prof_count = 0;
    for (int i = 0; i < 6; ++i) ctx->phase_ms[i] = 0.0;
    ctx->phase_count = 0;
    return TRPLK_OK;
}

trplk_status trplk_profile_phases(const trplk_ctx* ctx, double* ms, int64_t* count) {
    if (!ctx) return TRPLK_EINVAL;
    for (int i = 0; i < 6; ++i)
        if (ms) ms[i] = ctx->phase_ms[i];
    if (count) *count = ctx->phase_count;
    return TRPLK_OK;
}

trplk_status trplk_profile_kernels(const trplk_ctx* ctx, char* buf, size_t len) {
    if (!ctx || !buf || len == 0) return TRPLK_EINVAL;
    std::string out;
    for (int i = 0; i < 3; ++i) {
        const char* name = nullptr;
        const void* kf = (ctx->prof_fused && i == 2) ? nullptr : ctx->prof_kern[i];  // fused: no third group
        if (kf && cudaFuncGetName(&name, kf) != cudaSuccess) name = nullptr;
        std::string nm = name ? name : "";
        if (name) {
            int stt = 0;
            char* dm = abi::__cxa_demangle(name, nullptr, nullptr, &stt);
            if (dm && stt == 0) nm = dm;
            free(dm);
        }
        out += nm;
        if (i < 2) out += ";";
    }
    if (out.size() + 1 > len) return TRPLK_EINVAL;
    memcpy(buf, out.c_str(), out.size() + 1);
    return TRPLK_OK;
}

trplk_status trplk_profile_read(const trplk_ctx* ctx, double* ms, double* bytes, int64_t* count) {
    if (!ctx) return TRPLK_EINVAL;
    for (int i = 0; i < 3; ++i) {
        if (ms) ms[i] = ctx->prof_ms[i];
        if (bytes) bytes[i] = ctx->prof_bytes[i];
    }
    if (count) *count = ctx->prof_count;
    return TRPLK_OK;
}

}  // extern "C"
