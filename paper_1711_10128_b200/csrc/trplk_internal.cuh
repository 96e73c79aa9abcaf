// Internal declarations of the TRPL+K device path (kernels + engine).
// Not part of the ABI; see include/trplk.h for the boundary.
#pragma once
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

namespace trplk {

constexpr int QMAX = 64;           // TRPLK_MAX_BASIS
constexpr int NV_MAX = 2 * QMAX + 4; // values of one fused reduction
constexpr int CTA = 256;           // threads per CTA of the streaming kernels
constexpr int WARPS = CTA / 32;
constexpr int MAXCTA = 2048;       // largest grid of a reducing kernel
constexpr int MAXG = MAXCTA / 32;  // reduction groups (32 CTAs each)
constexpr int NCOUNTERS = 1 + MAXG;

constexpr int DIA_MAX = 32;       // most diagonals a DIA matrix may have

// Local sparse matrix (rows owned by this rank), one of two device formats chosen at create:
//  fmt 0  SELL-32: slice s holds rows [32s, 32s+32); entry j of lane l sits at
//         sptr[s] + 32*j + l; slot j=0 is the diagonal.  Padding: val 0, col = row.
//         Column ids are local: [0, nrows) owned, [nrows, nrows+nghost) ghost tail.
//  fmt 1  DIA: ndiag diagonals with global offsets offs[d] (col = row + offs[d]); values
//         dval[d*ldv + row] (0 where no entry).  Requires the ghost tail to be the contiguous
//         global ranges [row_begin-glo, row_begin) then [row_end, row_end+nghost-glo), so the
//         local index of row+off is computed, not loaded.  diag_slot = index of offset 0.
//         Constant diagonals (DIA-C, opt-in): bit d (d < 8) of cmask set = every stored entry of
//         diagonal d has the same bit pattern cv[d] (kept in the descriptor, i.e. in the kernel
//         parameters); the kernels then read, instead of the d-th value array, bit d of the
//         row's presence byte pmask[row] (0 past the last row) and use cv[d] where it is set,
//         +0.0 elsewhere -- exactly the stored values (a stencil's -1 couplings: 8 bytes per
//         row and diagonal become one bit).  dval stays fully populated (IC(0) factors from it).
struct Sell {
    int fmt = 0;
    int64_t nrows = 0;
    int64_t nslices = 0;
    const int64_t* sptr = nullptr;
    const int* col = nullptr;
    const double* val = nullptr;
    int ndiag = 0, diag_slot = 0;
    int64_t ldv = 0, glo = 0, nghost = 0;
    const double* dval = nullptr;
    int offs[DIA_MAX] = {};
    unsigned cmask = 0;
    const unsigned char* pmask = nullptr;
    double cv[8] = {};
};

// Presence word of a DIA-C row (bit d = entry of constant diagonal d stored).
__device__ __forceinline__ unsigned dia_pmask(const Sell& M, int64_t row) { return __ldg(M.pmask + row); }
// Value of diagonal d at a row: the stored array, or the constant where the row's bit is set.
__device__ __forceinline__ double dia_val(const Sell& M, int d, unsigned pm, const double* dv) {
    if (d < 8 && ((M.cmask >> d) & 1u)) return ((pm >> d) & 1u) ? M.cv[d < 8 ? d : 0] : 0.0;
    return __ldg(dv + (int64_t)d * M.ldv);
}

// Gate bits of Ctl::flags
enum : unsigned {
    F_CYCLE = 1u,      // seed of this cycle valid
    F_INNER = 2u,      // inner Lanczos loop still running (no breakdown, R16)
    F_KCOL0 = 4u,      // +K column j valid: F_KCOL0 << j
    F_BPASS3 = 1u << 30,  // block +K: third BCGS pass needed (R3); F_KCOL0 << j uses bits 2..17
    F_XD0 = 1u << 20,     // +K column j's first-pass dots still to do: F_XD0 << j (j < 8), cleared by the
                          // K1 launch that computed them alongside its own dots (set2 = 4)
};

// Norm slots of Ctl::nrm
enum { N_IN2 = 0, N_1SQ = 1, N_2SQ_EXP = 2, N_RES2 = 3, N_AUX = 4, N_SLOTS = 8 };

// Destination codes of a reduction
enum { D_NONE = 0, D_TCOL = 1, D_H0 = 2 /* D_H0 + slot */ };

// Device control block.  The host writes the head (k .. xprev) before every cycle.
struct Ctl {
    int k;            // current basis width
    unsigned flags;   // gate bits
    int t;            // target, 1-based
    int pass3;        // third CGS pass pending (R3)
    double rho;       // shift of this cycle (Alg.1 step 15)
    int xprev_col;    // first X^prev column in the previous cycle's buffer (Alg.1 step 10)
    // ---- device-written from here on (not overwritten by the per-cycle host push)
    int k_rr;         // width used by the last Rayleigh-Ritz
    int brk;          // breakdown events (diagnostic, cumulative)
    int pass3_count;  // third CGS passes taken (cumulative)
    int eig_sweeps;   // Jacobi sweeps of the last Rayleigh-Ritz (diagnostic)
    double nrm[N_SLOTS];
    double h[4][QMAX];
    double theta[QMAX];
};

// Arguments of the fused SpMV + preconditioner + dots kernel (K1 / K7 / Gram).
struct SdotsArgs {
    Sell A;            // op1 (A.nrows == 0 => z = x)
    Sell B;            // op2 (B.nrows == 0 => s = x, i.e. B = I)
    int64_t nrows;     // local rows
    const double* x;   // input vector (with ghosts if multiplied)
    int x_dyn;         // 0: x; 1: x + x_ld*(ctl->t-1+x_off); 2: x + x_ld*(ctl->xprev_col+x_off)
    int64_t x_ld;
    int x_off;
    const double* wext;// RESW: r = wext - theta s
    int out_mode;      // 0 none, 1 z, 2 PREC w=M(z-rho s), 3 RES r=z-theta s (+u=M r), 4 RESW
    double* out;       // written if non-null (z / w / r)
    double* uout;      // RES/RESW: u = M r if non-null
    const double* U;   // dot block
    int64_t ldu;
    int set1;          // vector for dot set 1: 0 none, 1 z, 2 out, 3 x
    int set2;          // vector for dot set 2 (same U): 0 none, 2 out, 4 x2 (an external vector)
    int k1, k2;        // #columns; <0 => ctl->k + (k+1) ... see k_from_ctl
    int k_from_ctl;    // 1: k1 = k2-style counts = ctl->k (set2 only if set2 != 0)
    int norm1, norm2;  // 0 none, 1 out.out, 2 x.z, 3 x.x, 4 z.z, 5 x2.x2 (norm2 only)
    int theta_idx;     // RES: theta = ctl->theta[theta_idx] (>=0) or ctl->theta[ctl->t-1] (-1)
    double theta_val;  // used when theta_idx == -2
    int dest1, dest2;  // D_TCOL / D_H0+slot / D_NONE
    int tcol_fixed;    // >=0: T column index for D_TCOL (no mirror); -1: ctl->k-1, mirrored
    int nslot1, nslot2;
    unsigned gate;
    int gate_pass3;
    double sigma, mfloor;
    int pmode;         // 2: M = Jacobi of A - rho B with this cycle's shift (w) / the residual's theta (u = M r)
    int count_prec;    // reserved
    Ctl* ctl;
    double* T;
    int ldT;
    double* part;      // [NV_MAX][maxcta]
    double* gpart;     // [NV_MAX][MAXG]
    unsigned* counter; // [NCOUNTERS]
    int maxcta;
    double* red_local; // multi-rank: local sums instead of finalize (nullptr => finalize)
    // row range split (halo overlap, K1 kernels k_step1_rs2 / k_step1_pipe): rows [row0, nrows)
    // (row0 a multiple of 32); this launch's CTAs are partial slots cta_off.. of a reduction over
    // cta_tot CTAs in several launches (0: this grid alone); grid_force > 0 fixes the grid size
    int64_t row0;
    int cta_off, cta_tot, grid_force;
    // set2 = 4: the second dot set is U^T x2 (x2 resolved like x: x2_dyn 2 = x2 + x2_ld *
    // (ctl->xprev_col + x2_off)) -- the next +K column's first CGS pass riding on a K1 that reads
    // U anyway; clear_done: flag bits the finalize clears (F_XD0 << j: those dots are done)
    const double* x2;
    int x2_dyn, x2_off;
    int64_t x2_ld;
    unsigned clear_done;
};

// Arguments of the CGS update kernel (K2 / K3 / fix-up).
struct UpdArgs {
    int64_t nrows;
    const double* x;   // vector being orthogonalised
    int x_dyn;         // as SdotsArgs::x_dyn
    int64_t x_ld;
    int x_off;
    const double* U;   // basis block
    int64_t ldu;
    int kv;            // #columns (>=0) or -1 => ctl->k
    int hslot;         // coefficients ctl->h[hslot]
    int mode;          // 0 NONE (y = x - U h -> out), 1 DOTS, 2 FINAL, 3 FIX
    int dots;          // DOTS/FINAL-pass3/FIX?: compute U^T y and y.y (B = I only)
    double* out;       // y written (NONE/DOTS, FINAL pass-3 path)
    double* dest;      // FINAL/FIX: normalised vector destination (column base pointer)
    int64_t dest_ld;   // dest + dest_ld * ctl->k when dest_dyn
    int dest_dyn;
    double* dest2;     // optional copy (+K scratch)
    int hout;          // DOTS: coefficient slot for U^T y; norm -> ctl->nrm[N_1SQ] (or N_2SQ_EXP in FINAL)
    int inc_k;         // FINAL/FIX: ctl->k += 1 on success
    unsigned gate;
    unsigned clear_on_brk;
    Ctl* ctl;
    double* part;
    double* gpart;
    unsigned* counter;
    int maxcta;
    double* red_local;
    int coop;   // FINAL launched cooperatively: a third pass (R3) runs inside the kernel (1 rank, B = I)
    int force3; // debug: take the third CGS pass unconditionally (tests of the pass-3 path)
};

// K3 of inner step j fused with K1 of step j + 1 (fused.cuh): FINAL update args, K1 args, the
// per-round completion counters (zero between launches) and the round lag (set at launch).
struct FusedArgs {
    UpdArgs u;
    SdotsArgs a;
    unsigned* rcnt;
    int64_t rcnt_cap;
    int dn, lag;  // rounds a tile's stencil reaches past its own; rounds between FINAL and K1
};
bool launch_fin_step1(const FusedArgs& f, int kmax, int maxoff, int slack, cudaStream_t s);
bool launch_step1_lean(const SdotsArgs& a, int kmax, cudaStream_t s);
// true for the kernels that read a DIA-C matrix's presence bits instead of its constant diagonals
// (k_step1_lean, k_fin_step1): their algorithmic matrix bytes are the compressed ones
bool kern_reads_diac(const void* kern);

// ------------------------------------------------------------- block kernels (block.cuh)
constexpr int BC = 8;                                // vectors per block launch (DMMA n = 8)
constexpr int BLK_NV = 2 * QMAX * BC + BC * BC;      // reduction values of one block launch
enum { BM_GRAM = 0, BM_UPD = 1, BM_SPMM = 2, BM_SPMW = 3 };

// Device state of one block CGS2 (+K augmentation): pass results and the small c x c factors.
struct BlkCtl {
    double HV[4][QMAX * BC];  // U^T V of the GRAM / UPD passes (ld QMAX)
    double G[4][BC * BC];     // V^T V of the passes (ld BC)
    double Hs[QMAX * BC];     // coefficients of the next UPD: (U^T W) Rinv
    double Rinv[BC * BC];     // upper triangle applied before the next update / the placement
    double lprod[BC];         // product of the Cholesky pivots so far (norm left of input vector j)
    double g0[BC];            // input squared norms (breakdown test, R3/R16)
    int c;                    // vectors in the block
    int acc;                  // accepted (not dependent) vectors
    int drop[BC];             // 1: vector j dependent (dropped, R16)
    int pos[BC];              // compacted position of accepted vector j
    int k0;                   // basis width before the block was appended
    int pass3;                // third pass pending (R3)
    int cin;                  // vectors entering the next block CGS2 (block inner loop: fit the basis)
};

struct BlkArgs {
    int64_t nrows;
    const double* U;
    int64_t ldu;
    int k;            // basis columns (k_from_ctl: ctl->k + k_off)
    int k_from_ctl, k_off;
    const double* Y;  // input vectors (ld ldy; SPMM: with ghost tails)
    int64_t ldy;
    int y_dyn;        // 2: Y + ldy * ctl->xprev_col (the X^prev columns of the previous block)
    int c;            // vectors (<= BC), or *c_dyn
    const int* c_dyn;
    const int* c_cap;    // non-null: c = min(c, *c_cap) (room left in the basis)
    const double* Rinv;  // UPD: optional c x c upper triangle (ld BC): Q = Y Rinv
    const double* H;     // UPD: k x c (ld QMAX): Y' = Q - U H
    double* Yout;        // UPD: Y' (may alias Y)
    int64_t ldyo;
    Sell A;              // SPMM / SPMW: Z = A Y
    double sigma, mfloor;  // SPMW: W = M (Z - rho Y) (rho = ctl->rho, Jacobi M of A - sigma I) -> Yout
    int mode;            // BM_GRAM / BM_UPD / BM_SPMM / BM_SPMW
    double* HV;          // result U^T V (ld QMAX); SPMW: U^T W
    double* G;           // result V^T V (ld BC)
    double* T;           // SPMM: T(i, k0 + j) = (U^T Z)(i, j), mirrored; k0 = *k0p
    int ldT;
    const int* k0p;
    unsigned gate;
    Ctl* ctl;
    double* part;
    double* gpart;
    unsigned* counter;
    int maxcta;
    double* red_local;
};

// IC(0) preconditioner (ic0.cuh)
struct Ic0Args {
    Sell A;                 // DIA (fmt 1)
    double sigma, floor;    // K = A - sigma I; pivot floor eps_d max|K_jj|
    double* L;              // [nlow + 1][ldl]: lower diagonals in A's offset order, then the diagonal
    int64_t n, ldl;
    int nlow;
    int lslot[DIA_MAX];     // A's diagonal slot of lower diagonal a
    int loff[DIA_MAX];      // its offset (< 0), ascending
    int pair[DIA_MAX][DIA_MAX];  // factor: lower diagonal index of offset loff[b] - loff[a] (b < a), or -1
    int* flags;             // per chunk done flag (zeroed before every launch); flags[nchunk] = ticket
    const double* v;        // solve: right-hand side
    double* y;              // solve: result
    int trans;              // 0: L y = v, 1: L^T y = v
    const Ctl* ctl;         // gate: the launch is a no-op unless (ctl->flags & gate) == gate
    unsigned gate;
};

void launch_ic0_factor(const Ic0Args& a, cudaStream_t s);
void launch_ic0_solve(const Ic0Args& a, cudaStream_t s);

// Single-CTA inner loop of the small-n latency path (small.cuh)
constexpr int SMALL_NMAX = 8192;  // rows handled by the small path (32 per thread)

struct SmallArgs {
    Sell A;
    int64_t nrows;
    double* U;  // current basis block (column k-1 = g_1 on entry)
    int64_t ldu;
    double *w, *w1, *w2;
    Ctl* ctl;
    double* T;
    int ldT;
    int m;  // inner steps of the cycle
    double sigma, mfloor;
    int pmode;  // as SdotsArgs::pmode
    unsigned gate, clear;
    int force3;
};


// Grid-wide persistent inner loop (inner_grid.cuh): SmallArgs plus the all-reduce buffer.
constexpr int GRID_NVP = 72;       // stride of one CTA's partial sums
constexpr int GRID_MAXCTA = 1024;  // partial buffer: 2 x GRID_MAXCTA x GRID_NVP doubles
struct GridArgs {
    SmallArgs s;
    double* part;
    unsigned long long* trace;  // optional (TRPLK_GRID_TRACE): phase timestamps of CTA 0, per step
};

// PL+1 (pl1.cuh): device scratch of the projected pencil of step 5 and the dot-pair list.
constexpr int PL1_QP = 34;  // Q_k columns: x, m <= 32 Krylov vectors, p
struct Pl1Dev {
    double L[PL1_QP * PL1_QP];  // Cholesky factor of Q^T B Q (compacted columns)
    double w[PL1_QP];           // primitive Ritz vector in Q's m+2 slots (zeros: unused)
    double sc[16];              // scalars written by pl1_dots
    int cols[PL1_QP];           // compact column -> Q slot
    int nq, fail;               // read together by the host
    int mg;                     // G_k columns built (ctl->k after step 4)
    int has_p;                  // p_k formed (||p~_k||_B > 0)
    double rho_cur, rho_prev;   // rho(x_k), rho(x_{k-1}) (device copies, so an iteration is a graph)
};
struct Pl1Pairs {
    const double* a[4];
    const double* b[4];
    int slot[4];
    int np;
};
constexpr int PL1_PART = 296 * 72;  // partials of pl1_dots / pl1_gram (296 CTAs x 2 NT, NC <= 8)
void pl1_prec(const Sell& A, const Sell& B, int64_t n, double sigma, double mfloor, const double* z,
              const double* s, const double* rho, double* v, int prec, cudaStream_t st);
void pl1_qmirror(double* H, int ldH, int d, cudaStream_t st);     // mirror the upper d x d triangle (P7)
void pl1_begin(Ctl* ctl, cudaStream_t st);                         // ctl->k = 0, flags = ~0, pass3 = 0
void pl1_shift_rho(Pl1Dev* d, const double* sc, cudaStream_t st);  // rho_prev = rho_cur; rho_cur = sc1/sc2
void pl1_dvec(int64_t n, const double* Ap, const double* Bp, const Pl1Dev* d, double* v, cudaStream_t st);
void pl1_dots(const Pl1Pairs& P, int64_t n, double* part, double* out, cudaStream_t st);
void pl1_dots_ranks(const Pl1Pairs& P, const double* all, int nranks, int stride, double* out, cudaStream_t st);
void pl1_reduce(const double* Hq, const double* Sq, int ldq, int m, Ctl* ctl, int has_p, double* T, int ldT,
                Pl1Dev* d, cudaStream_t st);
void pl1_scale_p(int64_t n, const double* x, const double* nrm2, double* y, Pl1Dev* d, cudaStream_t st);
void pl1_back(const double* Y, int ldY, int m, Pl1Dev* d, cudaStream_t st);
// H = Q^T A Q, S = Q^T B Q (nc x nc, ld nc) in one pass for 3 <= nc <= 8; false: not handled
bool pl1_gram(int nc, const double* Q, const double* AQ, const double* BQ, int64_t ld, int64_t n, double* part,
              double* H, double* S, cudaStream_t st);
void pl1_xt(int64_t n, const double* x, const double* g, const double* p, const Pl1Dev* d, int m, double* xt,
            cudaStream_t st);
void pl1_scale(int64_t n, const double* x, const double* nrm2, double* y, cudaStream_t st);
void pl1_res(int64_t n, const double* Ax, const double* Bx, const double* xAx, const double* xBx, double* r,
             cudaStream_t st);
void pl1_axpby(int64_t n, double a, const double* x, double b, const double* z, double* y, cudaStream_t st);
void pl1_pt(int64_t n, const double* g, const double* p, const double* num, const double* den, double den_floor,
            int variant, const Pl1Dev* d, int m, double* pt, cudaStream_t st);

// Kernel launchers (kernels.cu)
// Jacobi preconditioner entry M_ii = 1 / max(|A_ii - sigma B_ii|, mfloor) (reading R12);
// mfloor < 0 encodes M = I (trplk_options.precond = 1: no preconditioning, the thick-restart
// Lanczos reduction of eq 2.1, when k_plus = 0).
__device__ __forceinline__ double jacobi_minv(double ad, double bd, double sigma, double mfloor) {
    if (mfloor < 0.0) return 1.0;
    double d = fabs(ad - sigma * bd);
    d = d > mfloor ? d : mfloor;
    return 1.0 / d;
}

// Programmatic dependent launch (sm_90+): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its predecessor finishes;
// griddepcontrol.wait blocks until the predecessor grid has completed and its writes are visible
// (a no-op when launched normally), launch_dependents lets the successor launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Launch with programmatic stream serialization (the kernel calls pdl_wait before touching its
// predecessor's results).  TRPLK_PDL=0: plain launches.
inline bool pdl_on() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("TRPLK_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
    }
    return v == 1;
}

template <typename A>
inline void launch_pdl(void (*kern)(A), int grid, int block, int smem, cudaStream_t s, const A& a) {
    if (!pdl_on()) {
        kern<<<grid, block, smem, s>>>(a);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a);
}

// The kernel function most recently launched by this host thread (measurement: bench.py and the
// live profile name the instantiation that ran, trplk_profile_kernels).
extern thread_local const void* g_last_kern;
#define NOTE_KERN(k) (::trplk::g_last_kern = reinterpret_cast<const void*>(k))

bool launch_inner_small(const SmallArgs& a, int kmax, cudaStream_t s);
bool launch_block(const BlkArgs& a, int kmax, cudaStream_t s);
void launch_blk_finalize_multi(const BlkArgs& a, const double* red_all, int nranks, int stride, cudaStream_t s);
// BCGS2 control of a +K block (one small kernel per stage): stage 0 after the GRAM pass, 1 after
// the first UPD (Cholesky-QR, drops), 2 after the second UPD (Cholesky-QR, third-pass test),
// 3 after the gated third UPD; stage 2/3 also place the accepted vectors (ctl->k += acc).
void launch_blk_ctl(BlkCtl* b, Ctl* ctl, int stage, int c, const int* c_dyn, int seed, unsigned gate,
                    cudaStream_t s);
void launch_blk_room(BlkCtl* b, const Ctl* ctl, int kcap, unsigned gate, cudaStream_t s);
// Q(:, pos_j) = (W Rinv)(:, j) for accepted j into U(:, k0 + pos_j) and xk(:, pos_j); c = 0: b->c
void launch_blk_place(const double* W, int64_t ldw, const BlkCtl* b, const Ctl* ctl, double* U, int64_t ldu,
                      double* xk, int64_t ldx, int64_t nrows, int c, unsigned gate, cudaStream_t s);
// false: not applicable (kmax > 32 or no co-resident grid); nothing launched
bool launch_inner_grid(const GridArgs& a, int kmax, cudaStream_t s);
void launch_sdots(const SdotsArgs& a, int kmax, cudaStream_t s);
void launch_upd(const UpdArgs& a, int kmax, cudaStream_t s);
void launch_eig(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph, int k_fixed, unsigned gate,
                cudaStream_t s);
// TRPLK_EIG=tri: tridiagonalisation + multisection + inverse iteration for the nev lowest pairs
// (eig_tri.cu); nev <= 0: all k
void launch_eig_tri(Ctl* ctl, double* T, int ldT, double* Y, int ldY, int ph, int k_fixed, int nev, unsigned gate,
                    cudaStream_t s);
void launch_rotate(const double* U, int64_t ldu, int64_t nrows, const Ctl* ctl, int k_fixed,
                   const double* Y, int ldY, int ncol, double* X, int64_t ldx, unsigned gate,
                   cudaStream_t s, int kmax);
void launch_random(double* x, int64_t nrows, int64_t row0, int64_t n_global, uint64_t seed,
                   uint64_t stream, uint64_t col, cudaStream_t s);
void launch_finalize_sdots_multi(const SdotsArgs& sd, const double* red_all, int nranks, int stride,
                                 cudaStream_t s);
void launch_finalize_upd_multi(const UpdArgs& up, const double* red_all, int nranks, int stride,
                               cudaStream_t s);
void launch_gather(const double* x, const int* idx, int64_t n, double* out, cudaStream_t s);
void launch_copy_cols(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t nrows, int ncols,
                      cudaStream_t s);
// CSR (device copies of the caller's pinned arrays) -> DIA values, one thread per row; dval
// must be zeroed.  offs: the nd sorted diagonal offsets.
// DIA-C (constant diagonals): min/max stored bit pattern per diagonal (mnmx: 2 nd entries,
// initialised to {~0, 0}), then the presence words of the diagonals in cmask.
void launch_dia_const_scan(const double* dval, int64_t nrows, int64_t ldv, int nd, unsigned long long* mnmx,
                           cudaStream_t s);
void launch_dia_pmask(const double* dval, int64_t nrows, int64_t ldv, int nd, unsigned cmask, unsigned char* pm,
                      cudaStream_t s);
void launch_csr_to_dia(const int64_t* rp, const int64_t* ci, const double* va, int64_t nrows, int64_t row0,
                       const int* offs, int nd, int64_t ldv, double* dval, cudaStream_t s);
int kmax_bucket(int k);

}  // namespace trplk
