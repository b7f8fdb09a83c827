// ridc_device.cuh -- device side of the fused RIDC-FBE level step (sm_100a, fp64).
//
// One "work item" = one level-step of one tile of the state (a whole x-line,
// or a segment of a long 1-D line plus truncation halos).  The item fuses:
//
//   rhs  = eta + dt f^N(eta) + sum_k ( cs_k f^S(w_k) + cn_k f^N(w_k) )
//          (kernels.py:119-125 predictor_rhs, :137-147 corrector_rhs; the
//           -dt f^S(new) and -dt f^N(old) lag terms of engine.py:179-181
//           are folded into cs/cn of the window nodes; f^S, f^N are
//           recomputed from the stored states by stencils instead of being
//           read back, problems.py:119-124/:158-164, kernels.py:160-168)
//   x    = (I - dt L_S)^{-1} rhs
//          (replaces the dense Q^T b GEMV + back-substitution of qr_solve,
//           linalg.py:59-63; L_S is (cyclic) tridiagonal, problems.py:119-124,
//           :148-156, so the shifted operator factors into two first-order
//           recurrences:  periodic: (r/lam)(1 - lam E^-1)(1 - lam E),
//           Dirichlet: the Thomas LU with converging pivots.)
//
// Data path per item: coalesced fp64 loads of (j+2) state vectors from
// HBM/L2 into registers (one pass), rhs to padded shared memory, a
// block-wide affine scan (forward, then backward) for the recurrences, and
// one coalesced store of the new state.  Non-finite detection
// (engine.py:160-164) is fused into the store.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#ifdef RIDC_CHECKED
#include <cstdio>
#endif

namespace ridc {

enum Kind { ADV_DIFF_1D = 1, BURGERS_1D = 2, RD_1D = 3, ADV_DIFF_2D = 4, RD_2D = 5 };

constexpr int kMaxLevels = 12;              // engine.py:47 (MAX_LEVEL + 1)
constexpr int kMaxNodes = 2 * kMaxLevels + 1;  // own state + window (states, or f^S and f^N rows)
constexpr int kMaxChunk = 32;               // max elements per thread in the scan phase

struct DevProblem {
    int kind, nx, ny, periodic;
    double cax, cay;   // c_x/h_x, c_y/h_y
    double cdx, cdy;   // d_x/h_x^2, d_y/h_y^2
    double rho, bs;    // reaction rate, Burgers scale 1/(4 h_x)
};

// Factors of (I - dt*cdx*D_xx) for one x-line.
struct DevSolve {
    double lam;          // limit multiplier m_inf (= lambda)
    double g;            // limit scale g_inf (= lambda / r)
    const double* tab_m; // Dirichlet: Thomas multipliers m_i for i < ntab
    const double* tab_g; // Dirichlet: 1/pivot_i for i < ntab
    int ntab;
    int halo;            // truncation halo per side (segment mode), 0 = whole line
    int tile;            // output points per item along x
    int nseg;            // items per x-line (1 = whole-line exact mode)
    double pw[kMaxChunk];  // pw[e] = lam^(e+1): carry weights of a constant-coefficient chunk
    double zf4[4], zf8[8], zf16[16];  // forward-carry response of a backward chunk pass (K = 4/8/16)
    double mp8[10], mp16[10];         // M^(2^i), M = lam^K (repeated squaring of pw[K-1]), K = 8/16
    long long* dbg;                // optional phase trace (RIDC_PHASE_TIMING), CTA 0 only
};

// Checked build (RIDC_CHECKED: __graft_entry__.build(checked=True) ->
// libridc_b200_checked.so): bounds and protocol assertions in the kernels, in
// place of compute-sanitizer (closed on the GPU pool).  A failed check prints
// the site and traps, which surfaces as a CUDA error on the host.
#ifdef RIDC_CHECKED
#define RIDC_CHECK(cond)                                                                     \
    do {                                                                                     \
        if (!(cond)) {                                                                       \
            printf("RIDC_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__,   \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                            \
            __trap();                                                                        \
        }                                                                                    \
    } while (0)
#else
#define RIDC_CHECK(cond) do { } while (0)
#endif

// Phase trace: CTA 0, thread 0, first 8 items of a launch, 16 stamps each.
#define RIDC_STAMP(sv, item_no, idx)                                                         \
    do {                                                                                     \
        if (threadIdx.x == 0 && blockIdx.x == 0 && (sv).dbg && (item_no) < 8)                \
            (sv).dbg[(item_no) * 16 + (idx)] = clock64();                                    \
    } while (0)

struct StepItem {
    int nnodes;
    int level;
    long long target;
    const double* vec[kMaxNodes];
    double ca[kMaxNodes], cs[kMaxNodes], cn[kMaxNodes];
    double* out;
    double* out2;   // optional mirror (the consumer GPU's inbox slot, written over NVLink)
    int omap1;      // tensor map of the output ring + 1 (0: no TMA store -- plain stores)
    int opad;
    long long oslot;   // slot of `out` in that ring
    int vlev[kMaxNodes];          // ring (level) of node a   (tensor-map staging)
    long long vslot[kMaxNodes];   // slot of node a in that ring
};

struct Aff { double A, B; };   // y -> A*y + B

__device__ __forceinline__ Aff compose(Aff later, Aff earlier)
{
    return Aff{later.A * earlier.A, fma(later.A, earlier.B, later.B)};
}

// Shared-memory index with one pad double every 16: a thread owning E
// consecutive elements (E in {8,16}) then hits distinct 8-byte banks.
__device__ __forceinline__ int pad(int p) { return p + (p >> 4); }

__device__ __forceinline__ double ld_ro(const double* p) { return __ldg(p); }

// Value of row `rp` at column `col`, periodic wrap or zero Dirichlet ghost.
__device__ __forceinline__ double at(const double* rp, int col, int nx, bool periodic)
{
    if (col < 0) {
        if (!periodic) return 0.0;
        col += nx;
    } else if (col >= nx) {
        if (!periodic) return 0.0;
        col -= nx;
    }
    return ld_ro(rp + col);
}

// f^S and f^N at one point.  need_s / need_n skip unused halves (warp-uniform).
template <int KIND>
__device__ __forceinline__ void eval_point(const DevProblem& pb, const double* rp,
                                           const double* rn, const double* rs, int col,
                                           bool need_s, bool need_n, double& u, double& fs,
                                           double& fn)
{
    const int nx = pb.nx;
    constexpr bool periodic = KIND != BURGERS_1D;
    u = at(rp, col, nx, periodic);
    fs = 0.0;
    fn = 0.0;
    double ul = 0.0, ur = 0.0;
    const bool need_l = need_s || (need_n && KIND == BURGERS_1D);
    const bool need_r = need_s || (need_n && (KIND == BURGERS_1D || KIND == ADV_DIFF_1D ||
                                              KIND == ADV_DIFF_2D));
    if (need_l) ul = at(rp, col - 1, nx, periodic);
    if (need_r) ur = at(rp, col + 1, nx, periodic);
    if (need_s) fs = pb.cdx * (ul - 2.0 * u + ur);
    if (need_n) {
        if (KIND == ADV_DIFF_1D) {
            fn = pb.cax * (ur - u);
        } else if (KIND == BURGERS_1D) {
            fn = -(ur * ur - ul * ul) * pb.bs;
        } else if (KIND == RD_1D) {
            fn = pb.rho * u * (1.0 - u);
        } else {
            int c = col < 0 ? col + nx : (col >= nx ? col - nx : col);
            double un = ld_ro(rn + c), us = ld_ro(rs + c);
            double yd = pb.cdy * (un - 2.0 * u + us);
            if (KIND == ADV_DIFF_2D)
                fn = pb.cax * (ur - u) + pb.cay * (us - u) + yd;
            else
                fn = pb.rho * u * (1.0 - u) + yd;
        }
    }
}

// Barrier over the NT compute threads only (named barrier 1); a producer
// warp, when present, never joins it.
template <int N>
__device__ __forceinline__ void csync()
{
    asm volatile("bar.sync 1, %0;" ::"r"(N) : "memory");
}

// Block-wide exclusive scan of affine maps in thread order (reverse: from the
// last thread down).  Returns the composition of all chunks before this
// thread's; `total` receives the composition over the whole block.
// swarp needs 2*NW+1 entries: warp totals, then warp prefixes + block total.
template <int NT>
__device__ __forceinline__ Aff block_scan(Aff mine, bool reverse, Aff* swarp, Aff& total)
{
    constexpr int NW = NT / 32;
    static_assert(NW <= 32, "one warp scans the warp totals");
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Aff inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double A = reverse ? __shfl_down_sync(FULL, inc.A, d) : __shfl_up_sync(FULL, inc.A, d);
        double B = reverse ? __shfl_down_sync(FULL, inc.B, d) : __shfl_up_sync(FULL, inc.B, d);
        const bool ok = reverse ? (lane + d < 32) : (lane >= d);
        if (ok) inc = compose(inc, Aff{A, B});
    }
    double eA = reverse ? __shfl_down_sync(FULL, inc.A, 1) : __shfl_up_sync(FULL, inc.A, 1);
    double eB = reverse ? __shfl_down_sync(FULL, inc.B, 1) : __shfl_up_sync(FULL, inc.B, 1);
    const bool first = reverse ? (lane == 31) : (lane == 0);
    const Aff exc = first ? Aff{1.0, 0.0} : Aff{eA, eB};
    const bool last = reverse ? (lane == 0) : (lane == 31);
    if (last) swarp[warp] = inc;
    csync<NT>();
    if (warp == 0) {
        // lane l holds the l-th warp total in scan order
        const int w = reverse ? NW - 1 - lane : lane;
        Aff t = lane < NW ? swarp[w] : Aff{1.0, 0.0};
        Aff ti = t;
#pragma unroll
        for (int d = 1; d < NW; d <<= 1) {
            const double A = __shfl_up_sync(FULL, ti.A, d);
            const double B = __shfl_up_sync(FULL, ti.B, d);
            if (lane >= d) ti = compose(ti, Aff{A, B});
        }
        const double pA = __shfl_up_sync(FULL, ti.A, 1);
        const double pB = __shfl_up_sync(FULL, ti.B, 1);
        if (lane < NW) swarp[NW + w] = lane == 0 ? Aff{1.0, 0.0} : Aff{pA, pB};
        if (lane == NW - 1) swarp[2 * NW] = ti;
    }
    csync<NT>();
    total = swarp[2 * NW];
    return compose(exc, swarp[NW + warp]);
}

__device__ __forceinline__ void coef(const DevSolve& sv, int col, double& m, double& g)
{
    if (col >= 0 && col < sv.ntab) {
        m = sv.tab_m[col];
        g = sv.tab_g[col];
    } else {
        m = sv.lam;
        g = sv.g;
    }
}

// Encode (target, level) so that atomicMin keeps the earliest failing step.
__device__ __forceinline__ unsigned long long err_code(long long target, int level)
{
    return ((unsigned long long)target << 8) | (unsigned long long)level;
}

// Shared-memory layout of one item (doubles): the padded buffer used for
// the x-stencil neighbours and then for the recurrences.
template <int NT, int KMAX>
struct Smem {
    static constexpr int NW = NT / 32;
    static constexpr int CAP = NT * KMAX;
    static constexpr int TOTAL = CAP + CAP / 16 + 1;
};

// Geometry of one item.  Positions q = 0..Q-1 map to columns c_first + q
// (c_first = s0 - 1): the extended range plus one stencil neighbour on each
// side.  rhs lives on q in [1, Q-1).
struct Geo {
    int item_no;           // ordinal of the item within its CTA (phase trace)
    int row, seg, c0, tlen;
    int s0, S, out_lo;     // extended range [s0, s0+S), outputs at p in [out_lo, out_lo+tlen)
    bool cyclic;
    bool fast;             // truncated segment: no wrap / ghosts / coefficient tables
};

template <int KIND, int NT, int KMAX>
__device__ __forceinline__ Geo make_geo(const DevProblem& pb, const DevSolve& sv, int tile)
{
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr int CAP = NT * KMAX;
    Geo g;
    g.item_no = 0;
    g.row = tile / sv.nseg;
    const int seg = tile - g.row * sv.nseg;
    g.seg = seg;
    const int nx = pb.nx;
    g.c0 = seg * sv.tile;
    g.tlen = min(sv.tile, nx - g.c0);
    if (sv.nseg == 1) {
        g.s0 = 0; g.S = nx; g.out_lo = 0; g.cyclic = periodic;
    } else if (periodic) {
        g.s0 = g.c0 - sv.halo; g.S = g.tlen + 2 * sv.halo; g.out_lo = sv.halo; g.cyclic = false;
    } else {
        g.s0 = max(g.c0 - sv.halo, 0);
        const int send = min(g.c0 + g.tlen + sv.halo, nx);
        g.S = send - g.s0; g.out_lo = g.c0 - g.s0; g.cyclic = false;
    }
    g.fast = sv.nseg > 1 && g.S + 2 <= CAP && g.s0 - 1 >= 0 && g.s0 + g.S + 1 <= nx &&
             (sv.ntab == 0 || g.s0 - 1 >= sv.ntab);
    return g;
}

// Per-node coefficients of the pointwise accumulation (uniform over an item).
// A window node w with weights (ca, cs, cn) contributes
//   ca w + cn (pointwise parts of f^N(w)) + cs f^S(w) + cn (x-parts of f^N(w)),
// the pointwise part factored per kind so that it costs 1-3 FMAs per point:
//   RD_1D   ca w + cn rho w(1-w)                    = (a + b w) w
//   RD_2D   ... + cn dyy (wn - 2w + ws)             = (a + b w) w + c (wn + ws)
//   AD_2D   ca w + cn (cy (ws - w) + dyy (wn - 2w + ws)) = a w + b ws + c wn
//   AD_1D, Burgers: ca w (the x-advection / flux goes through WX)
struct NodeCoef {
    double a, b, c;   // pointwise factors (see above)
    double cs, cn;    // weights of the x-stencil accumulators
};

template <int KIND>
__host__ __device__ __forceinline__ NodeCoef node_coef(const DevProblem& pb, double ca, double cs, double cn)
{
    NodeCoef k;
    k.cs = cs;
    k.cn = cn;
    k.b = 0.0;
    k.c = 0.0;
    if (KIND == RD_1D) {
        k.a = fma(cn, pb.rho, ca);
        k.b = -(cn * pb.rho);
    } else if (KIND == RD_2D) {
        k.a = fma(-2.0 * cn, pb.cdy, fma(cn, pb.rho, ca));
        k.b = -(cn * pb.rho);
        k.c = cn * pb.cdy;
    } else if (KIND == ADV_DIFF_2D) {
        k.a = fma(-2.0 * cn, pb.cdy, fma(-cn, pb.cay, ca));
        k.b = cn * (pb.cay + pb.cdy);
        k.c = cn * pb.cdy;
    } else {
        k.a = ca;
    }
    return k;
}

// Fold one node value into the pointwise accumulators (see NodeCoef):
//   P += pointwise part, WS += cs w, WX += cn w (x-advection) | cn w^2 (Burgers).
// Branch-free: zero coefficients cost an FMA, never a select (callers keep
// vn / vs finite -- zero when the y-neighbours were not loaded).
template <int KIND>
__device__ __forceinline__ void accumulate_point(const NodeCoef& k, double v, double vn, double vs, double& P,
                                                 double& WS, double& WX)
{
    if (KIND == RD_1D) {
        P = fma(fma(k.b, v, k.a), v, P);
    } else if (KIND == RD_2D) {
        P = fma(k.c, vn + vs, fma(fma(k.b, v, k.a), v, P));
    } else if (KIND == ADV_DIFF_2D) {
        P = fma(k.c, vn, fma(k.b, vs, fma(k.a, v, P)));
    } else {
        P = fma(k.a, v, P);
    }
    WS = fma(k.cs, v, WS);
    if (KIND == BURGERS_1D) WX = fma(k.cn, v * v, WX);
    else if (KIND == ADV_DIFF_1D || KIND == ADV_DIFF_2D) WX = fma(k.cn, v, WX);
}

template <int KMAX>
__device__ __forceinline__ const double* zf_of(const DevSolve& sv)
{
    return KMAX == 4 ? sv.zf4 : (KMAX == 8 ? sv.zf8 : sv.zf16);
}

// Constant-coefficient solve of a truncated segment held as KMAX consecutive
// points per thread (thread t owns chunk t).  Both local recurrences run
// first (zero carries); the chunk-to-chunk carries then need only the B
// halves of the affine maps because every chunk multiplier is M = lam^KMAX:
//   forward  c_t = sum_{u<t} M^{t-1-u} Bf_u,
//   backward d_t = sum_{u>t} M^{u-t-1} (Bb_u + c_u zf_0),
// each a warp shuffle scan plus a scan of the warp totals that every warp
// repeats redundantly (one barrier per direction).  Finally
//   x_e = xloc_e + c_t zf_e + d_t lam^(KMAX-e).
template <int KMAX>
__device__ __forceinline__ const double* mp_of(const DevSolve& sv)
{
    static_assert(KMAX == 8 || KMAX == 16, "carry-power tables exist for K = 8 and 16");
    return KMAX == 8 ? sv.mp8 : sv.mp16;
}

// Per-lane carry powers of fast_solve: M^lane and M^(31-lane).  Loop-invariant:
// callers that solve many chunks compute them once.
struct FastLane { double ml, mr; };

template <int KMAX>
__device__ __forceinline__ FastLane fast_lane(const DevSolve& sv)
{
    const double* mp = mp_of<KMAX>(sv);
    const int lane = threadIdx.x & 31;
    double ml = 1.0, mr = 1.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (lane & (1 << i)) ml *= mp[i];
        if ((31 - lane) & (1 << i)) mr *= mp[i];
    }
    return FastLane{ml, mr};
}

template <int NT, int KMAX, bool CYCLIC = false>
__device__ __forceinline__ void fast_solve(const DevSolve& sv, double (&vv)[KMAX], double* sx, FastLane fl)
{
    static_assert(!CYCLIC || (NT & (NT - 1)) == 0, "cyclic closure needs a power-of-two thread count");
    constexpr int NW = NT / 32;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double m = sv.lam, g = sv.g;
    const double* zf = zf_of<KMAX>(sv);
    const double* mp = mp_of<KMAX>(sv);   // M^(2^i)
    double y = 0.0;
#pragma unroll
    for (int e = 0; e < KMAX; ++e) { y = fma(m, y, g * vv[e]); vv[e] = y; }
    const double bf = y;
    double x = 0.0;
#pragma unroll
    for (int e = KMAX - 1; e >= 0; --e) { x = fma(m, x, vv[e]); vv[e] = x; }
    const double bb = x;
    const double ml = fl.ml, mr = fl.mr;   // M^lane and M^(31-lane)
    // ---- forward carries
    double inc = bf;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const double t = __shfl_up_sync(FULL, inc, 1 << i);
        if (lane >= (1 << i)) inc = fma(mp[i], t, inc);
    }
    if (lane == 31) sx[warp] = inc;
    double ex = __shfl_up_sync(FULL, inc, 1);
    if (lane == 0) ex = 0.0;
    csync<NT>();
    double wi = lane < NW ? sx[lane] : 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if ((1 << i) >= NW) break;
        const double t = __shfl_up_sync(FULL, wi, 1 << i);
        if (lane >= (1 << i)) wi = fma(mp[5 + i], t, wi);
    }
    double cw = __shfl_sync(FULL, wi, warp > 0 ? warp - 1 : 0);
    if (warp == 0) cw = 0.0;
    double cf = fma(ml, cw, ex);
    // cyclic whole line of NT full chunks: y_{-1} = y_{S-1} = T_f / (1 - lam^S),
    // entering chunk t as M^t y_{-1}  (M^t = M^lane * (M^32)^warp)
    double mwf = 1.0, mwb = 1.0, mS = 1.0;
    if (CYCLIC) {
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if ((1 << (5 + i)) >= NT) break;
            if (warp & (1 << i)) mwf *= mp[5 + i];
            if ((NW - 1 - warp) & (1 << i)) mwb *= mp[5 + i];
        }
#pragma unroll
        for (int i = 0; i < 10; ++i)
            if ((1 << i) == NT) mS = mp[i];
        const double tf = __shfl_sync(FULL, wi, NW - 1);
        cf = fma(ml * mwf, tf / (1.0 - mS), cf);
    }
    // ---- backward carries
    double rinc = fma(cf, zf[0], bb);
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const double t = __shfl_down_sync(FULL, rinc, 1 << i);
        if (lane + (1 << i) < 32) rinc = fma(mp[i], t, rinc);
    }
    if (lane == 0) sx[NW + warp] = rinc;
    double exr = __shfl_down_sync(FULL, rinc, 1);
    if (lane == 31) exr = 0.0;
    csync<NT>();
    // reverse warp scan: lane l holds the total of warp NW-1-l
    double wr = lane < NW ? sx[NW + (NW - 1 - lane)] : 0.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if ((1 << i) >= NW) break;
        const double t = __shfl_up_sync(FULL, wr, 1 << i);
        if (lane >= (1 << i)) wr = fma(mp[5 + i], t, wr);
    }
    const int rl = NW - 1 - warp;   // my warp's position in reverse order
    double dw = __shfl_sync(FULL, wr, rl > 0 ? rl - 1 : 0);
    if (rl == 0) dw = 0.0;
    double dc = fma(mr, dw, exr);
    if (CYCLIC) {   // x_S = x_0 = T_b / (1 - lam^S), entering chunk t as M^(NT-1-t) x_S
        const double tb = __shfl_sync(FULL, wr, NW - 1);
        dc = fma(mr * mwb, tb / (1.0 - mS), dc);
    }
#pragma unroll
    for (int e = 0; e < KMAX; ++e) vv[e] = fma(dc, sv.pw[KMAX - 1 - e], fma(cf, zf[e], vv[e]));
}

// Phases 2-5 of an item, shared by the register-load and the TMA-staged paths:
// x-stencils of the accumulators, the two recurrences, the coalesced store.
template <int KIND, int NT, int KMAX, bool FAST>
__device__ __forceinline__ void finish_item(const DevProblem& pb, const DevSolve& sv,
                                            const StepItem& it, const Geo& geo, const double* P,
                                            const double* WS, const double* WX, double* sbuf,
                                            Aff* swarp, unsigned long long* err)
{
    constexpr int CAP = NT * KMAX;
    constexpr bool has_wx = KIND == ADV_DIFF_1D || KIND == BURGERS_1D || KIND == ADV_DIFF_2D;
    const int nx = pb.nx;
    const int tid = threadIdx.x;
    const int cf = geo.s0 - 1;
    const int Q = geo.S + 2;
    const size_t rbase = (size_t)geo.row * nx;
    auto valid = [&](int q) { return q < Q; };
    (void)nx;
    const int ino = geo.item_no;
    RIDC_STAMP(sv, ino, 2);
    // ---- phase 2: x-stencils of WS (then WX) through shared memory
    // (FAST: every position is computed; rhs outside [1, Q-1) is zeroed below)
    // Strided position q = tid + k*NT has padded index pq + k*SK (NT is a multiple
    // of 16); its neighbours sit at pq + k*SK + dm / + dp.
    constexpr int SK = NT + NT / 16;
    const int pq = pad(tid);
    const int dm = pad(tid + NT - 1) - NT - NT / 16 - pq;   // pad(q-1) - pad(q)  (tid-1, wrapped into the row above)
    const int dp = pad(tid + 1) - pq;                       // pad(q+1) - pad(q)
    bool need_ws = false, need_wx = false;
    for (int a = 0; a < it.nnodes; ++a) {
        need_ws |= it.cs[a] != 0.0;
        need_wx |= it.cn[a] != 0.0;
    }
    need_wx = need_wx && has_wx;
    double rhs[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) rhs[k] = P[k];
    if (need_ws) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (FAST || valid(tid + k * NT)) sbuf[pq + k * SK] = WS[k];
        csync<NT>();
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int q = tid + k * NT;
            if (FAST ? (q >= 1 && q < CAP - 1) : (q >= 1 && q < Q - 1))
                rhs[k] = fma(pb.cdx, (sbuf[pq + k * SK + dm] - 2.0 * WS[k]) + sbuf[pq + k * SK + dp], rhs[k]);
        }
        csync<NT>();
    }
    if (need_wx) {
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            if (FAST || valid(tid + k * NT)) sbuf[pq + k * SK] = WX[k];
        csync<NT>();
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int q = tid + k * NT;
            if (FAST ? (q >= 1 && q < CAP - 1) : (q >= 1 && q < Q - 1)) {
                if (KIND == BURGERS_1D)
                    rhs[k] = fma(-pb.bs, sbuf[pq + k * SK + dp] - sbuf[pq + k * SK + dm], rhs[k]);
                else
                    rhs[k] = fma(pb.cax, sbuf[pq + k * SK + dp] - WX[k], rhs[k]);
            }
        }
        csync<NT>();
    }
    // scan coordinates: FAST scans all CAP positions (rhs 0 outside [1, Q-1):
    // those lie in the truncation halo); otherwise e = q - 1 in [0, S).
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const int q = tid + k * NT;
        if (FAST) sbuf[pq + k * SK] = (q == 0 || q >= Q - 1) ? 0.0 : rhs[k];
        else if (q >= 1 && q < Q - 1) sbuf[pad(q - 1)] = rhs[k];
    }
    csync<NT>();
    RIDC_STAMP(sv, ino, 3);
    // ---- phases 3-4: y_i = g_i rhs_i + m_i y_{i-1}, then x_i = y_i + m_i x_{i+1}
    const int S = FAST ? CAP : geo.S;
    const int e0 = FAST ? cf : geo.s0;          // column of scan index 0
    const int base = tid * KMAX;
    const int nm = FAST ? KMAX : max(0, min(KMAX, S - base));
    double vv[KMAX];
    static_assert(16 % KMAX == 0 || KMAX % 16 == 0, "chunk padding assumes KMAX | 16 or 16 | KMAX");
    const int pc = pad(base);   // pad(base + e) == pc + e for e < KMAX
#pragma unroll
    for (int e = 0; e < KMAX; ++e) vv[e] = (FAST || e < nm) ? sbuf[pc + e] : 0.0;
    const bool cmode = FAST || (sv.ntab == 0) || (e0 + base >= sv.ntab);
    const double m = sv.lam, g = sv.g;
    if constexpr (FAST) {
        RIDC_STAMP(sv, ino, 4);
        fast_solve<NT, KMAX>(sv, vv, reinterpret_cast<double*>(swarp), fast_lane<KMAX>(sv));
        RIDC_STAMP(sv, ino, 7);
    } else {
    {
        double y = 0.0, A = 1.0;
        if (cmode) {
#pragma unroll
            for (int e = 0; e < KMAX; ++e)
                if (FAST || e < nm) { y = fma(m, y, g * vv[e]); vv[e] = y; }
            A = FAST ? sv.pw[KMAX - 1] : (nm > 0 ? sv.pw[nm - 1] : 1.0);
        } else {
#pragma unroll
            for (int e = 0; e < KMAX; ++e)
                if (e < nm) {
                    double mm, gg;
                    coef(sv, e0 + base + e, mm, gg);
                    y = fma(mm, y, gg * vv[e]);
                    A *= mm;
                    vv[e] = y;
                }
        }
        Aff tot;
        RIDC_STAMP(sv, ino, 4);
        const Aff pre = block_scan<NT>(Aff{A, y}, false, swarp, tot);
        RIDC_STAMP(sv, ino, 5);
        const double yinit = (!FAST && geo.cyclic) ? tot.B / (1.0 - tot.A) : 0.0;
        const double cin = fma(pre.A, yinit, pre.B);
        if (cmode) {
#pragma unroll
            for (int e = 0; e < KMAX; ++e)
                if (FAST || e < nm) vv[e] = fma(sv.pw[e], cin, vv[e]);
        } else {
            double Pm = 1.0;
#pragma unroll
            for (int e = 0; e < KMAX; ++e)
                if (e < nm) {
                    double mm, gg;
                    coef(sv, e0 + base + e, mm, gg);
                    Pm *= mm;
                    vv[e] = fma(Pm, cin, vv[e]);
                }
        }
    }
    {
        double x = 0.0, A = 1.0;
        if (cmode) {
#pragma unroll
            for (int e = KMAX - 1; e >= 0; --e)
                if (FAST || e < nm) { x = fma(m, x, vv[e]); vv[e] = x; }
            A = FAST ? sv.pw[KMAX - 1] : (nm > 0 ? sv.pw[nm - 1] : 1.0);
        } else {
#pragma unroll
            for (int e = KMAX - 1; e >= 0; --e)
                if (e < nm) {
                    double mm, gg;
                    coef(sv, e0 + base + e, mm, gg);
                    x = fma(mm, x, vv[e]);
                    A *= mm;
                    vv[e] = x;
                }
        }
        Aff tot;
        RIDC_STAMP(sv, ino, 6);
        const Aff pre = block_scan<NT>(Aff{A, x}, true, swarp, tot);
        RIDC_STAMP(sv, ino, 7);
        const double xinit = (!FAST && geo.cyclic) ? tot.B / (1.0 - tot.A) : 0.0;
        const double cin = fma(pre.A, xinit, pre.B);
        if (cmode) {
#pragma unroll
            for (int e = 0; e < KMAX; ++e)
                if (FAST || e < nm) vv[e] = fma(sv.pw[(FAST ? KMAX : nm) - 1 - e], cin, vv[e]);
        } else {
            double Pm = 1.0;
#pragma unroll
            for (int e = KMAX - 1; e >= 0; --e)
                if (e < nm) {
                    double mm, gg;
                    coef(sv, e0 + base + e, mm, gg);
                    Pm *= mm;
                    vv[e] = fma(Pm, cin, vv[e]);
                }
        }
    }
    }
#pragma unroll
    for (int e = 0; e < KMAX; ++e)
        if (FAST || e < nm) sbuf[pc + e] = vv[e];
    csync<NT>();

    RIDC_STAMP(sv, ino, 8);
    // ---- phase 5: coalesced store of the tile + fused finite check
    // finite check folded into one FMA per point: x*0 is NaN iff x is Inf/NaN
    double chk = 0.0;
    double* orow = it.out + rbase + e0;
    double* orow2 = it.out2 ? it.out2 + rbase + e0 : nullptr;
    const int olo = FAST ? geo.out_lo + 1 : geo.out_lo;   // in scan coordinates
    if (orow2) {   // pipeline: also the peer store into the next level's inbox (NVLink)
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int e = tid + k * NT;
            if ((unsigned)(e - olo) < (unsigned)geo.tlen) {
                const double xo = sbuf[pq + k * SK];
                chk = fma(xo, 0.0, chk);
                orow[e] = xo;
                orow2[e] = xo;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int e = tid + k * NT;
            if ((unsigned)(e - olo) < (unsigned)geo.tlen) {
                const double xo = sbuf[pq + k * SK];
                chk = fma(xo, 0.0, chk);
                orow[e] = xo;
            }
        }
    }
    const bool bad = chk != chk;
    if (bad) atomicMin(err, err_code(it.target, it.level));
    RIDC_STAMP(sv, ino, 9);
}

// One work item (FAST: interior segment, every position valid, constant
// coefficients -- no predication anywhere).  smem: Smem<NT,KMAX>::TOTAL doubles.
//
// Phase 1 streams the (j+2) node states once, all loads of a node in flight
// together (the next node's are issued before the current one is consumed).
// The operators are linear in the window states except the pointwise
// reaction and the Burgers flux (linear in u^2), so the window contributes
// through three pointwise accumulators:
//   P  = sum ca_k u_k + sum cn_k (pointwise parts of f^N: reaction, y-stencil)
//   WS = sum cs_k u_k          (f^S applied once: cdx * second difference)
//   WX = sum cn_k u_k | u_k^2  (x-advection / Burgers flux applied once)
// Phase 2 applies the x-stencils through shared memory; phases 3-4 run the
// two first-order recurrences on register chunks with block-wide affine
// scans; phase 5 stores the tile coalesced with the fused finite check.
template <int KIND, int NT, int KMAX, bool FAST>
__device__ __forceinline__ void item_body(const DevProblem& pb, const DevSolve& sv,
                                          const StepItem& it, const Geo& geo, double* sbuf,
                                          Aff* swarp, unsigned long long* err)
{
    constexpr int CAP = NT * KMAX;
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr bool two_d = KIND == ADV_DIFF_2D || KIND == RD_2D;
    constexpr bool has_wx = KIND == ADV_DIFF_1D || KIND == BURGERS_1D || KIND == ADV_DIFF_2D;
    constexpr bool prefetch = !two_d;
    const int nx = pb.nx, ny = pb.ny;
    const int tid = threadIdx.x;
    const int row = geo.row;
    const int cf = geo.s0 - 1;              // column of q = 0
    const int Q = geo.S + 2;
    const size_t rbase = (size_t)row * nx;
    const size_t rn_base = (size_t)(row == 0 ? ny - 1 : row - 1) * nx;
    const size_t rs_base = (size_t)(row == ny - 1 ? 0 : row + 1) * nx;

    auto valid = [&](int q) { return q < Q; };
    auto col_of = [&](int q) {
        int c = cf + q;
        if (!FAST && periodic) c = c < 0 ? c + nx : (c >= nx ? c - nx : c);
        return c;
    };
    auto ghost = [&](int q) { return !FAST && !periodic && (cf + q < 0 || cf + q >= nx); };

    // ---- phase 1: pointwise accumulation over all nodes
    double P[KMAX], WS[KMAX], WX[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) { P[k] = 0.0; WS[k] = 0.0; WX[k] = 0.0; }

    double ua[KMAX], ub[KMAX], un[KMAX], us[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) { un[k] = 0.0; us[k] = 0.0; }
    auto load = [&](int a, double* u) {
        const double* rp = it.vec[a] + rbase;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int q = tid + k * NT;
            u[k] = 0.0;
            if (valid(q) && !ghost(q)) u[k] = ld_ro(rp + col_of(q));
        }
    };
    auto load_y = [&](int a) {
        const double* rn = it.vec[a] + rn_base;
        const double* rs = it.vec[a] + rs_base;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int q = tid + k * NT;
            un[k] = 0.0;
            us[k] = 0.0;
            if (valid(q)) {
                const int c = col_of(q);
                un[k] = ld_ro(rn + c);
                us[k] = ld_ro(rs + c);
            }
        }
    };
    auto accumulate = [&](int a, const double* u) {
        const NodeCoef nc = node_coef<KIND>(pb, it.ca[a], it.cs[a], it.cn[a]);
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
            accumulate_point<KIND>(nc, u[k], two_d ? un[k] : 0.0, two_d ? us[k] : 0.0, P[k], WS[k], WX[k]);
    };
    const int nn = it.nnodes;
    if (prefetch) {
        load(0, ua);
        for (int a = 0; a < nn; a += 2) {
            if (a + 1 < nn) load(a + 1, ub);
            accumulate(a, ua);
            if (a + 1 < nn) {
                if (a + 2 < nn) load(a + 2, ua);
                accumulate(a + 1, ub);
            }
        }
    } else {
        for (int a = 0; a < nn; ++a) {
            load(a, ua);
            if (two_d && it.cn[a] != 0.0) load_y(a);
            accumulate(a, ua);
        }
    }

    finish_item<KIND, NT, KMAX, FAST>(pb, sv, it, geo, P, WS, WX, sbuf, swarp, err);
}

template <int KIND, int NT, int KMAX>
__device__ __forceinline__ void process_item(const DevProblem& pb, const DevSolve& sv,
                                             const StepItem& it, int tile, double* sbuf,
                                             Aff* swarp, unsigned long long* err)
{
    const Geo geo = make_geo<KIND, NT, KMAX>(pb, sv, tile);
    if (geo.fast)
        item_body<KIND, NT, KMAX, true>(pb, sv, it, geo, sbuf, swarp, err);
    else
        item_body<KIND, NT, KMAX, false>(pb, sv, it, geo, sbuf, swarp, err);
}

}  // namespace ridc
