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

namespace ridc {

enum Kind { ADV_DIFF_1D = 1, BURGERS_1D = 2, RD_1D = 3, ADV_DIFF_2D = 4, RD_2D = 5 };

constexpr int kMaxLevels = 12;              // engine.py:47 (MAX_LEVEL + 1)
constexpr int kMaxNodes = 2 * kMaxLevels + 1;  // own state + window (states, or f^S and f^N rows)

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
};

struct StepItem {
    int nnodes;
    int level;
    long long target;
    const double* vec[kMaxNodes];
    double ca[kMaxNodes], cs[kMaxNodes], cn[kMaxNodes];
    double* out;
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

// Block-wide exclusive scan of affine maps in thread order (reverse: from the
// last thread down).  Returns the composition of all chunks before this
// thread's; `total` receives the composition over the whole block.
template <int NT>
__device__ __forceinline__ Aff block_scan(Aff mine, bool reverse, Aff* swarp, Aff& total)
{
    constexpr int NW = NT / 32;
    const unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    Aff inc = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        double A = reverse ? __shfl_down_sync(FULL, inc.A, d) : __shfl_up_sync(FULL, inc.A, d);
        double B = reverse ? __shfl_down_sync(FULL, inc.B, d) : __shfl_up_sync(FULL, inc.B, d);
        bool ok = reverse ? (lane + d < 32) : (lane >= d);
        if (ok) inc = compose(inc, Aff{A, B});
    }
    double eA = reverse ? __shfl_down_sync(FULL, inc.A, 1) : __shfl_up_sync(FULL, inc.A, 1);
    double eB = reverse ? __shfl_down_sync(FULL, inc.B, 1) : __shfl_up_sync(FULL, inc.B, 1);
    const bool first = reverse ? (lane == 31) : (lane == 0);
    Aff exc = first ? Aff{1.0, 0.0} : Aff{eA, eB};
    const bool last = reverse ? (lane == 0) : (lane == 31);
    if (last) swarp[warp] = inc;
    __syncthreads();
    Aff wp{1.0, 0.0}, tot{1.0, 0.0};
    if (!reverse) {
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            Aff s = swarp[w];
            if (w < warp) wp = compose(s, wp);
            tot = compose(s, tot);
        }
    } else {
#pragma unroll
        for (int w = NW - 1; w >= 0; --w) {
            Aff s = swarp[w];
            if (w > warp) wp = compose(s, wp);
            tot = compose(s, tot);
        }
    }
    __syncthreads();
    total = tot;
    return compose(exc, wp);
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

// One work item.  sbuf: padded shared buffer of >= pad(NT*KMAX) doubles.
template <int KIND, int NT, int KMAX>
__device__ __forceinline__ void process_item(const DevProblem& pb, const DevSolve& sv,
                                             const StepItem& it, int tile, double* sbuf,
                                             Aff* swarp, unsigned long long* err)
{
    const int nx = pb.nx, ny = pb.ny;
    const int tid = threadIdx.x;
    const int row = tile / sv.nseg;
    const int seg = tile - row * sv.nseg;
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr bool two_d = KIND == ADV_DIFF_2D || KIND == RD_2D;

    // ---- geometry: extended range [s0, s0 + S), outputs at [out_lo, out_lo + tlen)
    const int c0 = seg * sv.tile;
    const int tlen = min(sv.tile, nx - c0);
    int s0, S, out_lo;
    bool exact_l, exact_r, cyclic;
    if (sv.nseg == 1) {
        s0 = 0; S = nx; out_lo = 0;
        cyclic = periodic; exact_l = exact_r = !periodic;
    } else if (periodic) {
        s0 = c0 - sv.halo; S = tlen + 2 * sv.halo; out_lo = sv.halo;
        cyclic = false; exact_l = exact_r = false;
    } else {
        s0 = max(c0 - sv.halo, 0);
        const int send = min(c0 + tlen + sv.halo, nx);
        S = send - s0; out_lo = c0 - s0;
        cyclic = false; exact_l = (s0 == 0); exact_r = (send == nx);
    }
    (void)exact_l; (void)exact_r;

    const size_t rbase = (size_t)row * nx;
    const size_t rn_base = (size_t)(row == 0 ? ny - 1 : row - 1) * nx;
    const size_t rs_base = (size_t)(row == ny - 1 ? 0 : row + 1) * nx;

    // ---- phase 1: fused rhs over the extended range, registers
    double acc[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) acc[k] = 0.0;
    for (int a = 0; a < it.nnodes; ++a) {
        const double* v = it.vec[a];
        const double ca = it.ca[a], cs = it.cs[a], cn = it.cn[a];
        const bool need_s = cs != 0.0, need_n = cn != 0.0;
        const double* rp = v + rbase;
        const double* rn = two_d ? v + rn_base : nullptr;
        const double* rs = two_d ? v + rs_base : nullptr;
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
            const int p = tid + k * NT;
            if (p < S) {
                double u, fs, fn;
                eval_point<KIND>(pb, rp, rn, rs, s0 + p, need_s, need_n, u, fs, fn);
                double t = acc[k];
                if (ca != 0.0) t = t + ca * u;
                if (need_s) t = t + cs * fs;
                if (need_n) t = t + cn * fn;
                acc[k] = t;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const int p = tid + k * NT;
        if (p < S) sbuf[pad(p)] = acc[k];
    }
    __syncthreads();

    // ---- phase 2: forward recurrence y_i = g_i rhs_i + m_i y_{i-1}
    const int E = (S + NT - 1) / NT;
    const int lo = min(tid * E, S), hi = min(lo + E, S);
    {
        double y = 0.0, A = 1.0;
        for (int e = lo; e < hi; ++e) {
            double m, g;
            coef(sv, s0 + e, m, g);
            y = fma(m, y, g * sbuf[pad(e)]);
            A *= m;
            sbuf[pad(e)] = y;
        }
        Aff tot;
        Aff pre = block_scan<NT>(Aff{A, y}, false, swarp, tot);
        const double yinit = cyclic ? tot.B / (1.0 - tot.A) : 0.0;
        const double cin = fma(pre.A, yinit, pre.B);
        if (cin != 0.0) {
            double P = 1.0;
            for (int e = lo; e < hi; ++e) {
                double m, g;
                coef(sv, s0 + e, m, g);
                P *= m;
                sbuf[pad(e)] = fma(P, cin, sbuf[pad(e)]);
            }
        }
    }
    __syncthreads();
    // ---- phase 3: backward recurrence x_i = y_i + m_i x_{i+1}
    {
        double x = 0.0, A = 1.0;
        for (int e = hi - 1; e >= lo; --e) {
            double m, g;
            coef(sv, s0 + e, m, g);
            x = fma(m, x, sbuf[pad(e)]);
            A *= m;
            sbuf[pad(e)] = x;
        }
        Aff tot;
        Aff pre = block_scan<NT>(Aff{A, x}, true, swarp, tot);
        const double xinit = cyclic ? tot.B / (1.0 - tot.A) : 0.0;
        const double cin = fma(pre.A, xinit, pre.B);
        if (cin != 0.0) {
            double P = 1.0;
            for (int e = hi - 1; e >= lo; --e) {
                double m, g;
                coef(sv, s0 + e, m, g);
                P *= m;
                sbuf[pad(e)] = fma(P, cin, sbuf[pad(e)]);
            }
        }
    }
    __syncthreads();

    // ---- phase 4: coalesced store of the tile + fused finite check
    bool bad = false;
    double* orow = it.out + rbase;
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
        const int p = tid + k * NT;
        if (p >= out_lo && p < out_lo + tlen) {
            const double x = sbuf[pad(p)];
            bad |= !isfinite(x);
            orow[s0 + p] = x;
        }
    }
    if (__syncthreads_or(bad) && tid == 0) atomicMin(err, err_code(it.target, it.level));
    // sbuf is reused by the next item only after the caller's barrier
}

}  // namespace ridc
