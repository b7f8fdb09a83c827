// ridc_sweep2d_levels.cuh -- the tick of the lagged level pipeline on 2-D grids
// as row sweeps (all active levels, the x-line-implicit periodic kinds).
//
// One launch per pipeline tick (the tick kernel's schedule: level j computes
// step k - j(j+1)/2, engine.py:363-371).  CTA c owns the row block [r0, r1)
// and, for every active level in turn, streams the rows r0-1 .. r1 of the
// level's nodes -- its own state and the j+1 window states of level j-1, the
// node list and weights of build_item (_window_span / _orient / the lag terms
// of _correct_core, engine.py:124-187) -- through a ring of TMA row stages.
// Each node row q is read ONCE and folded into three right-hand sides:
//   rhs(q-1) += s_a w          (row q is the south neighbour of q-1)   -> registers A
//   rhs(q)   += center_a(w)    (pointwise part, x-diffusion f^S, x-advection) -> registers B
//   rhs(q+1) += n_a w          (row q is the north neighbour of q+1)   -> shared memory C
// with the node coefficients of node_coef (ridc_device.cuh) and g of the solve
// folded in.  After the last node of row q, rhs(q-1) is complete: the cyclic
// x-line solve (the block scans of fast_solve with the closure) and 256-bit
// stores of the level's new row; then B -> A, C -> B.
//
// Bytes per tick: every node row read once, every new row written once --
// SURVEY.md §8d's compulsory 16 B/pt (FEBE) and 8 (j+3) B/pt (level j).  The
// tick kernel stages rows r-1, r, r+1 of every node per x-line item (3 reads
// of each node row from L2).  States agree with the tick kernel to rounding.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"
#include "ridc_sweep.cuh"
#include "ridc_tma.cuh"
// EngineParams, TickParams, build_item: ridc_kernels.cuh (which includes this file after them)

namespace ridc {

// row stages: 5 x 32 KB (nx = 4096) or 2 x 64 KB (nx = 8192), + the north
// accumulator row + the active levels' item descriptors
template <int NT>
struct SweepLevSmem {
    static constexpr int NS = 2;   // (experiment: 2 stages so that two 256-thread CTAs fit an SM)
    static constexpr int ROWB = NT * 128;
    static constexpr size_t OFF_C = (size_t)NS * ROWB;
    static constexpr size_t OFF_BAR = OFF_C + ROWB;
    static constexpr size_t OFF_ITEMS = OFF_BAR + 2 * NS * 8;
    static constexpr size_t bytes(int nact) { return OFF_ITEMS + (size_t)nact * sizeof(StepItem) + 1024; }
};

struct SweepLevParams {
    double lam, g;
    double cyc;                // 1 / (1 - lam^nx)
    double pw[16], zf[16], mp[10];
    int P, GW, gpr, gdata, nx, ny;
};

template <int KIND, int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1)
    k_sweep2d_levels(EngineParams ep, TickParams tp, const __grid_constant__ SweepLevParams sp,
                     const __grid_constant__ TmapSet tm)
{
    static_assert(KIND == ADV_DIFF_2D || KIND == RD_2D, "2-D kinds");
    using S = SweepLevSmem<NT>;
    constexpr int K = 16, NW = NT / 32, NS = S::NS;
    constexpr int BR = NT < 256 ? NT : 256, NBOX = NT / BR;
    extern __shared__ __align__(1024) char smraw[];
    char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    char* cbuf = base + S::OFF_C;                                   // north accumulator row (swizzled groups)
    uint64_t* full = reinterpret_cast<uint64_t*>(base + S::OFF_BAR);
    uint64_t* empty = full + NS;
    StepItem* items = reinterpret_cast<StepItem*>(base + S::OFF_ITEMS);
    __shared__ double sx[2 * NW];
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int ny = sp.ny;
    const int r0 = (int)((long long)cta * ny / G), r1 = (int)((long long)(cta + 1) * ny / G);
    const int nl = r1 - r0 + 2;                                     // rows r0-1 .. r1 per level
    const double lam = sp.lam;

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid < tp.nact) build_item(ep, tp.level[tid], tp.target[tid], items[tid]);
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NW);
        }
        mbar_fence_init();
    }
    double ml = 1.0, mr = 1.0, mwf = 1.0, mwb = 1.0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        if (lane & (1 << i)) ml *= sp.mp[i];
        if ((31 - lane) & (1 << i)) mr *= sp.mp[i];
        if ((1 << (5 + i)) < NT) {
            if (warp & (1 << i)) mwf *= sp.mp[5 + i];
            if ((NW - 1 - warp) & (1 << i)) mwb *= sp.mp[5 + i];
        }
    }
    const double mlc = ml * mwf * sp.cyc, mrc = mr * mwb * sp.cyc;
#pragma unroll
    for (int i = 0; i < K / 2; ++i) sts128(const_cast<char*>(swz(cbuf, tid, i)), 0.0, 0.0);
    __syncthreads();

    // the global sequence of node rows: (level a, row k, node n), in this order
    struct Cursor { int a, k, n; };
    Cursor pc{0, 0, 0};   // thread 0: next node row to load
    long long issued = 0;
    auto issue_next = [&]() {
        if (pc.a >= tp.nact) return;
        const StepItem& it = items[pc.a];
        const int s = (int)(issued % NS);
        if (issued >= NS) mbar_wait(&empty[s], (uint32_t)(((issued - NS) / NS) & 1));
        int q = r0 - 1 + pc.k;
        q = q < 0 ? q + ny : (q >= ny ? q - ny : q);
        RIDC_CHECK(q >= 0 && q < ny && it.vlev[pc.n] >= 0 && it.vlev[pc.n] < ep.levels &&
                   it.vslot[pc.n] >= 0 && it.vslot[pc.n] < ep.cap[it.vlev[pc.n]]);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(NBOX * BR * 128));
        for (int b = 0; b < NBOX; ++b)
            tma_load_3d(base + (size_t)s * S::ROWB + b * BR * 128, &tm.map[it.vlev[pc.n]], 0,
                        q * sp.gpr + sp.gdata + b * BR, (int)it.vslot[pc.n], &full[s]);
        ++issued;
        if (++pc.n == it.nnodes) {
            pc.n = 0;
            if (++pc.k == nl) { pc.k = 0; ++pc.a; }
        }
    };
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0)
        for (int i = 0; i < NS; ++i) issue_next();

    auto solve = [&](double (&v)[K]) {   // the cyclic x-line solve (ridc_sweep2d.cuh)
        double y = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e) {
            y = fma(lam, y, v[e]);
            v[e] = y;
        }
        double inc = y;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const double t = __shfl_up_sync(FULL, inc, 1 << i);
            if (lane >= (1 << i)) inc = fma(sp.mp[i], t, inc);
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
            if (lane >= (1 << i)) wi = fma(sp.mp[5 + i], t, wi);
        }
        double cw = __shfl_sync(FULL, wi, warp > 0 ? warp - 1 : 0);
        if (warp == 0) cw = 0.0;
        const double tf = __shfl_sync(FULL, wi, NW - 1);
        const double cf = fma(mlc, tf, fma(ml, cw, ex));
        double x = 0.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e) {
            x = fma(lam, x, v[e]);
            v[e] = x;
        }
        double rinc = fma(cf, sp.zf[0], x);
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            const double t = __shfl_down_sync(FULL, rinc, 1 << i);
            if (lane + (1 << i) < 32) rinc = fma(sp.mp[i], t, rinc);
        }
        if (lane == 0) sx[NW + warp] = rinc;
        double exr = __shfl_down_sync(FULL, rinc, 1);
        if (lane == 31) exr = 0.0;
        csync<NT>();
        double wr = lane < NW ? sx[NW + (NW - 1 - lane)] : 0.0;
#pragma unroll
        for (int i = 0; i < 5; ++i) {
            if ((1 << i) >= NW) break;
            const double t = __shfl_up_sync(FULL, wr, 1 << i);
            if (lane >= (1 << i)) wr = fma(sp.mp[5 + i], t, wr);
        }
        const int rl = NW - 1 - warp;
        double dw = __shfl_sync(FULL, wr, rl > 0 ? rl - 1 : 0);
        if (rl == 0) dw = 0.0;
        const double tb = __shfl_sync(FULL, wr, NW - 1);
        const double dc = fma(mrc, tb, fma(mr, dw, exr));
#pragma unroll
        for (int e = 0; e < K; ++e) v[e] = fma(dc, sp.pw[K - 1 - e], fma(cf, sp.zf[e], v[e]));
    };

    const DevProblem& pb = ep.pb;
    long long m = 0;   // node rows consumed
    const int tl = tid > 0 ? tid - 1 : NT - 1, tr = tid + 1 < NT ? tid + 1 : 0;   // periodic x neighbours
    for (int a = 0; a < tp.nact; ++a) {
        const StepItem& it = items[a];
        const int nn = it.nnodes;
        RIDC_CHECK(nn >= 1 && nn <= kMaxNodes && it.out == ep.ring[it.level] + it.oslot * ep.Vs);
        double* const out0 = it.out + sp.GW + tid * K;   // + row * P
        bool bad = false;
        // one grid row (k) of this level: every node's row folded into A, B and C
        auto row = [&](int k, double (&A)[K], double (&B)[K]) {
            const bool last = k + 1 == nl;
            for (int n = 0; n < nn; ++n, ++m) {
                const int s = (int)(m % NS);
                mbar_wait(&full[s], (uint32_t)((m / NS) & 1));
                const char* st = base + (size_t)s * S::ROWB;
                const NodeCoef nc = node_coef<KIND>(pb, it.ca[n], it.cs[n], it.cn[n]);
                const double g = sp.g;
                const double gs = g * (KIND == RD_2D ? nc.c : nc.b);   // south coefficient
                const double gn = g * nc.c;                             // north coefficient
                const double sxx = g * nc.cs * pb.cdx;                  // x-diffusion of the node (f^S)
                const double sax = KIND == ADV_DIFF_2D ? g * nc.cn * pb.cax : 0.0;   // x-advection
                const double ca0 = g * nc.a - 2.0 * sxx - sax, cl = sxx, cr = sxx + sax, cq = g * nc.b;
                double2 w = lds128(swz(st, tid, 0));
                double wprev = lds128(swz(st, tl, 7)).y;   // w_{c-1} of my first point
#pragma unroll
                for (int i = 0; i < K / 2; ++i) {
                    const double2 wn = i + 1 < K / 2 ? lds128(swz(st, tid, i + 1))
                                                     : make_double2(lds128(swz(st, tr, 0)).x, 0.0);
                    A[2 * i] = fma(gs, w.x, A[2 * i]);
                    A[2 * i + 1] = fma(gs, w.y, A[2 * i + 1]);
                    if (!last) {
                        double b0 = fma(cr, w.y, fma(cl, wprev, fma(ca0, w.x, B[2 * i])));
                        double b1 = fma(cr, wn.x, fma(cl, w.x, fma(ca0, w.y, B[2 * i + 1])));
                        if (KIND == RD_2D) {   // the reaction's u^2 part: g b w^2
                            b0 = fma(cq * w.x, w.x, b0);
                            b1 = fma(cq * w.y, w.y, b1);
                        }
                        B[2 * i] = b0;
                        B[2 * i + 1] = b1;
                        char* cp = const_cast<char*>(swz(cbuf, tid, i));
                        const double2 c = lds128(cp);
                        sts128(cp, fma(gn, w.x, c.x), fma(gn, w.y, c.y));
                    }
                    wprev = w.y;
                    w = wn;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
                if (tid == 0) issue_next();
            }
            if (k >= 2) {   // rhs of row r0 - 2 + k complete
                solve(A);
                bad |= !chunk_finite(A);
                double* o = out0 + (size_t)(r0 - 2 + k) * sp.P;
#pragma unroll
                for (int e = 0; e < K; e += 4) stg256(o + e, A[e], A[e + 1], A[e + 2], A[e + 3]);
            }
            // the next row's north part: C -> A (the caller swaps A and B), C = 0
#pragma unroll
            for (int i = 0; i < K / 2; ++i) {
                char* cp = const_cast<char*>(swz(cbuf, tid, i));
                const double2 c = lds128(cp);
                A[2 * i] = c.x;
                A[2 * i + 1] = c.y;
                sts128(cp, 0.0, 0.0);
            }
        };
        double A[K], B[K];
#pragma unroll
        for (int e = 0; e < K; ++e) {
            A[e] = 0.0;
            B[e] = 0.0;
        }
        for (int k = 0; k < nl; k += 2) {
            row(k, A, B);
            if (k + 1 < nl) row(k + 1, B, A);
        }
        if (bad) atomicMin(ep.err, err_code(it.target, it.level));
    }
    // the bulk loads all landed (every issued row was consumed): nothing in flight at exit
}

}  // namespace ridc
