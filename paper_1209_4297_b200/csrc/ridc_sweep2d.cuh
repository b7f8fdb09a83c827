// ridc_sweep2d.cuh -- streaming FEBE step on 2-D grids (RIDC order 1; the
// x-line-implicit advection-diffusion and reaction-diffusion kinds, periodic).
//
// One launch per time step.  CTA c owns the row block [r0, r1) and streams the
// previous state's rows r0-1 .. r1 through NSTAGE TMA row stages, each row read
// ONCE: the explicit y-coupling of f^N (problems.py analogue of the 2-D
// SplitIVP, SURVEY.md §7 hard part 5) is linear in the north and south rows, so
// a loaded row q contributes to three right-hand sides at once
//   rhs(q-1) += s_coef w_q        (q is row q-1's south neighbour) -> rhs(q-1) complete
//   rhs(q)   += center(w_q)       (the pointwise part and the x-advection)
//   rhs(q+1)  = n_coef w_q        (q is row q+1's north neighbour)
// with g of the solve folded into every coefficient.  A completed rhs(q-1)
// goes straight into the cyclic x-line solve (fast_solve's constant-multiplier
// block scans + the closure y_{-1} = T / (1 - lam^nx)) and leaves with 256-bit
// stores.  Two register arrays rotate along the sweep; the row is re-read from
// shared memory rather than kept in registers.
//
// Traffic per step: every row read once (+ 2 boundary rows per block) and
// written once: 16 B/pt, SURVEY.md §8d's compulsory figure (the tick kernel
// stages rows r-1, r, r+1 per x-line item: 3 reads from L2).
// nx = 16 NT exactly (every thread a full 16-point chunk: the cyclic closure).
// States agree with the tick kernel to rounding (different association).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"
#include "ridc_tma.cuh"

namespace ridc {

constexpr int kSweep2Stages = 3;

template <int NT>
constexpr size_t sweep2d_smem() { return (size_t)kSweep2Stages * NT * 128 + 2 * kSweep2Stages * 8 + 1024; }

struct Sweep2DParams {
    DevProblem pb;
    double lam;
    double c0, c1;             // center, g folded: RD (c0 + c1 w) w; AD c0 w_c + c1 w_{c+1}
    double cs, cn;             // south / north neighbour coefficients (g folded)
    double cyc;                // 1 / (1 - lam^nx): the cyclic closure
    double pw[16];             // lam^(e+1)
    double zf[16];             // forward-carry response of a chunk's backward pass
    double mp[10];             // M^(2^i), M = lam^16
    double* ring;
    long long cap, Vs;
    int P, GW, gpr, gdata;     // padded row pitch / ghost width / tensor-map groups
    int nx, ny;
    long long per;
    unsigned long long* err;
};

template <int KIND, int NT>
__global__ void __launch_bounds__(NT, 512 / NT)
    k_sweep2d_febe(const __grid_constant__ Sweep2DParams sp, const __grid_constant__ TmapSet tm, long long off,
                   long long target)
{
    static_assert(KIND == ADV_DIFF_2D || KIND == RD_2D, "2-D kinds");
    constexpr int K = 16, NW = NT / 32, NS = kSweep2Stages;
    using L = ChunkSmem<NT, 1, NS, 16>;
    constexpr int NBOX = NT / L::BR;
    extern __shared__ __align__(1024) char smraw[];
    char* stage = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + (size_t)NS * L::STAGE);
    uint64_t* empty = full + NS;
    __shared__ double sx[2 * NW];
    __shared__ unsigned s_cnt[NS];   // warps done with each stage (refill when all are)
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, cta = blockIdx.x;
    const int ny = sp.ny;
    const int r0 = (int)((long long)cta * ny / G), r1 = (int)((long long)(cta + 1) * ny / G);
    const int nl = r1 - r0 + 2;                     // rows loaded: r0-1 .. r1
    const long long src = (off + target - 1) % sp.cap, dst = (off + target) % sp.cap;
    RIDC_CHECK(src != dst && r1 > r0 && sp.nx == 16 * NT && (long long)sp.ny * sp.P <= sp.Vs);
    double* out0 = sp.ring + dst * sp.Vs + sp.GW + tid * K;   // + row * P
    const double lam = sp.lam;

    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NW);
            s_cnt[i] = 0u;
        }
        mbar_fence_init();
    }
    // carry powers: M^lane, M^(31-lane), (M^32)^warp, (M^32)^(NW-1-warp)
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
    __syncthreads();
    auto issue = [&](int k) {   // one lane: loaded row k (grid row r0 - 1 + k) into stage k % NS
        const int s = k % NS;
        int q = r0 - 1 + k;
        q = q < 0 ? q + ny : (q >= ny ? q - ny : q);
        mbar_arrive_expect_tx(&full[s], (uint32_t)(NBOX * L::BR * 128));
        for (int b = 0; b < NBOX; ++b)
            tma_load_3d(stage + (size_t)s * L::STAGE + b * L::BR * 128, &tm.map[0], 0,
                        q * sp.gpr + sp.gdata + b * L::BR, (int)src, &full[s]);
    };
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (tid == 0)
        for (int k = 0; k < NS && k < nl; ++k) issue(k);

    // the cyclic x-line solve of v (g folded), fast_solve<NT, 16, true> without the g multiply
    auto solve = [&](double (&v)[K]) {
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

    bool bad = false;
    // one loaded row k: complete rhs(q-1) in A and solve + store it, then
    // B += center(w_q), A = north contribution of q to rhs(q+1)
    auto row = [&](int k, double (&A)[K], double (&B)[K]) {
        const int s = k % NS;
        mbar_wait(&full[s], (uint32_t)((k / NS) & 1));
        const char* st = stage + (size_t)s * L::STAGE;
#pragma unroll
        for (int i = 0; i < K / 2; ++i) {
            const double2 w = lds128(swz(st, tid, i));
            A[2 * i] = fma(sp.cs, w.x, A[2 * i]);
            A[2 * i + 1] = fma(sp.cs, w.y, A[2 * i + 1]);
        }
        if (k >= 2) {   // rhs(q - 1) complete: row r0 - 2 + k of my block
            solve(A);
            bad |= !chunk_finite(A);
            double* o = out0 + (size_t)(r0 - 2 + k) * sp.P;
#pragma unroll
            for (int e = 0; e < K; e += 4) stg256(o + e, A[e], A[e + 1], A[e + 2], A[e + 3]);
        }
        if (k + 1 < nl) {
            if (KIND == RD_2D) {
#pragma unroll
                for (int i = 0; i < K / 2; ++i) {
                    const double2 w = lds128(swz(st, tid, i));
                    B[2 * i] = fma(fma(sp.c1, w.x, sp.c0), w.x, B[2 * i]);
                    B[2 * i + 1] = fma(fma(sp.c1, w.y, sp.c0), w.y, B[2 * i + 1]);
                    A[2 * i] = sp.cn * w.x;
                    A[2 * i + 1] = sp.cn * w.y;
                }
            } else {   // upwind x-advection: point c takes c0 w_c + c1 w_{c+1} (periodic in x)
                double2 w = lds128(swz(st, tid, 0));
#pragma unroll
                for (int i = 0; i < K / 2; ++i) {
                    const double nxt = i + 1 < K / 2 ? 0.0 : lds128(swz(st, tid + 1 < NT ? tid + 1 : 0, 0)).x;
                    const double2 wn = i + 1 < K / 2 ? lds128(swz(st, tid, i + 1)) : make_double2(nxt, 0.0);
                    B[2 * i] = fma(sp.c1, w.y, fma(sp.c0, w.x, B[2 * i]));
                    B[2 * i + 1] = fma(sp.c1, wn.x, fma(sp.c0, w.y, B[2 * i + 1]));
                    A[2 * i] = sp.cn * w.x;
                    A[2 * i + 1] = sp.cn * w.y;
                    w = wn;
                }
            }
        }
        // the stage goes back to the TMA once every warp consumed it: the LAST
        // warp to finish issues the refill (a shared counter), so no warp ever
        // blocks waiting for the slowest one (thread 0 used to, holding warp 0)
        __syncwarp();
        if (lane == 0) {
            __threadfence_block();   // my warp's reads of the stage before the count
            if (atomicAdd(&s_cnt[s], 1u) == (unsigned)(NW - 1)) {
                s_cnt[s] = 0u;
                __threadfence_block();
                if (k + NS < nl) issue(k + NS);
            }
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
    if (bad) atomicMin(sp.err, err_code((target - 1) % sp.per + 1, 0));
}

}  // namespace ridc
