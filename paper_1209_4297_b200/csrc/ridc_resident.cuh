// ridc_resident.cuh -- register-resident FEBE march (levels == 1, 1-D lines).
//
// The predictor level alone (RIDC order 1: forward/backward Euler IMEX,
// engine.py:167-175 _predict_core) needs, per step, only its own state.
// When the line's segments fit one CTA each on the GPU (N <= ~148 x 7000
// points: configs C1 and C2), a single cooperative launch marches every
// step with each thread's 16-point chunk kept in registers:
//
//   step s:  [halo threads reload their chunk from the ring slot of step s-1,
//             after the two neighbour segments published it]
//            accumulate -> x-stencils -> two recurrences (chunk_rhs_solve,
//            the very code of the tick kernel: bitwise the same states)
//            -> publish the columns a neighbour's halo can reach (+ periodic
//               ghosts) into ring slot s % cap, then a release flag.
//
// Only the truncation-halo edges (~2 x 470 of ~7100 columns) round-trip
// through L2 per step, instead of the whole state; the full tile is written
// once, after the last step (or every step when the trajectory is recorded).
// Neighbour skew is at most one step, so the two-slot ring is race-free:
// a segment writes slot s % 2 only after both neighbours finished step s-1,
// i.e. after they read slot (s-2) % 2 for the last time.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"

namespace ridc {

struct ResidentParams {
    DevProblem pb;
    DevSolve sv;
    ChunkLayout lay;
    const ChunkGeo* cgeo;
    double* ring;            // level-0 ring, cap slots of Vs doubles (padded layout)
    long long cap, Vs;
    double dt;
    long long steps;         // restarts * per (FEBE restarts are plain continuation)
    long long per;           // steps per restart interval (error-step numbering)
    int edge_w;              // columns within edge_w of a tile end are published every step
    int full_every;          // 1: publish whole tiles every step (trajectory recording)
    uint4* mail;             // mailbox: 2 parities x Vs tagged lines (padded column index)
    unsigned tag0;           // run epoch: step s is tagged tag0 + s
    unsigned long long* err; // earliest non-finite (step, level), atomicMin
    unsigned* abort;         // watchdog: set when a neighbour wait times out
    long long spin_limit;    // watchdog budget per wait (clock64 cycles)
    long long* dbg;          // optional phase trace (RIDC_PHASE_TIMING): CTA 0, thread 0, steps 1..8
    int exp;                 // diagnostics only (RIDC_RES_EXP, wrong results): 1 skip the halo waits,
                             // 2 skip the edge pushes -- isolates the exchange cost from the compute
};

// slots: steps 1..4 -> rows 0..3, steps S-3..S -> rows 4..7; col 6: globaltimer (ns) at row start
#define RIDC_RSTAMP(rp, s, idx)                                                              \
    do {                                                                                     \
        if ((rp).dbg && threadIdx.x == 0 && blockIdx.x == 0) {                               \
            const long long _r = (s) <= 4 ? (s) - 1 : ((s) > (rp).steps - 4 ? (s) - (rp).steps + 7 : -1); \
            if (_r >= 0) {                                                                   \
                (rp).dbg[_r * 16 + (idx)] = clock64();                                       \
                if ((idx) == 0) {                                                            \
                    unsigned long long _g;                                                   \
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_g));                  \
                    (rp).dbg[_r * 16 + 6] = (long long)_g;                                   \
                }                                                                            \
            }                                                                                \
        }                                                                                    \
    } while (0)

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Low-latency mailbox line (the LL format of NCCL's low-latency protocol): one
// value per 16-byte line {lo32, tag, hi32, tag}, written by one vector store,
// so a reader that sees both tags equal to the step it wants has the value --
// no separate flag, no writer-side fence.
__device__ __forceinline__ void st_line(uint4* p, double v, unsigned tag)
{
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"((unsigned)b), "r"(tag),
                 "r"((unsigned)(b >> 32)), "r"(tag)
                 : "memory");
}

__device__ __forceinline__ uint4 ld_line(const uint4* p)
{
    uint4 v;
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

__device__ __forceinline__ double line_value(uint4 v)
{
    return __longlong_as_double((long long)(((unsigned long long)v.z << 32) | v.x));
}

__device__ __forceinline__ int floor_div_dev(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// 16 consecutive doubles from L2 (bypassing L1: other SMs wrote them)
__device__ __forceinline__ void load_chunk_cg(const double* src, double (&u)[kChunk])
{
    const double2* s2 = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int i = 0; i < kChunk / 2; ++i) {
        const double2 v = __ldcg(s2 + i);
        u[2 * i] = v.x;
        u[2 * i + 1] = v.y;
    }
}

template <int KIND, int NT, int MODE>
__device__ __forceinline__ void resident_step(const ResidentParams& rp, const ChunkGeo& cg, bool mine,
                                              double (&u)[kChunk], double* edge, Aff* swarp, FastLane fl)
{
    constexpr int K = kChunk;
    constexpr bool has_wx = KIND == ADV_DIFF_1D || KIND == BURGERS_1D;
    double P[K], WS[K], WX[K];
#pragma unroll
    for (int e = 0; e < K; ++e) {
        P[e] = 0.0;
        WS[e] = 0.0;
        WX[e] = 0.0;
    }
    // the predictor's single node: ca = 1, cs = 0, cn = dt (build_item, level 0)
    if (mine) {
        const NodeCoef nc = node_coef<KIND>(rp.pb, 1.0, 0.0, rp.dt);
#pragma unroll
        for (int e = 0; e < K; ++e) accumulate_point<KIND>(nc, u[e], 0.0, 0.0, P[e], WS[e], WX[e]);
    }
    chunk_rhs_solve<KIND, NT, MODE>(rp.pb, rp.sv, cg, false, has_wx && rp.dt != 0.0, mine, P, WS, WX, u, edge,
                                    swarp, 99, fl);
}

// Finite check of 16 values: four independent FMA chains (x * 0 is NaN iff x is not finite).
__device__ __forceinline__ bool chunk_finite(const double (&u)[kChunk])
{
    double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
    for (int e = 0; e < kChunk; e += 4) {
        c0 = fma(u[e], 0.0, c0);
        c1 = fma(u[e + 1], 0.0, c1);
        c2 = fma(u[e + 2], 0.0, c2);
        c3 = fma(u[e + 3], 0.0, c3);
    }
    const double c = (c0 + c1) + (c2 + c3);
    return c == c;
}

// MODE: the solve mode every segment shares (0 truncated, 1 cyclic whole
// line, 2 Dirichlet ends), or -1 to dispatch per segment.
//
// Neighbour protocol (segmented lines): no per-step CTA barrier, no fences.
// Threads holding tile columns a neighbour's halo reads (edge chunks, and
// their periodic ghost copies) write each new value as a tagged mailbox line
// of parity s & 1 right after step s.  A halo thread polls the last line of
// its chunk until the tag reads tag0 + s, then reads all 16 lines and re-polls
// any whose tags are not yet current (one line in flight while waiting keeps
// the polling traffic off the L2).  Interior warps never wait: they
// accumulate and run their local recurrences until the block scan's barrier.
// Parity buffers are race-free: a segment overwrites its step-s lines at step
// s+2 only after reading the neighbour's step s+1 lines, which the neighbour
// wrote after consuming (through its block scans) the step-s lines.
template <int KIND, int NT, int MODE>
__global__ void __launch_bounds__(NT, 1) k_resident_febe(const __grid_constant__ ResidentParams rp)
{
    static_assert(KIND == ADV_DIFF_1D || KIND == BURGERS_1D || KIND == RD_1D, "1-D kinds only");
    constexpr int K = kChunk;
    constexpr bool periodic = KIND != BURGERS_1D;
    __shared__ double edge[4 * NT];
    __shared__ double xpush[4][32 * 17];   // per edge warp: transpose buffer of the coalesced push
    __shared__ int s_pubw[NT / 32];
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    const int tid = threadIdx.x;
    const int seg = blockIdx.x, nseg = rp.sv.nseg;
    const ChunkGeo cg = rp.cgeo[seg];
    const bool mine = tid < cg.ng;
    const int col0 = (cg.g0 + tid) * K;   // data column of my first point
    const int lo = cg.c0, hi = cg.c0 + cg.tlen;
    const int nx = rp.pb.nx, GW = rp.lay.GW, W = rp.edge_w;
    // halo chunk: (partly) outside my tile -- pulled every step from the mailbox
    const bool halo = mine && nseg > 1 && (col0 < lo || col0 + K > hi);
    // edge chunk: tile columns a neighbour's halo (or a periodic ghost) reads
    const bool pub = mine && nseg > 1 && col0 + K > lo && col0 < hi && (col0 - lo < W || hi - (col0 + K) < W);
    const bool inside = mine && col0 >= lo && col0 + K <= hi;
    // edge warps (holding pushed columns) get a transpose slot for coalesced pushes
    const int lane = tid & 31, wid = tid >> 5;
    const unsigned pub_mask = __ballot_sync(0xffffffffu, pub);
    if (lane == 0) s_pubw[wid] = pub_mask != 0u;
    __syncthreads();
    int pslot = -1;
    if (pub_mask) {
        pslot = 0;
        for (int w = 0; w < wid; ++w) pslot += s_pubw[w];
        if (pslot >= 4) pslot = -1;   // more than four edge warps: scattered push for the rest
    }
    const int wcol0 = col0 - lane * K;   // first column of my warp's 32 chunks
    // the chunk line polled first: my last column outside the tile (Dirichlet
    // ghosts beyond the line are zero and never pushed)
    int probe = -1;
    if (halo)
        for (int e = 0; e < K; ++e) {
            const int c = col0 + e;
            if ((c < lo || c >= hi) && (periodic || (c >= 0 && c < nx))) probe = e;
        }

    double u[K];
#pragma unroll
    for (int e = 0; e < K; ++e) u[e] = 0.0;
    if (mine) load_chunk_cg(rp.ring + GW + col0, u);   // slot 0: the seeded initial state
    const FastLane fl = fast_lane<K>(rp.sv);
    bool dead = false;                                  // watchdog fired: stop waiting, drain

    for (long long s = 1; s <= rp.steps; ++s) {
        RIDC_RSTAMP(rp, s, 0);
        if (s > 1 && halo && !(rp.exp & 1)) {
            const unsigned want = rp.tag0 + (unsigned)(s - 1);
            const uint4* box = rp.mail + (size_t)((s - 1) & 1) * rp.Vs + GW + col0;
            const long long t0 = clock64();
            auto timed_out = [&] {
                if (!dead && (clock64() - t0 > rp.spin_limit || *(volatile unsigned*)rp.abort)) {
                    atomicExch(rp.abort, 1u);
                    dead = true;
                }
                return dead;
            };
            if (probe >= 0) {
                uint4 pv = ld_line(box + probe);
                while ((pv.y != want || pv.w != want) && !timed_out()) pv = ld_line(box + probe);
            }
            uint4 v[K];
#pragma unroll
            for (int e = 0; e < K; ++e) v[e] = ld_line(box + e);
#pragma unroll
            for (int e = 0; e < K; ++e) {
                const int c = col0 + e;
                if (!periodic && (c < 0 || c >= nx)) { u[e] = 0.0; continue; }   // Dirichlet ghost
                while ((v[e].y != want || v[e].w != want) && !timed_out()) v[e] = ld_line(box + e);
                u[e] = line_value(v[e]);
            }
        }
        RIDC_RSTAMP(rp, s, 2);
        if (MODE >= 0) {
            resident_step<KIND, NT, (MODE >= 0 ? MODE : 0)>(rp, cg, mine, u, edge, swarp, fl);
        } else {
            switch (cg.mode) {
            case 0: resident_step<KIND, NT, 0>(rp, cg, mine, u, edge, swarp, fl); break;
            case 1: resident_step<KIND, NT, 1>(rp, cg, mine, u, edge, swarp, fl); break;
            default: resident_step<KIND, NT, 2>(rp, cg, mine, u, edge, swarp, fl);
            }
        }
        RIDC_RSTAMP(rp, s, 3);
        // push the edge columns of step s (and their periodic ghost copies)
        if (rp.exp & 2) {
        } else if (pslot >= 0) {
            // coalesced push: transpose through shared memory, then 32 consecutive lines per store
            double* xb = xpush[pslot];
            if (pub) {
#pragma unroll
                for (int e = 0; e < K; ++e) xb[lane * 17 + e] = u[e];
            }
            __syncwarp();
            const unsigned tag = rp.tag0 + (unsigned)s;
            uint4* box = rp.mail + (size_t)(s & 1) * rp.Vs + GW;
#pragma unroll
            for (int i = 0; i < K; ++i) {
                const int idx = i * 32 + lane, c = wcol0 + idx;
                if (((pub_mask >> (idx >> 4)) & 1u) && c >= lo && c < hi) {
                    const double val = xb[(idx >> 4) * 17 + (idx & 15)];
                    st_line(box + c, val, tag);
                    if (periodic && c < GW) st_line(box + c + nx, val, tag);
                    if (periodic && c >= nx - GW) st_line(box + c - nx, val, tag);
                }
            }
            __syncwarp();
        } else if (pub) {
            const unsigned tag = rp.tag0 + (unsigned)s;
            uint4* box = rp.mail + (size_t)(s & 1) * rp.Vs + GW;
#pragma unroll
            for (int e = 0; e < K; ++e) {
                const int c = col0 + e;
                if (c >= lo && c < hi) {
                    st_line(box + c, u[e], tag);
                    if (periodic && c < GW) st_line(box + c + nx, u[e], tag);
                    if (periodic && c >= nx - GW) st_line(box + c - nx, u[e], tag);
                }
            }
        }
        // finite check over my tile columns; the whole tile to the ring at the end
        const bool full = s == rp.steps || rp.full_every;
        double* out = full ? rp.ring + (s % rp.cap) * rp.Vs + GW : nullptr;   // trajectory: cap = steps + 1
        bool bad = false;
        if (inside) {
            bad = !chunk_finite(u);
            if (full) {
#pragma unroll
                for (int e = 0; e < K; e += 2)
                    *reinterpret_cast<double2*>(out + col0 + e) = make_double2(u[e], u[e + 1]);
            }
        } else if (mine) {
            double chk = 0.0;
#pragma unroll
            for (int e = 0; e < K; ++e) {
                const int c = col0 + e;
                if (c >= lo && c < hi) {
                    chk = fma(u[e], 0.0, chk);
                    if (full) out[c] = u[e];
                }
            }
            bad = chk != chk;
        }
        if (bad) atomicMin(rp.err, err_code((s - 1) % rp.per + 1, 0));
        RIDC_RSTAMP(rp, s, 4);
        RIDC_RSTAMP(rp, s, 5);
    }
}

}  // namespace ridc
