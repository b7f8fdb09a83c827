// ridc_levels.cuh -- resident level march: every RIDC level of a 1-D line as
// one persistent CTA group, the lagged pipeline driven by device-side flags.
//
// The reference runs level j as a thread that claims rows of level j-1's
// LevelBuffer once the watermark passes them, publishes its own rows and
// releases the producer's (engine.py:284-459).  Here level j is a group of
// co-resident CTAs, one per segment of the line (the tick kernel's tiling,
// so the states are bitwise those of the tick kernel), that marches all
// steps of an interval in ONE launch with its segment's state in registers:
//
//   step t:  [halo chunks: the neighbour segments' step t-1 edges, tagged
//             mailbox lines as in the resident FEBE march]
//            node 0 (own state, registers) + window nodes: thread 0 waits
//            until the producer published step `newest` for every producer
//            segment my staged columns read (per-segment flags, acquire),
//            then streams each window state of level j-1 with TMA into
//            shared-memory stages (the tick kernel's swizzled layout)
//            -> x-stencils, the two recurrences (chunk_rhs_solve)
//            -> push my edge columns to the mailbox (neighbour halos)
//            -> release the producer's slots I no longer need (per segment)
//            -> if not the top level: wait until the consumer released the
//               slot I overwrite, store my tile (+ periodic ghosts) into the
//               consumer's inbox with coalesced stores; its flag (release at
//               system scope) is raised after the next step's solve, once
//               the stores drained (the last step's at once).
//
// The lanes table says where each level's rings and flags live.  One launch
// may hold every level of a line (one GPU: the CTA groups of all levels are
// co-resident, cooperative launch) or just one (the one-level-per-GPU
// pipeline: inbox, flags and the consumer's inbox are IPC-mapped peer memory
// and the stores cross NVLink).  Flag values carry the run epoch in the high
// 32 bits, so nothing is cleared between runs.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_chunk.cuh"
#include "ridc_device.cuh"
#include "ridc_resident.cuh"
#include "ridc_tma.cuh"

namespace ridc {

constexpr int kResDeps = 4;   // producer segments one consumer segment reads (and vice versa)

// Dynamic shared memory of the level kernel: NSTAGE TMA stages of the window
// nodes (the tick kernel's swizzled 1-row stage), the scratch holding my new
// state for the coalesced stores, the stencil edges, the stage mbarriers.
template <int NT, int NSTAGE>
struct LevSmem {
    static constexpr int STAGE = NT * 128;   // ChunkSmem<NT, 1, NSTAGE, 16>::STAGE
    static constexpr size_t OFF_SCR = (size_t)NSTAGE * STAGE;
    static constexpr size_t OFF_EDGE = OFF_SCR + STAGE;
    static constexpr size_t OFF_BAR = OFF_EDGE + 4 * NT * sizeof(double);
    static constexpr size_t BYTES = OFF_BAR + 2 * NSTAGE * sizeof(uint64_t);
};

struct LevelLane {
    int level;                     // j
    int in_map;                    // tensor map (TmapSet index) of my inbox ring, level > 0
    const double* own0;            // padded slot holding the interval's state0
    double* fin;                   // padded slot receiving my final tile
    long long in_off, in_cap;      // producer step t lives in inbox slot (in_off + t) % in_cap
    unsigned long long* in_pub;    // [nseg] producer's published step per segment (my memory)
    unsigned long long* in_rel;    // [nseg] my released-below per segment (producer's memory)
    double* out;                   // consumer's inbox ring, or null (top level)
    long long out_off, out_cap;
    unsigned long long* out_pub;   // [nseg] the consumer's in_pub
    unsigned long long* out_rel;   // [nseg] the consumer's released-below (my memory)
    uint4* mail;                   // own-level halo mailbox: 2 parities x Vs tagged lines
};

struct LevelsParams {
    DevProblem pb;
    DevSolve sv;
    ChunkLayout lay;
    const ChunkGeo* cgeo;
    const LevelLane* lanes;        // blockIdx.x / nseg -> lane
    const int* deps;               // [nseg][kResDeps] producer segments my staged columns read (-1: none)
    const int* readers;            // [nseg][kResDeps] consumer segments reading my tile (-1: none)
    const double* weights;
    int steady_off[kMaxLevels], startup_off[kMaxLevels];
    double dt;
    long long per;                 // steps of this interval
    long long Vs;
    unsigned long long epoch;      // flag value of step t: epoch << 32 | t
    int pub_every;                 // publish the consumer's flag every this many steps (>= 1)
    unsigned tag0;                 // mailbox tag of step t: tag0 + t
    int edge_w;                    // columns within edge_w of a tile end are pushed every step
    unsigned long long* err;
    unsigned* abort;
    long long spin_limit;
};

// Flag accesses at system scope (SYS: the levels sit on different GPUs and
// the flags / data cross NVLink) or GPU scope (every level on this device).
template <bool SYS>
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p)
{
    unsigned long long v;
    if (SYS) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Publication: every store of the CTA ordered before this thread (a CTA
// barrier) becomes visible before the flag (release fence + relaxed store).
template <bool SYS>
__device__ __forceinline__ void publish_u64(unsigned long long* p, unsigned long long v)
{
    if (SYS) asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("fence.acq_rel.gpu;\n\tst.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Release counter: the window reads it covers are TMA loads whose data is
// already in shared memory (their mbarriers completed), so no fence orders
// them -- a relaxed store suffices.
template <bool SYS>
__device__ __forceinline__ void store_relaxed_u64(unsigned long long* p, unsigned long long v)
{
    if (SYS) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spin (one thread) until flags[s] >= want for every listed segment.  `seen`
// caches the smallest value observed at the last poll: a wait it already
// covers costs nothing (the acquire that observed it ordered that data).
template <bool SYS>
__device__ __forceinline__ bool wait_flags(const unsigned long long* flags, const int* segs,
                                           unsigned long long want, unsigned long long& seen,
                                           const LevelsParams& rp, bool& dead)
{
    if (seen >= want) return true;
    const long long t0 = clock64();
    unsigned long long lo = ~0ull;
    for (int k = 0; k < kResDeps; ++k) {
        const int s = segs[k];
        if (s < 0) break;
        unsigned long long v;
        while (!dead && (v = ld_acquire_u64<SYS>(flags + s)) < want) {
            if (clock64() - t0 > rp.spin_limit || *(volatile unsigned*)rp.abort) {
                atomicExch(rp.abort, 1u);
                dead = true;
            }
        }
        if (!dead) lo = v < lo ? v : lo;
    }
    if (!dead) seen = lo;
    return !dead;
}

// MINB = 2 (4096-point items, NT = 256): two CTAs per SM at the 128-register
// cap, so twice the levels x segments fit the co-residency limit (2^16 points
// at p = 8); chosen only when one CTA per SM does not fit (it spills)
template <int KIND, int NT, int MODE, int NSTAGE, bool SYS, int MINB = 1>
__global__ void __launch_bounds__(NT, MINB)
    k_resident_levels(const __grid_constant__ LevelsParams rp, const __grid_constant__ TmapSet tm)
{
    static_assert(KIND == ADV_DIFF_1D || KIND == BURGERS_1D || KIND == RD_1D, "1-D kinds only");
    using L = LevSmem<NT, NSTAGE>;
    constexpr int K = kChunk;
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr bool has_wx = KIND == ADV_DIFF_1D || KIND == BURGERS_1D;
    extern __shared__ __align__(1024) char smraw[];
    char* stage = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
    char* scr = stage + L::OFF_SCR;   // my level's new state, swizzled like a stage
    double* edge = reinterpret_cast<double*>(stage + L::OFF_EDGE);
    uint64_t* full = reinterpret_cast<uint64_t*>(stage + L::OFF_BAR);
    uint64_t* empty = full + NSTAGE;
    __shared__ Aff swarp[2 * (NT / 32) + 1];
    __shared__ int s_dead;

    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int nseg = rp.sv.nseg;
    const int seg = blockIdx.x % nseg;
    // my lane's table in shared memory: read once, no per-step global reloads
    // (stores to the rings could alias a global table) and no registers held
    __shared__ LevelLane s_ln;
    if (tid == 0) s_ln = rp.lanes[blockIdx.x / nseg];
    __syncthreads();
    const LevelLane& ln = s_ln;
    const int j = ln.level;
    double* const out = ln.out;
    const ChunkGeo cg = rp.cgeo[seg];
    const bool mine = tid < cg.ng;
    const int col0 = (cg.g0 + tid) * K;
    const int lo = cg.c0, hi = cg.c0 + cg.tlen;
    const int nx = rp.pb.nx, GW = rp.lay.GW, W = rp.edge_w;
    const bool halo = mine && nseg > 1 && (col0 < lo || col0 + K > hi);
    const bool pub = mine && nseg > 1 && col0 + K > lo && col0 < hi && (col0 - lo < W || hi - (col0 + K) < W);
    const bool inside = mine && col0 >= lo && col0 + K <= hi;
    const unsigned pub_mask = __ballot_sync(0xffffffffu, pub);
    if (tid == 0) {
        s_dead = 0;
        for (int i = 0; i < NSTAGE; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int wcol0 = col0 - lane * K;
    int probe = -1;
    if (halo)
        for (int e = 0; e < K; ++e) {
            const int c = col0 + e;
            if ((c < lo || c >= hi) && (periodic || (c >= 0 && c < nx))) probe = e;
        }
    const int* deps = rp.deps + seg * kResDeps;
    const int* readers = rp.readers + seg * kResDeps;

    double u[K];
#pragma unroll
    for (int e = 0; e < K; ++e) u[e] = 0.0;
    if (mine) load_chunk_cg(ln.own0 + GW + col0, u);
    const FastLane fl = fast_lane<K>(rp.sv);
    bool dead = false;
    long long n = 0;   // TMA loads issued so far (load n lands in stage n % NSTAGE)
    const unsigned long long ep = rp.epoch << 32;
    // thread 0's protocol state (shared memory: keeps it out of every thread's registers)
    __shared__ unsigned long long seen_in, seen_rel;   // flag values already observed
    __shared__ long long published;                    // last step whose flag is raised
    if (tid == 0) { seen_in = 0; seen_rel = 0; published = 0; }

    // Coalesced stores of step ts (in the scratch) into the consumer's inbox
    // slot, + periodic ghost copies: issued at the start of the next step, so
    // they drain while the halo threads wait and the solve runs
    long long pend = 0;
    auto store_tile = [&](long long ts) {
        if (s_dead) return;
        // LevelBuffer.publish's capacity rule (engine.py:305-318): the consumer released the slot
        RIDC_CHECK(ts - ln.out_cap + 1 <= 0 || seen_rel >= (ep | (unsigned long long)(ts - ln.out_cap + 1)));
        double* o = out + ((ln.out_off + ts) % ln.out_cap) * rp.Vs + GW;
        const int glo = (lo - cg.g0 * kChunk + kChunk - 1) / kChunk, ghi = (hi - cg.g0 * kChunk) / kChunk;
        const bool ghosts = periodic && (lo < GW || hi > nx - GW);
#pragma unroll
        for (int k = 0; k < K / 2; ++k) {
            const int q = tid + k * NT;
            const int g = q >> 3, i = q & 7;
            if (g < cg.ng) {
                const double2 v = lds128(swz(scr, g, i));
                const int c = (cg.g0 + g) * kChunk + 2 * i;
                if ((unsigned)(g - glo) < (unsigned)(ghi - glo)) {
                    *reinterpret_cast<double2*>(o + c) = v;
                } else {
                    if (c >= lo && c < hi) o[c] = v.x;
                    if (c + 1 >= lo && c + 1 < hi) o[c + 1] = v.y;
                }
                if (ghosts && (c < GW || c + 2 > nx - GW)) {
                    const double vv2[2] = {v.x, v.y};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int cc = c + h;
                        if (cc >= lo && cc < hi) {
                            if (cc < GW) o[cc + nx] = vv2[h];
                            if (cc >= nx - GW) o[cc - nx] = vv2[h];
                        }
                    }
                }
            }
        }
    };

    // thread 0: window node a of step tt (build_item's order) as TMA load m into stage m % NSTAGE
    long long issued = 0;   // thread 0: loads issued so far (load numbers < issued)
    auto issue_node = [&](long long tt, int a, long long m) {
        if (m + 1 > issued) issued = m + 1;
        const int s = (int)(m % NSTAGE);
        if (m >= NSTAGE) mbar_wait(&empty[s], (uint32_t)(((m - NSTAGE) / NSTAGE) & 1));
        const long long ns = tt >= j ? tt - a : a;
        const long long slot = (ln.in_off + ns) % ln.in_cap;
        // the window reads only published producer steps (engine.py:363-371 _ready)
        RIDC_CHECK(ns == 0 || seen_in >= (ep | (unsigned long long)ns));
        issue_chunk_node<NT, 1, NSTAGE, kChunk>(tm, ln.in_map, slot, 0, 1, rp.lay.gpr, rp.lay.gdata, cg,
                                                stage + (size_t)s * L::STAGE, &full[s]);
    };
    unsigned pre_mask = 0;   // thread 0: first nodes of the next step already issued

    for (long long t = 1; t <= rp.per; ++t) {
        // ---- window of level j-1 (build_item, ridc_engine.cu): steady t >= j
        // nodes t, t-1, ..., t-j (i_new 0, i_old 1); startup nodes 0..j
        const bool steady = t >= j;
        const double* w = j == 0 ? nullptr
                          : steady ? rp.weights + rp.steady_off[j]
                                   : rp.weights + rp.startup_off[j] + (t - 1) * (j + 1);
        const int i_new = steady ? 0 : (int)t, i_old = steady ? 1 : (int)t - 1;
        if (j > 0 && tid == 0) {
            // the first NSTAGE nodes, unless prefetched during the previous step's solve
            if (wait_flags<SYS>(ln.in_pub, deps, ep | (unsigned long long)(steady ? t : j), seen_in, rp, dead)) {
                // the producer's generic (peer) stores, acquired above, before the async-proxy reads
                asm volatile("fence.proxy.async.global;" ::: "memory");
                for (int a = 0; a < NSTAGE && a <= j; ++a)
                    if (!(pre_mask & (1u << a))) issue_node(t, a, n + a);
            }
            pre_mask = 0;
            if (dead) s_dead = 1;
        }
        if (pend) store_tile(pend);   // step t-1 to the consumer
        // ---- own-state halo chunks: the neighbours' step t-1 edges
        if (t > 1 && halo) {
            const unsigned want = rp.tag0 + (unsigned)(t - 1);
            const uint4* box = ln.mail + (size_t)((t - 1) & 1) * rp.Vs + GW + col0;
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
                if (!periodic && (c < 0 || c >= nx)) { u[e] = 0.0; continue; }
                while ((v[e].y != want || v[e].w != want) && !timed_out()) v[e] = ld_line(box + e);
                u[e] = line_value(v[e]);
            }
        }
        // ---- node 0: my own state (ca 1, cs 0, cn dt), then the window nodes in order
        double P[K], WS[K], WX[K];
#pragma unroll
        for (int e = 0; e < K; ++e) { P[e] = 0.0; WS[e] = 0.0; WX[e] = 0.0; }
        bool need_ws = false, need_wx = rp.dt != 0.0;
        if (mine) {
            const NodeCoef nc = node_coef<KIND>(rp.pb, 1.0, 0.0, rp.dt);
#pragma unroll
            for (int e = 0; e < K; ++e) accumulate_point<KIND>(nc, u[e], 0.0, 0.0, P[e], WS[e], WX[e]);
        }
        if (j > 0) {
            __syncthreads();   // s_dead from thread 0's producer wait (CTA-uniform control flow)
            if (!s_dead) {
                for (int a = 0; a <= j; ++a, ++n) {
                    const int s = (int)(n % NSTAGE);
                    mbar_wait(&full[s], (uint32_t)((n / NSTAGE) & 1));
                    const double cs = w[a] - (a == i_new ? rp.dt : 0.0);
                    const double cn = w[a] - (a == i_old ? rp.dt : 0.0);
                    need_ws |= cs != 0.0;
                    need_wx |= cn != 0.0;
                    const NodeCoef nc = node_coef<KIND>(rp.pb, 0.0, cs, cn);
                    const char* st = stage + (size_t)s * L::STAGE;
                    if (mine) {
#pragma unroll
                        for (int i = 0; i < K / 2; ++i) {
                            const double2 v = lds128(swz(st, tid, i));
                            accumulate_point<KIND>(nc, v.x, 0.0, 0.0, P[2 * i], WS[2 * i], WX[2 * i]);
                            accumulate_point<KIND>(nc, v.y, 0.0, 0.0, P[2 * i + 1], WS[2 * i + 1], WX[2 * i + 1]);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty[s]);
                    if (tid == 0 && a + NSTAGE <= j) issue_node(t, a + NSTAGE, n + NSTAGE);
                }
                // prefetch: the next step's first nodes whose producer steps are
                // already published stream in while this step solves
                if (tid == 0 && t < rp.per && !dead) {
                    const long long t1 = t + 1;
                    for (int a = 0; a < NSTAGE && a <= j; ++a) {
                        const long long ns = t1 >= j ? t1 - a : a;
                        if (seen_in >= (ep | (unsigned long long)ns)) {   // acquired earlier: published
                            issue_node(t1, a, n + a);
                            pre_mask |= 1u << a;
                        }
                    }
                }
            }
        }
        need_wx = need_wx && has_wx;
        double rhs[K];
        if (MODE >= 0) {
            chunk_rhs_solve<KIND, NT, (MODE >= 0 ? MODE : 0), K>(rp.pb, rp.sv, cg, need_ws, need_wx, mine, P, WS,
                                                                 WX, rhs, edge, swarp, 99, fl);
        } else {   // mixed segments (Dirichlet ends, truncated middles): the tick kernel's per-segment mode
            switch (cg.mode) {
            case 0: chunk_rhs_solve<KIND, NT, 0, K>(rp.pb, rp.sv, cg, need_ws, need_wx, mine, P, WS, WX, rhs, edge,
                                                    swarp, 99, fl); break;
            case 1: chunk_rhs_solve<KIND, NT, 1, K>(rp.pb, rp.sv, cg, need_ws, need_wx, mine, P, WS, WX, rhs, edge,
                                                    swarp, 99, fl); break;
            default: chunk_rhs_solve<KIND, NT, 2, K>(rp.pb, rp.sv, cg, need_ws, need_wx, mine, P, WS, WX, rhs, edge,
                                                     swarp, 99, fl);
            }
        }
#pragma unroll
        for (int e = 0; e < K; ++e) u[e] = rhs[e];
        // deferred, batched publication: steps up to t-1 (their stores were
        // ordered before the solve's block barriers), every pub_every steps --
        // one release fence per batch instead of one per step
        if (out && t > 1 && tid == 0 && !s_dead && (t - 1) % rp.pub_every == 0) {
            publish_u64<SYS>(ln.out_pub + seg, ep | (unsigned long long)(t - 1));
            published = t - 1;
        }
        // ---- step t into the scratch (swizzled groups), then my edge columns
        // for the neighbour segments' halos straight from it (coalesced lines)
        if (mine)
#pragma unroll
            for (int i = 0; i < K / 2; ++i) sts128(const_cast<char*>(swz(scr, tid, i)), u[2 * i], u[2 * i + 1]);
        if (pub_mask) {
            __syncwarp();
            const unsigned tag = rp.tag0 + (unsigned)t;
            uint4* box = ln.mail + (size_t)(t & 1) * rp.Vs + GW;
#pragma unroll
            for (int i = 0; i < K; ++i) {
                const int idx = i * 32 + lane, c = wcol0 + idx;
                if (((pub_mask >> (idx >> 4)) & 1u) && c >= lo && c < hi) {
                    const int g = wid * 32 + (idx >> 4), e = idx & 15;
                    const double val = *reinterpret_cast<const double*>(swz(scr, g, e >> 1) + 8 * (e & 1));
                    st_line(box + c, val, tag);
                    if (periodic && c < GW) st_line(box + c + nx, val, tag);
                    if (periodic && c >= nx - GW) st_line(box + c - nx, val, tag);
                }
            }
        }
        // every window read of this step is done (the scans' barriers): release
        // the producer's slots below my next window (LevelBuffer.release_through)
        if (j > 0 && tid == 0 && !dead)
            store_relaxed_u64<SYS>(ln.in_rel + seg, ep | (unsigned long long)(t + 1 - j > 0 ? t + 1 - j : 0));
        if (out) {
            // the consumer's slot of step t must be free before its stores (next step)
            const long long need = t - ln.out_cap + 1;
            if (tid == 0 && need > 0 && !dead && seen_rel < (ep | (unsigned long long)need)) {
                // about to wait on the consumer: first publish what it may be waiting for
                if (published < t - 1 && !s_dead) {
                    publish_u64<SYS>(ln.out_pub + seg, ep | (unsigned long long)(t - 1));
                    published = t - 1;
                }
                if (!wait_flags<SYS>(ln.out_rel, readers, ep | (unsigned long long)need, seen_rel, rp, dead))
                    s_dead = 1;
            }
            __syncthreads();   // the whole scratch of step t, and the slot is free
            pend = t;
        }
        // ---- finite check of my tile columns; the final tile at the end
        const bool last = t == rp.per;
        bool bad = false;
        if (inside) {
            bad = !chunk_finite(u);
            if (last) {
#pragma unroll
                for (int e = 0; e < K; e += 2)
                    *reinterpret_cast<double2*>(ln.fin + GW + col0 + e) = make_double2(u[e], u[e + 1]);
            }
        } else if (mine) {
            double chk = 0.0;
#pragma unroll
            for (int e = 0; e < K; ++e) {
                const int c = col0 + e;
                if (c >= lo && c < hi) {
                    chk = fma(u[e], 0.0, chk);
                    if (last) ln.fin[GW + c] = u[e];
                }
            }
            bad = chk != chk;
        }
        if (bad) atomicMin(rp.err, err_code(t, j));
        // a timed-out wait (watchdog) leaves the remaining steps' waits
        // skipped: the CTA drains without blocking; the host reports it
    }
    if (out && pend) {   // the last step's tile, then its flag
        store_tile(pend);
        __syncthreads();
        if (tid == 0 && !s_dead) publish_u64<SYS>(ln.out_pub + seg, ep | (unsigned long long)pend);
    }
    // a watchdog exit can leave prefetched window loads in flight: the CTA must
    // not retire while the TMA still writes its shared memory
    if (tid == 0)
        for (long long m = n; m < issued; ++m) mbar_wait(&full[m % NSTAGE], (uint32_t)((m / NSTAGE) & 1));
}

}  // namespace ridc
