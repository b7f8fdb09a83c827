// ridc_chunk.cuh -- chunk-layout level step: swizzled tensor-map TMA staging,
// register-resident stencils / recurrences / stores (sm_100a, fp64).
//
// Memory: every ring slot holds ny padded rows; row r, data column c lives
// at  r*P + GW + c  (P, GW multiples of 16).  Columns [-GW, 0) and
// [nx, nx+GW) are ghosts: periodic copies maintained by the writer of the
// source columns (zeros for the Dirichlet kind), so no item ever needs a
// wrapped copy.  A slot is a 3-D tensor  {16 doubles, groups, slots}: one
// group = one 128-byte row of the tensor map.
//
// An item (one level-step of one segment / whole line) maps thread t to the
// 16 consecutive points of group g0+t.  The producer (thread 0) stages each
// node's groups with cp.async.bulk.tensor (SWIZZLE_128B); a thread reads its
// chunk as 8 conflict-free 128-bit shared loads.  The x-stencils need only
// the two edge values of the neighbouring chunks (one shared exchange), the
// two recurrences run in registers with block scans for the carries, and the
// new state is stored straight from registers (16-byte stores), plus the
// ghost copies and, in the multi-GPU pipeline, the consumer's inbox.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ridc_device.cuh"
#include "ridc_tma.cuh"

namespace ridc {

constexpr int kChunk = 16;   // points per 128-byte group (and per thread in the 1-D configs)

// Per-segment item geometry (host table).
struct ChunkGeo {
    int g0;       // first staged group, relative to the row's data start (may be < 0: ghosts)
    int ng;       // groups staged = threads owning a chunk
    int c0, tlen; // output data columns [c0, c0 + tlen)
    int s_end;    // scanned positions [0, s_end) relative to column 16*g0
    int mode;     // 0: truncated segment, constant coefficients (fast_solve)
                  // 1: exact cyclic whole line; 2: exact Dirichlet start/end (tables)
};

struct TmapSet {
    CUtensorMap map[kMaxLevels];   // one per level ring: {16, groups/slot, slots}
};

// Layout of the staged rows of one node in a stage.  NT threads of KC points
// each cover NG = NT*KC/16 groups (KC = 16: one group per thread; KC = 8: two
// threads per group, for 16-warp CTAs on 4096-point lines).
template <int NT, int ROWS, int NSTAGE, int KC = kChunk>
struct ChunkSmem {
    static constexpr int NG = NT * KC / kChunk;                  // groups per item
    static constexpr int BR = NG < 256 ? NG : 256;              // groups per box
    static constexpr int ROWB = NG * 128;                        // bytes per staged row
    static constexpr int STAGE = ROWS * ROWB;                    // bytes per stage
    static constexpr size_t OFF_EDGE = (size_t)NSTAGE * STAGE;   // 4*NT doubles: chunk edges
    static constexpr size_t OFF_BAR = OFF_EDGE + 4 * NT * sizeof(double);
    static constexpr size_t BYTES = OFF_BAR + 2 * NSTAGE * sizeof(uint64_t);
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

// Bulk tensor store of a staged box (the TMA's 128-byte swizzle, as loaded)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}

__device__ __forceinline__ double2 lds128(const char* p)
{
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
    return v;
}

__device__ __forceinline__ void sts128(char* p, double a, double b)
{
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(smem_u32(p)), "d"(a), "d"(b) : "memory");
}

// element pair i (points 2i, 2i+1) of staged group g under SWIZZLE_128B
__device__ __forceinline__ const char* swz(const char* rowbase, int g, int i)
{
    return rowbase + g * 128 + ((i ^ (g & 7)) << 4);
}

// Issue the tensor copies of node a of an item: ROWS rows (2-D: r, r-1, r+1)
// x ceil(ng / BR) boxes of BR groups.
template <int NT, int ROWS, int NSTAGE, int KC>
__device__ __forceinline__ void issue_chunk_node(const TmapSet& tm, int lev, long long slot, int row,
                                                 int ny, int gpr, int gdata, const ChunkGeo& cg,
                                                 char* st, uint64_t* full)
{
    using L = ChunkSmem<NT, ROWS, NSTAGE, KC>;
    const int nbox = (cg.ng + L::BR - 1) / L::BR;
    mbar_arrive_expect_tx(full, (uint32_t)(ROWS * nbox * L::BR * 128));
    const int rr[3] = {row, row == 0 ? ny - 1 : row - 1, row == ny - 1 ? 0 : row + 1};
#pragma unroll
    for (int r = 0; r < ROWS; ++r)
        for (int b = 0; b < nbox; ++b)
            tma_load_3d(st + r * L::ROWB + b * L::BR * 128, &tm.map[lev], 0,
                        rr[r] * gpr + gdata + cg.g0 + b * L::BR, (int)slot, full);
}

}  // namespace ridc

namespace ridc {

// Phases 2-4 of a chunk item (x-stencils, then the two recurrences) on the
// pointwise accumulators of thread t's chunk; rhs receives the new state.
// Shared by the tick kernel (TMA-staged nodes) and the resident FEBE kernel
// (register-held state), so both produce bitwise the same states.
template <int KIND, int NT, int MODE, int K = kChunk>
__device__ __forceinline__ void chunk_rhs_solve(const DevProblem& pb, const DevSolve& sv, const ChunkGeo& cg,
                                                bool need_ws, bool need_wx, bool mine,
                                                const double (&P)[K], const double (&WS)[K],
                                                const double (&WX)[K], double (&rhs)[K],
                                                double* edge, Aff* swarp, int item_no, FastLane fl)
{
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr bool has_wx = KIND == ADV_DIFF_1D || KIND == BURGERS_1D || KIND == ADV_DIFF_2D;
    const int tid = threadIdx.x;
    // ---- phase 2: x-stencils; the neighbour chunks' edge values via shared memory
    const int col0 = cg.g0 * kChunk + tid * K;      // data column of my first point
    int nlast = K - 1;                              // my last valid point (whole lines: partial chunk)
    if (MODE == 1 || MODE == 2) nlast = min(K, cg.s_end - tid * K) - 1;
    need_wx = need_wx && has_wx;
    double wsl = 0.0, wsr = 0.0, wxl = 0.0, wxr = 0.0;   // left / right neighbour values
    if (need_ws || need_wx) {
        double lastws = 0.0, lastwx = 0.0;
#pragma unroll
        for (int e = 0; e < K; ++e)
            if (e == nlast) { lastws = WS[e]; lastwx = WX[e]; }
        edge[tid] = WS[0];
        edge[NT + tid] = lastws;
        edge[2 * NT + tid] = WX[0];
        edge[3 * NT + tid] = lastwx;
        csync<NT>();
        // threads holding data: whole staged groups (truncated segments), or the
        // line's positions (whole lines may end inside a group)
        const int nthr = MODE == 0 ? cg.ng * (kChunk / K) : (cg.s_end + K - 1) / K;
        const bool first = tid == 0, last = tid == nthr - 1;
        if (!first) { wsl = edge[NT + tid - 1]; wxl = edge[3 * NT + tid - 1]; }
        else if (MODE == 1) { wsl = edge[NT + nthr - 1]; wxl = edge[3 * NT + nthr - 1]; }   // cyclic
        if (!last) { wsr = edge[tid + 1]; wxr = edge[2 * NT + tid + 1]; }
        else if (MODE == 1) { wsr = edge[0]; wxr = edge[2 * NT]; }
        // MODE 2: zero Dirichlet ghosts; MODE 0: ends lie in the truncation halo
        csync<NT>();
    }
#pragma unroll
    for (int e = 0; e < K; ++e) {
        double r = P[e];
        if (need_ws) {
            const double l = e == 0 ? wsl : WS[e - 1];
            const double rr = e == K - 1 ? wsr : WS[e + 1];
            const double rn = (MODE != 0 && e == nlast) ? wsr : rr;
            r = fma(pb.cdx, (l - 2.0 * WS[e]) + rn, r);
        }
        if (need_wx) {
            const double l = e == 0 ? wxl : WX[e - 1];
            const double rr = e == K - 1 ? wxr : WX[e + 1];
            const double rn = (MODE != 0 && e == nlast) ? wxr : rr;
            if (KIND == BURGERS_1D) r = fma(-pb.bs, rn - l, r);
            else r = fma(pb.cax, rn - WX[e], r);
        }
        // threads past the staged groups feed zeros into the scans (their
        // accumulators are zero already unless a stencil pulled in a neighbour)
        rhs[e] = (need_ws || need_wx) ? (mine ? r : 0.0) : r;
    }
    RIDC_STAMP(sv, item_no, 3);

    // ---- phases 3-4: the two recurrences
    if (MODE == 0) {
        RIDC_STAMP(sv, item_no, 4);
        fast_solve<NT, K>(sv, rhs, reinterpret_cast<double*>(swarp), fl);
        RIDC_STAMP(sv, item_no, 7);
    } else if (MODE == 1 && periodic && (NT & (NT - 1)) == 0 && cg.s_end == NT * K) {
        // whole periodic line filling every chunk: constant-multiplier scans + cyclic closure
        fast_solve<NT, K, true>(sv, rhs, reinterpret_cast<double*>(swarp), fl);
    } else {
        const int nm = max(0, min(K, cg.s_end - tid * K));
        const bool cyclic = MODE == 1 && periodic;
        const double m = sv.lam, g = sv.g;
        double y = 0.0, A = 1.0;
#pragma unroll
        for (int e = 0; e < K; ++e)
            if (e < nm) {
                double mm = m, gg = g;
                if (sv.ntab > 0) coef(sv, col0 + e, mm, gg);
                y = fma(mm, y, gg * rhs[e]);
                A *= mm;
                rhs[e] = y;
            }
        Aff tot;
        Aff pre = block_scan<NT>(Aff{A, y}, false, swarp, tot);
        double cin = fma(pre.A, cyclic ? tot.B / (1.0 - tot.A) : 0.0, pre.B);
        double Pm = 1.0;
#pragma unroll
        for (int e = 0; e < K; ++e)
            if (e < nm) {
                double mm = m, gg = g;
                if (sv.ntab > 0) coef(sv, col0 + e, mm, gg);
                Pm *= mm;
                rhs[e] = fma(Pm, cin, rhs[e]);
            }
        double x = 0.0;
        A = 1.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e)
            if (e < nm) {
                double mm = m, gg = g;
                if (sv.ntab > 0) coef(sv, col0 + e, mm, gg);
                x = fma(mm, x, rhs[e]);
                A *= mm;
                rhs[e] = x;
            }
        pre = block_scan<NT>(Aff{A, x}, true, swarp, tot);
        cin = fma(pre.A, cyclic ? tot.B / (1.0 - tot.A) : 0.0, pre.B);
        Pm = 1.0;
#pragma unroll
        for (int e = K - 1; e >= 0; --e)
            if (e < nm) {
                double mm = m, gg = g;
                if (sv.ntab > 0) coef(sv, col0 + e, mm, gg);
                Pm *= mm;
                rhs[e] = fma(Pm, cin, rhs[e]);
            }
    }
}

struct ChunkLayout {
    int P;       // row pitch (doubles, multiple of 16)
    int GW;      // ghost columns per side (multiple of 16)
    int gpr;     // groups per row = P / 16
    int gdata;   // group of data column 0 within a row = GW / 16
};

// One chunk-layout item.  MODE: 0 truncated (fast_solve), 1 cyclic whole
// line, 2 exact Dirichlet start/end with coefficient tables.
template <int KIND, int NT, int ROWS, int NSTAGE, int MODE, int KC, class Refill>
__device__ __forceinline__ void chunk_item(const DevProblem& pb, const DevSolve& sv, const ChunkLayout& lay,
                                           const TmapSet& tm, const StepItem& it, const ChunkGeo& cg,
                                           int row, char* stage, double* edge, uint64_t* full,
                                           uint64_t* empty, long long& n, Refill&& refill, Aff* swarp,
                                           unsigned long long* err, int item_no, FastLane fl)
{
    using L = ChunkSmem<NT, ROWS, NSTAGE, KC>;
    constexpr int K = KC;                     // points per thread
    constexpr int HP = kChunk / KC;           // threads per group
    constexpr bool periodic = KIND != BURGERS_1D;
    constexpr bool two_d = ROWS == 3;
    const int tid = threadIdx.x, lane = tid & 31;
    RIDC_CHECK(row >= 0 && row < pb.ny && cg.c0 >= 0 && cg.c0 + cg.tlen <= pb.nx && cg.ng <= NT * KC / kChunk &&
               it.nnodes >= 1 && it.nnodes <= kMaxNodes);
    const int gq = tid / HP;                  // my group
    const int ip0 = (tid % HP) * (K / 2);     // my first element pair within it
    const bool mine = gq < cg.ng;             // owns (part of) a staged group

    double P[K], WS[K], WX[K];
#pragma unroll
    for (int e = 0; e < K; ++e) { P[e] = 0.0; WS[e] = 0.0; WX[e] = 0.0; }

    RIDC_STAMP(sv, item_no, 0);
    // ---- phase 1: stream the nodes (thread t reads its group as 8 x 128-bit)
    for (int a = 0; a < it.nnodes; ++a, ++n) {
        const int s = (int)(n % NSTAGE);
        const char* st = stage + (size_t)s * L::STAGE;
        mbar_wait(&full[s], (uint32_t)((n / NSTAGE) & 1));
        if (a == 0) RIDC_STAMP(sv, item_no, 1);
        const NodeCoef nc = node_coef<KIND>(pb, it.ca[a], it.cs[a], it.cn[a]);
        if (mine) {
#pragma unroll
            for (int i = 0; i < K / 2; ++i) {
                const double2 v = lds128(swz(st, gq, ip0 + i));
                double2 vn = make_double2(0.0, 0.0), vs = make_double2(0.0, 0.0);
                if (two_d) {
                    vn = lds128(swz(st + L::ROWB, gq, ip0 + i));
                    vs = lds128(swz(st + 2 * L::ROWB, gq, ip0 + i));
                }
                accumulate_point<KIND>(nc, v.x, vn.x, vs.x, P[2 * i], WS[2 * i], WX[2 * i]);
                accumulate_point<KIND>(nc, v.y, vn.y, vs.y, P[2 * i + 1], WS[2 * i + 1], WX[2 * i + 1]);
            }
        }
        if (a + 1 < it.nnodes) {   // the last node's stage is released after the store (scratch)
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
            if (tid == 0) refill(n, s);
        }
    }
    const long long n_last = n - 1;
    const int s_last = (int)(n_last % NSTAGE);
    char* sbufc = stage + (size_t)s_last * L::STAGE;   // store transpose scratch (NT x 128 B)
    RIDC_STAMP(sv, item_no, 2);

    bool need_ws = false, need_wx = false;
    for (int a = 0; a < it.nnodes; ++a) {
        need_ws |= it.cs[a] != 0.0;
        need_wx |= it.cn[a] != 0.0;
    }
    double rhs[K];
    chunk_rhs_solve<KIND, NT, MODE, K>(pb, sv, cg, need_ws, need_wx, mine, P, WS, WX, rhs, edge, swarp, item_no,
                                       fl);
    RIDC_STAMP(sv, item_no, 8);

    // ---- phase 5: store.  Chunks go to shared memory swizzled (conflict-free),
    // come back as consecutive 16-byte pieces (conflict-free) and leave as
    // coalesced 512-byte warp stores (+ periodic ghosts, + the pipeline mirror).
    if (mine)
#pragma unroll
        for (int i = 0; i < K / 2; ++i) sts128(const_cast<char*>(swz(sbufc, gq, ip0 + i)), rhs[2 * i], rhs[2 * i + 1]);
    // order these generic shared writes before the TMA that will refill this stage
    // (and before the bulk tensor store below)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    csync<NT>();
    // Whole lines of a multiple of 16 points (no mirror): the row leaves as bulk
    // tensor stores of the swizzled scratch (one instruction per box, no per-thread
    // store pass); periodic ghosts and the finite check come from registers.
    const bool tma_out = (MODE == 1 || MODE == 2) && it.omap1 > 0 && it.out2 == nullptr && cg.g0 == 0 &&
                         (pb.nx & 15) == 0 && cg.ng % L::BR == 0;
    if (tma_out) {
        if (tid == 0) {
            for (int b = 0; b < cg.ng / L::BR; ++b)
                tma_store_3d(&tm.map[it.omap1 - 1], sbufc + (size_t)b * L::BR * 128, 0,
                             row * lay.gpr + lay.gdata + b * L::BR, (int)it.oslot);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        double chk = 0.0;
        if (mine) {
            const int c0 = gq * kChunk + ip0 * 2;   // data column of my first point
            double* o1 = it.out + (size_t)row * lay.P + lay.GW;
#pragma unroll
            for (int e = 0; e < K; ++e) chk = fma(rhs[e], 0.0, chk);
            if (periodic) {
                if (c0 < lay.GW)
#pragma unroll
                    for (int e = 0; e < K; ++e) o1[c0 + e + pb.nx] = rhs[e];
                if (c0 + K > pb.nx - lay.GW)
#pragma unroll
                    for (int e = 0; e < K; ++e) o1[c0 + e - pb.nx] = rhs[e];
            }
        }
        if (chk != chk) atomicMin(err, err_code(it.target, it.level));
    } else {
        double chk = 0.0;
        const size_t rofs = (size_t)row * lay.P + lay.GW;   // data column 0 of my row
        double* o1 = it.out + rofs;
        double* o2 = it.out2 ? it.out2 + rofs : nullptr;
        const bool mirror = o2 != nullptr;                  // item-uniform
        const int lo = cg.c0, hi = cg.c0 + cg.tlen;
        const int nx = pb.nx, GW = lay.GW;
        // groups wholly inside the tile: [glo, ghi) relative to g0 (item-uniform)
        const int glo = (lo - cg.g0 * kChunk + kChunk - 1) / kChunk, ghi = (hi - cg.g0 * kChunk) / kChunk;
        // only items touching a line end write periodic ghost copies
        const bool ghosts = periodic && (lo < GW || hi > nx - GW);
#pragma unroll
        for (int k = 0; k < K / 2; ++k) {
            const int q = tid + k * NT;           // 16-byte piece: group q/8, pair q%8
            const int g = q >> 3, i = q & 7;
            if (g < cg.ng) {
                const double2 v = lds128(swz(sbufc, g, i));
                const int c = (cg.g0 + g) * kChunk + 2 * i;   // data column of v.x
                if ((unsigned)(g - glo) < (unsigned)(ghi - glo)) {
                    chk = fma(v.x, 0.0, fma(v.y, 0.0, chk));
                    *reinterpret_cast<double2*>(o1 + c) = v;
                    if (mirror) *reinterpret_cast<double2*>(o2 + c) = v;
                } else {
                    if (c >= lo && c < hi) { chk = fma(v.x, 0.0, chk); o1[c] = v.x; if (mirror) o2[c] = v.x; }
                    if (c + 1 >= lo && c + 1 < hi) { chk = fma(v.y, 0.0, chk); o1[c + 1] = v.y; if (mirror) o2[c + 1] = v.y; }
                }
                if (ghosts && (c < GW || c + 2 > nx - GW)) {
                    const double vv2[2] = {v.x, v.y};
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int cc = c + h;
                        if (cc >= lo && cc < hi) {
                            if (cc < GW) { o1[cc + nx] = vv2[h]; if (mirror) o2[cc + nx] = vv2[h]; }
                            if (cc >= nx - GW) { o1[cc - nx] = vv2[h]; if (mirror) o2[cc - nx] = vv2[h]; }
                        }
                    }
                }
            }
        }
        if (chk != chk) atomicMin(err, err_code(it.target, it.level));
    }
    // release the last node's stage (used as scratch) to the producer, once the
    // bulk store has read it
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s_last]);
    if (tid == 0) {
        if (tma_out) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        refill(n_last, s_last);
    }
    RIDC_STAMP(sv, item_no, 9);
}

}  // namespace ridc
