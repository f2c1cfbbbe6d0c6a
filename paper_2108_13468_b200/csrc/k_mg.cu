// k_mg.cu -- corner multigrid kernels of the two-exponential-layer preconditioner
// and the exact M_II sweep, sm_100a, fp64:
// downstream Gauss-Seidel smoothing, residual + FE-scaled restriction
// (P:1276-1280), and the outer stationary-iteration update with the FE-rescaled corner norm
// (reading R6).
//
// Downstream sweep (K3/K4 "wave", DESIGN.md "Corner GS" / "M_II").  The GS sweep
//     D z(i,j) = q(i,j) + aE z(i+1,j) + aN z(i,j+1),   j descending, i descending,
// with zero inflow beyond the top / right edge, runs in one of two forms:
//   YFORM: y = D z obeys  y = q + ya y(i+1,j) + yn y(i,j+1),  ya = aE/D_E, yn = aN/D_N, and
//          z = y / D is formed when the result is written back (corner MG levels; M_II in
//          unweighted mode);
//   z-form: z = q + ca z(i+1,j) + cn z(i,j+1), ca = aE/D, cn = aN/D, where the caller's q is
//          already divided by D (M_II in Jacobi mode: the preconditioner input is D v, R11).
// One corner GS sweep is q = b from zero, or q = b + aW e'(i-1,j) + aS e'(i,j-1) (k_gs_prep,
// fused with the prolongation e' = e + P e_c).
//
// Schedule: one warp per 32-row strip, one lane per row, lane t two columns behind lane t-1 (the
// North value, computed by lane t-1 two steps earlier, arrives by __shfl_up_sync; the East value
// is the lane's own previous result).  With that 2-column skew the band of operands a warp needs
// for 16 consecutive steps is a rectangle in the *sheared* view of an array, element (X, R) at
// address base + R (pitch-2) + X, i.e. row R shifted right by 2R columns.  Each array gets one
// such overlapping 2D TMA tensor map (the row stride (pitch-2)*8 B is a multiple of 16 B), and a
// warp stages a 32-row x 16-column box per array per chunk with one cp.async.bulk.tensor
// (128B swizzle, mbarrier completion) into a 3-slot ring -- two chunks in flight, plus a TMA L2
// prefetch 4 chunks ahead.  At local step k every lane reads box column 15-k of its row.  Results
// go to a padded 2-slot band and are written back as coalesced row segments (the write-back of
// chunk c-1 is interleaved with the steps of chunk c).  Warps of a CTA are chained through a
// shared-memory edge ring.  Tiles of a level run in parallel, each recomputing a certified halo of
// `halo_y` rows above and `halo_x` columns right of its output tile from zero inflow (DESIGN.md
// "Certified halos": |error| <= rho^min(halo) max|y|, rho = max (ya+yn) < 1 per level, halo with
// rho^halo <= 1e-17), so the result equals the sequential sweep to below fp64 rounding.  Without a
// certified halo (M_II: no influence decay in region I at small eps, SURVEY [chk-9]) the row
// strips are chained top-to-bottom across CTAs through global memory (cooperative launch), which
// is the sequential sweep.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <tuple>
#include <type_traits>

#include "kernels.cuh"
#include "tma.cuh"

namespace spp {

constexpr int WCW = 16;          // columns per chunk (box width, 128 bytes)
constexpr int WNS = 3;           // staging ring slots
constexpr int WNA = 4;           // boxes per slot: q (overwritten in place by y), a1, a2, 1/D
constexpr int WBOX = 32 * WCW;   // doubles per box (4 KB)
// doubles per staging slot: 4 boxes in y-form (16 KB), 3 in z-form (12 KB; no 1/D box)
__host__ __device__ constexpr int wslot(bool yform) { return (yform ? WNA : WNA - 1) * WBOX; }
constexpr int WMAXW = 5;         // sweeping warps per CTA (max; 5 only in z-form); +W write-back +1 TMA
constexpr int WEB = 512;         // edge ring (columns): slack between a warp and the one below it
// L2 prefetch distance (chunks; 0 = none).  Measured: none is best -- at cfg5's 4096^2 level 0
// the prefetched boxes of 129 tiles (8 chunks ahead: ~60 MB in flight) were evicted before use
// (cfg5 41.0 -> 39.1 ms per solve without them, cfg4 20.66 -> 20.43 ms).  L2 eviction-priority
// hints on the boxes (keep the certified halos, drop the rest) cut cfg4's level-0 DRAM traffic
// from 188 to 138 MB per sweep but were slower (20.50 / 39.4 ms) and are not used.
#ifndef SPP_WPF
#define SPP_WPF 0
#endif
constexpr int WPF = SPP_WPF;
constexpr int WLAG = 2;
// timing experiments only (wrong results): compile with -DEXP_...
#ifdef EXP_NOSPIN
constexpr bool EXPF_NOSPIN = true;
#else
constexpr bool EXPF_NOSPIN = false;
#endif
#ifdef EXP_NOMBAR
constexpr bool EXPF_NOMBAR = true;
#else
constexpr bool EXPF_NOMBAR = false;
#endif
#ifdef EXP_NOSTS
constexpr bool EXPF_NOSTS = true;
#else
constexpr bool EXPF_NOSTS = false;
#endif
#ifdef EXP_NOEDGE
constexpr bool EXPF_NOEDGE = true;
#else
constexpr bool EXPF_NOEDGE = false;
#endif          // lane-to-lane skew (columns)

struct WaveMaps { CUtensorMap q, a1, a2, cd; };


// chain inflow slots are preset to this NaN (all bits set); the sweep only produces values by
// fma/select, whose NaNs are canonical (0x7fff...), never this pattern
constexpr unsigned long long kChainSentinel = ~0ull;
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire_cta(const int *p)
{
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(double *p, double v)
{
    asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)));
}
// two consecutive values (16-byte aligned p); each 8-byte element is single-copy atomic, which is
// all the value-polling consumer needs
__device__ __forceinline__ void st_relaxed2(double *p, double v0, double v1)
{
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(__double_as_longlong(v0)),
                 "l"(__double_as_longlong(v1)));
}

// predicated forms (the predicate inside the asm: no branch around it)
__device__ __forceinline__ void st_relaxed_if(bool pr, double *p, double v)
{
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %2, 0; @q st.relaxed.gpu.global.b64 [%0], %1; }" ::"l"(p),
                 "l"(__double_as_longlong(v)), "r"((unsigned)pr));
}
__device__ __forceinline__ void st_relaxed2_if(bool pr, double *p, double v0, double v1)
{
    asm volatile("{ .reg .pred q; setp.ne.u32 q, %3, 0; @q st.relaxed.gpu.global.v2.b64 [%0], {%1, %2}; }" ::"l"(p),
                 "l"(__double_as_longlong(v0)), "l"(__double_as_longlong(v1)), "r"((unsigned)pr));
}

// Race-detection build (SPP_STRESS, build.py with SPP_STRESS=1): every hand-off point of the
// sweep -- a sweeping warp's chunk start and its publication to the warp / strip below, the
// write-back warp's slot reads, the TMA producer's issue -- first sleeps a pseudo-random
// 0..~4 us (a hash of the launch's start clock, the block, the warp and the chunk), so the
// producers and consumers of every edge ring, chain buffer and staging slot run in orders the
// normal build never produces.  The results must stay bit-for-bit those of the normal build
// (tools/stress_check.py): any missing acquire / release or a consumer reading a slot early
// shows up as a difference.
#ifdef SPP_STRESS
__device__ __forceinline__ void stress_delay(unsigned long long seed, int where, int c)
{
    unsigned long long h = seed ^ ((unsigned long long)(blockIdx.x + 977u * blockIdx.y) << 20) ^
                           ((unsigned long long)(threadIdx.x >> 5) << 40) ^ ((unsigned long long)where << 50) ^ (unsigned)c;
    h ^= h >> 33; h *= 0xff51afd7ed558ccdull; h ^= h >> 33; h *= 0xc4ceb9fe1a85ec53ull; h ^= h >> 33;
    if ((h & 3u) == 0u) __nanosleep((unsigned)((h >> 8) & 4095u));
}
#define SPP_STRESS_DELAY(where, c) stress_delay(stress_seed, where, c)
#else
#define SPP_STRESS_DELAY(where, c) ((void)0)
#endif

template <bool YFORM, bool CHAIN>
__global__ void __launch_bounds__((2 * WMAXW + 1) * 32) k_wave(WaveArgs a, const __grid_constant__ WaveMaps m)
{
    constexpr int WSLOT = wslot(YFORM);                 // doubles per staging slot
    constexpr int WWARP = WNS * WSLOT;                  // doubles per warp (1 KB multiple)
    extern __shared__ double smem_raw[];
    __shared__ double edge[WMAXW][WEB];
    __shared__ int prod[WMAXW], cons[WMAXW];
    __shared__ __align__(16) double cin[WCW];          // chain inflow of the chunk (warp 0)
    __shared__ __align__(16) double ezero[WCW];        // zero inflow (warp 0 without a chain)
    if (threadIdx.x < WCW) ezero[threadIdx.x] = 0.0;
    // Per (sweeping warp, slot): full = the TMA boxes landed; ready = the sweeping warp stored its
    // results in the slot; empty = the write-back warp stored them to global memory (slot free).
    __shared__ __align__(8) unsigned long long bars[WMAXW][WNS], rbars[WMAXW][WNS], ebars[WMAXW][WNS];
    // warps 0..W-1 sweep 32-row strips; warp W+w writes back the results of warp w; warp 2W is
    // the TMA producer (lane w serves warp w)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = ((blockDim.x >> 5) - 1) / 2;
#ifdef SPP_STRESS
    unsigned long long stress_seed;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(stress_seed));
    stress_seed = __shfl_sync(0xffffffffu, stress_seed, 0);   // one seed per warp (warp-uniform sleeps)
#endif
    if (threadIdx.x < WMAXW) { prod[threadIdx.x] = 0; cons[threadIdx.x] = 0; }
    if (wid < W && lane == 0)
        for (int s = 0; s < WNS; ++s) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bars[wid][s])));
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&rbars[wid][s])));
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&ebars[wid][s])));
        }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const int nl = a.nl;
    // tile (CHAIN: blockIdx.y = row strip block, full width); rows 1..nr_out are output rows,
    // the block's rows above them (up to nr) only halo
    const int out_top = a.nr_out - (int)blockIdx.y * a.rows_out;
    const int out_bot = max(1, out_top - a.rows_out + 1);
    const int top = min(a.nr, out_top + a.halo_y);
    const int out_right = nl - (int)blockIdx.x * a.cols_out;
    const int out_left = max(1, out_right - a.cols_out + 1);
    // The TMA box origin X0 = right + ioff + 2(wtop + joff) - 15 - 16c must be even (16-byte
    // aligned) for the swizzled box, so (right + ioff) must be odd: otherwise one more column is
    // swept -- a genuine halo column inside the level, or the zero ghost column nl+1 where q = 0
    // and the sweep stays exactly 0.
    const int right0 = min(nl, out_right + a.halo_x);
    const int right = ((right0 + a.ioff) & 1) ? right0 : right0 + 1;
    const int ncols = right - out_left + 1;
    const int nch = (ncols + WLAG * 31 + WCW - 1) / WCW;
    // 128B-swizzled TMA boxes need 1 KB aligned shared memory (pointer arithmetic on the shared
    // array keeps the accesses in the shared state space: LDS/STS, not generic LD/ST)
    double *smem = smem_raw + (((1024u - ((unsigned)__cvta_generic_to_shared(smem_raw) & 1023u)) & 1023u) >> 3);
    if (wid == 2 * W) {                                 // ---- TMA producer warp ----
        const int pw = lane;
        const int pwtop = top - 32 * pw;
        if (pw >= W || pwtop < out_bot) return;
        const unsigned ring_s = (unsigned)__cvta_generic_to_shared(smem + (size_t)pw * WWARP);
        // box origin in the sheared view: X = col + 2R (array coordinates), rows wtop-31..wtop
        const int Xb = right + a.ioff + WLAG * (pwtop + a.joff) - (WCW - 1);
        const int R0 = pwtop - 31 + a.joff;
        const unsigned bytes = (YFORM ? 4 : 3) * WBOX * 8;
        for (int c = 0; c < nch; ++c) {
            const int sl = c % WNS;
            if (c >= WNS) mbar_wait((unsigned)__cvta_generic_to_shared(&ebars[pw][sl]), (unsigned)(((c / WNS) - 1) & 1));
            SPP_STRESS_DELAY(1, c);
            const unsigned bar = (unsigned)__cvta_generic_to_shared(&bars[pw][sl]);
            const unsigned dst = ring_s + (unsigned)(sl * WSLOT * 8);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            const int x = Xb - c * WCW;
            tma_load(dst, &m.q, x, R0, bar);
            tma_load(dst + WBOX * 8, &m.a1, x, R0, bar);
            tma_load(dst + 2 * WBOX * 8, &m.a2, x, R0, bar);
            if (YFORM) tma_load(dst + 3 * WBOX * 8, &m.cd, x, R0, bar);
            if (WPF > 0 && c + WPF < nch) {
                const int xp = Xb - (c + WPF) * WCW;
                tma_prefetch(&m.q, xp, R0); tma_prefetch(&m.a1, xp, R0); tma_prefetch(&m.a2, xp, R0);
                if (YFORM) tma_prefetch(&m.cd, xp, R0);
            }
        }
        return;
    }
    const bool wbw = wid >= W;                          // write-back warp
    const int w = wbw ? wid - W : wid;                  // the sweeping warp (strip) served
    const int wtop = top - 32 * w;
    if (wtop < out_bot) return;                         // no rows for this strip
    double *ring = smem + (size_t)w * WWARP;
    if (wbw) {                                          // ---- write-back warp ----
        // element e -> band row t = 2e + lane/16, box column x' = lane%16 (chunk column
        // k = 15 - x'), grid row wtop - t, column right - 16c - 15 + x' + 2t: two coalesced
        // 128-byte row segments per instruction
        const int th = lane >> 4, kk = lane & 15;
        const int pv = (int)a.pv;
        double *const zw = a.z + ((wtop - th + a.joff) * pv + right - (WCW - 1) + kk + WLAG * th + a.ioff);
        const int dwv = 2 * WLAG - 2 * pv;
        unsigned rowmask = 0;                           // elements whose row is an output row
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int t = 2 * e + th;
            if (wtop - t >= out_bot && wtop - t <= out_top) rowmask |= 1u << e;
        }
        // element e of chunk c has sweep index idx = 16c + 15 - kk - WLAG*th - 2*WLAG*e; it is
        // an output column when lo <= idx < ncols (lo = right - out_right): a contiguous e range
        static_assert(WLAG == 2, "the write-back mask divides by 2*WLAG with a shift");
        const int wb_lo = right - out_right;
        const int wb_b0 = (WCW - 1) - kk - WLAG * th;
        int offs[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) {
            const int br = 31 - (2 * e + th);
            offs[e] = br * WCW + ((((kk >> 1) ^ (br & 7))) << 1) + (kk & 1);
        }
        for (int c = 0; c < nch; ++c) {
            const int base = c * WCW + wb_b0;
            const int emax = (base - wb_lo) >> 2;       // floor division (2*WLAG = 4)
            const int emin = ((base - ncols) >> 2) + 1;
            unsigned msk = 0u;
            if (emax >= 0 && emin <= 15) {
                const unsigned hi = emax >= 15 ? 0xffffu : ((2u << emax) - 1u);
                const unsigned lo = emin <= 0 ? 0u : ((1u << emin) - 1u);
                msk = rowmask & hi & ~lo;
            }
            SPP_STRESS_DELAY(2, c);
            mbar_wait((unsigned)__cvta_generic_to_shared(&rbars[w][c % WNS]), (unsigned)((c / WNS) & 1));
            // chunks with nothing to store (halo warps, the staircase ends of a tile) skip the slot
            // reads: 16 shared-memory loads per lane and chunk that only compete with the sweeps
            if (__any_sync(0xffffffffu, msk != 0u)) {
                const double *sl = ring + (size_t)(c % WNS) * WSLOT;
                double *zp = zw - c * WCW;
                double v[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = YFORM ? sl[3 * WBOX + offs[e]] * sl[offs[e]] : sl[offs[e]];
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    if (msk & (1u << e)) *zp = v[e];
                    zp += dwv;
                }
            }
            __syncwarp();                               // every lane's loads of the slot consumed
            if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&ebars[w][c % WNS])) : "memory");
        }
        return;
    }
    // ---- sweeping warp ----
    const int nwa = min(W, (top - out_bot) / 32 + 1);
    const bool has_consumer = w + 1 < nwa;
    const bool chain_in = CHAIN && w == 0 && (blockIdx.y > 0 || a.ext_in != nullptr);
    const bool chain_out = CHAIN && w == nwa - 1 && ((int)blockIdx.y + 1 < (int)gridDim.y || a.chain_last);
    // this lane's row; element (box row 31-t, column x') lives at double offset
    // (31-t)*16 + ((x'/2) ^ ((31-t)&7))*2 + (x'&1)   (128B swizzle)
    const int rowoff = (31 - lane) * WCW, sw = (31 - lane) & 7;
    const int row = wtop - lane;
    const bool rvalid = row >= out_bot;
    const bool rows_all = wtop - 31 >= out_bot;         // all 32 rows of the warp are swept rows
    unsigned long long vin = kChainSentinel;            // chain inflow value in flight (warp 0)
    double z1 = 0.0, z2 = 0.0;                          // own results of the last step (pair)
    int xo[8];                                          // swizzled offsets of this lane's pairs
#pragma unroll
    for (int st = 0; st < 8; ++st) xo[st] = rowoff + (((7 - st) ^ sw) << 1);
#ifdef SPP_WAVE_PROF
    long long tp_spin = 0, tp_bar = 0, tp_steps = 0, tp_wb = 0;
    const long long tp0 = clock64();
    unsigned long long gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
#define SPP_TP(v) const long long v = clock64()
#else
#define SPP_TP(v)
#endif
    for (int c = 0; c < nch; ++c) {
        // chunks without edge handling (warp-uniform test).  Tiled sweeps: every lane's element
        // valid.  Exact chain: no chunk with columns right of the block (sweep index < 0: the first
        // four), which must come out exactly 0 -- the zero inflow at the block's right edge; values
        // left of it (index >= ncols) and below its rows feed only positions outside it (the
        // write-back, the published counts and the polled chain inflow stop at ncols; the chain
        // buffer rows have n + 32 > ncols + 15 slots), so they need nothing.
        const bool fast = CHAIN ? c * WCW - WLAG * 31 >= 0
                                : rows_all && c * WCW - WLAG * 31 >= 0 && c * WCW + WCW - 1 < ncols;
        // North inflow of lane 0 for the columns of this chunk (all wait loops warp-uniform: a
        // lane-divergent spin sends the shuffles below down the slow emulation path)
        SPP_TP(ta);
        SPP_STRESS_DELAY(3, c);
        const int need = min(ncols, c * WCW + WCW);
#ifdef EXP_NOSPIN
        if (false) {
#else
        if (w > 0) {
#endif
            while (ld_acquire_cta(&prod[w - 1]) < need) __nanosleep(32);   // back off: spinning loads slow the working warps' smem traffic
        } else if (chain_in && !EXPF_NOSPIN) {
            // the strip above publishes its bottom row value by value into a buffer preset to the
            // sentinel (no fence on the producer side): lanes 0..15 poll the chunk's 16 columns
            // (the load for chunk c was issued during chunk c-1: vin, so the L2 round trip overlaps
            // the steps; only a value not yet published is polled again)
            const unsigned long long *src = reinterpret_cast<const unsigned long long *>(
                blockIdx.y > 0 ? a.chain_buf + (long)(blockIdx.y - 1) * a.chain_ld : a.ext_in) + c * WCW + (lane & 15);
            const bool mine = lane < 16 && c * WCW + lane < ncols;
            if (c == 0 && mine) vin = ld_relaxed_u64(src);
            for (unsigned spins = 0; !__all_sync(0xffffffffu, !mine || vin != kChainSentinel); ++spins) {
                if (spins > (1u << 26)) __trap();       // a lost value: fail the launch, never hang
                __nanosleep(32);
                if (mine) vin = ld_relaxed_u64(src);
            }
            if (lane < 16) cin[lane] = mine ? __longlong_as_double((long long)vin) : 0.0;
            __syncwarp();
            if (lane < 16 && (c + 1) * WCW + lane < ncols) vin = ld_relaxed_u64(src + WCW);   // chunk c+1
        }
        SPP_TP(t1);
        if (has_consumer && !EXPF_NOSPIN) {             // back-pressure on the edge ring
            const int lim = c * WCW + WCW - WLAG * 31 - WEB;
            if (lim > 0) { while (*((volatile int *)&cons[w + 1]) < lim) __nanosleep(32); }
        }
        SPP_TP(t2);
        // the North inflow is read by lane 0 at the step that uses it (a broadcast 128-bit load
        // with the step's operand loads; eight loads ahead of the operand wait put their latency
        // in front of every chunk: M_II 1.84 -> 1.71 ms per cfg4 solve)
        const double *Eb = w > 0 ? &edge[w - 1][(c * WCW) & (WEB - 1)] : (chain_in ? cin : ezero);
        SPP_TP(tb);
        if (!EXPF_NOMBAR) mbar_wait((unsigned)__cvta_generic_to_shared(&bars[w][c % WNS]), (unsigned)((c / WNS) & 1));
        __syncwarp();
        SPP_TP(tc);
        double *sq = ring + (size_t)(c % WNS) * WSLOT;
        // Two columns per step (the lane skew is two columns, so lane t-1 finished this pair one
        // step earlier, and the pair shares one 16-byte swizzle unit: one 128-bit load per array).
        // Every shared-memory load of the chunk is issued before the first store: a store ahead
        // of a possibly aliasing load would serialise the load behind it.
        // The operands of a step are loaded at that step (volatile asm: the compiler keeps them
        // there).  Issued as one burst of 24 128-bit loads before the steps, they queued in the
        // shared-memory pipe ahead of the shuffles of the dependent step chain (measured: cfg4
        // 21.0 -> 19.3 ms/solve; loading one or two steps ahead, or storing per step, is slower).
        // The stores below touch only the q slots of this chunk's columns: no load aliases them.
        auto lds2 = [](const double *pp) {
            double2 v;
            asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(pp)));
            return v;
        };
        if (w > 0 && lane == 0) *((volatile int *)&cons[w]) = need;
        auto steps = [&](auto fast_tag) {
            constexpr bool F = decltype(fast_tag)::value;
            double Z[16];
#pragma unroll
            for (int st = 0; st < 8; ++st) {
                const double2 Q = lds2(sq + xo[st]);                 // (2st+1, 2st) as (lo, hi)
                const double2 A1 = lds2(sq + WBOX + xo[st]);
                const double2 A2 = lds2(sq + 2 * WBOX + xo[st]);
                double n0 = __shfl_up_sync(0xffffffffu, z2, 1);    // lane t-1's pair of the last step
                double n1 = __shfl_up_sync(0xffffffffu, z1, 1);
                const double2 Es = lds2(Eb + 2 * st);             // North inflow (lane 0)
                if (lane == 0) { n0 = Es.x; n1 = Es.y; }
                double za, zc;
                if (CHAIN) {
                    // exact chain (M_II), right of the block (first four chunks only): q = 0 there,
                    // and with the zero initial East value and lane 0's inflow (index >= 0 always)
                    // every value there is exactly +0 -- the block edge's zero inflow -- with
                    // neither a mask nor a select on the step chain (the pair (idx, idx+1) has idx
                    // even: both columns on the same side).  M_II 1.54 -> 1.50 ms per cfg4 solve
                    // against a select of the East input at idx = 0 (and that one against per-value
                    // masks: 1.70 -> 1.53).  On the tiled levels the same change measured slower
                    // (mg_sweep 6.26 -> 6.51 ms per solve), so they keep the masks below.
                    double qy = Q.y, qx = Q.x;
                    if (!F) {
                        const bool in = c * WCW + 2 * st - WLAG * lane >= 0;
                        qy = in ? qy : 0.0; qx = in ? qx : 0.0;
                    }
                    za = fma(A1.y, z1, fma(A2.y, n0, qy));           // column 2st   (east one first)
                    zc = fma(A1.x, za, fma(A2.x, n1, qx));           // column 2st+1
                } else {
                    za = fma(A1.y, z1, fma(A2.y, n0, Q.y));
                    zc = fma(A1.x, za, fma(A2.x, n1, Q.x));
                    if (!F) {                              // edge chunk: zero outside the block
                        // one AND per value on the chain (the masks do not depend on it); a ternary
                        // compiled to three dependent selects.  (Masking the operands instead keeps
                        // the masks off the chain but costs six ANDs per step: measured slower on the
                        // tiled levels, 6.37 -> 6.90 ms of sweeps per cfg4 solve.)
                        const int idx = c * WCW + 2 * st - WLAG * lane;
                        const unsigned ua = (unsigned)idx < (unsigned)ncols, uc = (unsigned)(idx + 1) < (unsigned)ncols;
                        const long long ma = -(long long)(rvalid & ua), mc = -(long long)(rvalid & uc);
                        za = __longlong_as_double(__double_as_longlong(za) & ma);
                        zc = __longlong_as_double(__double_as_longlong(zc) & mc);
                    }
                }
                Z[2 * st] = za; Z[2 * st + 1] = zc;
                z2 = za; z1 = zc;
            }
            if (!EXPF_NOSTS) {
#pragma unroll
            for (int st = 0; st < 8; ++st)
                *reinterpret_cast<double2 *>(sq + xo[st]) = make_double2(Z[2 * st + 1], Z[2 * st]);   // y in place of q
            }
            // hand the bottom row to the next strip (lane 31's pairs): branch-free predicated
            // stores on interior chunks, element-wise checks at the edges
            SPP_STRESS_DELAY(5, c);                       // delays the hand-off stores below
            double *eo = &edge[w][0];
            double *co = CHAIN ? a.chain_buf + (long)blockIdx.y * a.chain_ld : nullptr;
            if (F) {
                const bool e31 = lane == 31 && has_consumer && !EXPF_NOEDGE;
                const bool c31 = CHAIN && lane == 31 && chain_out && !EXPF_NOEDGE;
#pragma unroll
                for (int st = 0; st < 8; ++st) {
                    const int idx = c * WCW + 2 * st - WLAG * 31;
                    if (e31) *reinterpret_cast<double2 *>(eo + (idx & (WEB - 1))) = make_double2(Z[2 * st], Z[2 * st + 1]);
                    if (c31) st_relaxed2(co + idx, Z[2 * st], Z[2 * st + 1]);
                }
            } else {
                // edge chunk: the same stores, predicated (the conditions are warp-uniform but for
                // lane == 31; a lane-31-only branch around them had the warp reconverge per chunk)
                const bool e31 = lane == 31 && has_consumer && !EXPF_NOEDGE;
                const bool c31 = CHAIN && lane == 31 && chain_out && !EXPF_NOEDGE;
#pragma unroll
                for (int st = 0; st < 8; ++st) {
                    const int idx = c * WCW + 2 * st - WLAG * 31;
                    const bool two = idx >= 0 && idx + 1 < ncols, one = idx >= 0 && idx + 1 == ncols;   // last odd column
                    const int io = two || one ? idx : 0;
                    double *ep = eo + (io & (WEB - 1));
                    if (e31 && two) *reinterpret_cast<double2 *>(ep) = make_double2(Z[2 * st], Z[2 * st + 1]);
                    if (e31 && one) *ep = Z[2 * st];
                    if (CHAIN) {
                        st_relaxed2_if(c31 && two, co + io, Z[2 * st], Z[2 * st + 1]);
                        st_relaxed_if(c31 && one, co + io, Z[2 * st]);
                    }
                }
            }
        };
        if (fast) steps(std::true_type{});
        else steps(std::false_type{});
        SPP_TP(td);
        const int done = min(ncols, max(0, c * WCW + WCW - WLAG * 31));
        __syncwarp();
        SPP_STRESS_DELAY(4, c);
        if (lane == 0) asm volatile("mbarrier.arrive.shared.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&rbars[w][c % WNS])) : "memory");
        if (lane == 31 && has_consumer)                 // release: the edge values before the count
            asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&prod[w])), "r"(done) : "memory");
#ifdef SPP_WAVE_PROF
        SPP_TP(te);
        tp_spin += tb - ta; tp_bar += tc - tb; tp_steps += td - tc; tp_wb += te - td;
        if (lane == 0 && a.prof && blockIdx.x == 0 && blockIdx.y < 2 && c < 160) {
            long long *tl = a.prof + 8 * 8 * 8192 + (((long)blockIdx.y * 8 + w) * 160 + c) * 8;
            tl[0] = ta; tl[1] = t1; tl[2] = t2; tl[3] = tb; tl[4] = tc; tl[5] = td; tl[6] = te; tl[7] = 1;
        }
#endif
    }
#ifdef SPP_WAVE_PROF
    if (lane == 0 && a.prof) {
        unsigned long long gt1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
        long long *o = a.prof + 8 * ((blockIdx.y * gridDim.x + blockIdx.x) * 8 + w);
        o[0] = clock64() - tp0; o[1] = tp_spin; o[2] = tp_bar; o[3] = tp_steps; o[4] = tp_wb; o[5] = nch;
        o[6] = (long long)gt0; o[7] = (long long)gt1;
    }
#endif
}

static size_t wave_smem(int warps, bool yform) { return sizeof(double) * (size_t)warps * WNS * wslot(yform) + 1024; }

#ifdef SPP_WAVE_PROF
// debugging build only: per-warp cycle breakdown (spin = waits on the warp above / chain,
// bar = waits on the TMA boxes, steps = the recurrence, wb = hand-offs) and the warps' start /
// end times relative to the launch's first warp, for the SPP_WAVE_PROF_HIT-th launch (default 3)
// over a level of SPP_WAVE_PROF_N columns (default: the corner, n)
static void wave_prof_dump(Ctx *c, long long *prof, const char *what, int nctas, int nl)
{
    static int hits = 0;
    const char *en = getenv("SPP_WAVE_PROF_N"), *eh = getenv("SPP_WAVE_PROF_HIT");
    const int want = en ? atoi(en) : c->n, hit = eh ? atoi(eh) : 3;
    if (!what || nl != want || ++hits != hit) return;
    const int nw = std::min(nctas, 512) * 8;
    std::vector<long long> h(8 * (size_t)nw);
    cudaMemcpyAsync(h.data(), prof, sizeof(long long) * 8 * nw, cudaMemcpyDeviceToHost, c->st);
    cudaStreamSynchronize(c->st);
    long long g0 = -1, g1 = 0;
    for (int k = 0; k < nw; ++k)
        if (h[8 * k]) { g0 = g0 < 0 ? h[8 * k + 6] : std::min(g0, h[8 * k + 6]); g1 = std::max(g1, h[8 * k + 7]); }
    fprintf(stderr, "[wave-prof] %s n=%d: %d CTAs, first warp start -> last warp end %.2f us\n", what, nl, nctas, (g1 - g0) * 1e-3);
    if (getenv("SPP_WAVE_TL")) {                        // per-chunk timeline of CTA rows 0, 1 (clock64)
        std::vector<long long> tl(2 * 8 * 160 * 8);
        cudaMemcpy(tl.data(), prof + 8 * 8 * 8192, sizeof(long long) * tl.size(), cudaMemcpyDeviceToHost);
        long long t0 = -1;
        for (int w = 0; w < 8; ++w) if (tl[((0 * 8 + w) * 160) * 8 + 7]) t0 = t0 < 0 ? tl[((0 * 8 + w) * 160) * 8] : std::min(t0, tl[((0 * 8 + w) * 160) * 8]);
        for (int y = 0; y < 2; ++y)
            for (int w = 0; w < 8; ++w)
                for (int cc = 0; cc < 160; ++cc) {
                    const long long *r = &tl[((y * 8 + w) * 160 + cc) * 8];
                    if (!r[7] || (cc > 12 && cc % 16 != 0)) continue;
                    fprintf(stderr, "[wave-tl] y%d w%d c%3d: start %8lld | wait %6lld bp %6lld E %5lld mbar %5lld steps %5lld post %5lld\n",
                            y, w, cc, y == 0 ? r[0] - t0 : r[0], r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4],
                            r[6] - r[5]);
                }
    }
    for (int k = 0; k < nw; ++k)
        if (h[8 * k] && (k / 8 < 4 || k / 8 == nctas - 1))
            fprintf(stderr, "[wave-prof]  cta %d warp %d: start %+.2f us end %+.2f us | cycles total %lld spin %lld bar %lld "
                            "steps %lld wb %lld | nch %lld\n", k / 8, k % 8, (h[8 * k + 6] - g0) * 1e-3,
                    (h[8 * k + 7] - g0) * 1e-3, h[8 * k], h[8 * k + 1], h[8 * k + 2], h[8 * k + 3], h[8 * k + 4], h[8 * k + 5]);
}
#endif

// SPP_DEBUG_SYNC=1: synchronise and report after every launch of this file (debugging aid)
static void dbg_sync(Ctx *c, const char *what)
{
    static int on = -1;
    if (on < 0) { const char *e = getenv("SPP_DEBUG_SYNC"); on = (e && e[0] == '1') ? 1 : 0; }
    if (!on || c->capturing) return;
    cudaError_t e = cudaStreamSynchronize(c->st);
    if (e == cudaSuccess) e = cudaGetLastError();
    fprintf(stderr, "[spp-debug] %s: %s\n", what, cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------------- tensor maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

struct CoarseArgs;
__global__ void k_coarse_vcycle(CoarseArgs a);
cudaError_t wave_init()
{
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        SPP_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&g_encode, cudaEnableDefault, &q));
        if (!g_encode || q != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
    }
    const int smy = (int)wave_smem(4, true), smz = (int)wave_smem(WMAXW, false);
    SPP_CUDA_TRY(cudaFuncSetAttribute(k_wave<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smy));
    SPP_CUDA_TRY(cudaFuncSetAttribute(k_wave<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smz));
    SPP_CUDA_TRY(cudaFuncSetAttribute(k_wave<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smy));
    SPP_CUDA_TRY(cudaFuncSetAttribute(k_wave<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smz));
    SPP_CUDA_TRY(cudaFuncSetAttribute(k_coarse_vcycle, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    return cudaSuccess;
}

// Sheared view of a padded array of `rows` rows x `pitch` doubles: element (X, R) at
// base + R (pitch - 2) + X; box 16 x 32, 128B swizzle.  Cached per (pointer, pitch, rows).
static const CUtensorMap *sheared_map(Ctx *c, const double *base, long pitch, long rows)
{
    auto key = std::make_tuple((const void *)base, pitch, rows);
    auto it = c->tmaps.find(key);
    if (it != c->tmaps.end()) return &it->second;
    CUtensorMap tm;
    cuuint64_t dim[2] = {(cuuint64_t)(pitch + WLAG * rows + 64), (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)(pitch - WLAG) * sizeof(double)};
    cuuint32_t box[2] = {WCW, 32}, es[2] = {1, 1};
    CUresult rc = g_encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dim, str, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) return nullptr;
    return &(c->tmaps[key] = tm);
}

// Generic 2D fp64 tensor map (dims d0 x d1 elements, row stride in bytes, box b0 x b1), cached.
const CUtensorMap *tmap2d(Ctx *c, const void *base, unsigned long long d0, unsigned long long d1,
                          unsigned long long stride_bytes, unsigned b0, unsigned b1, bool swz128)
{
    auto key = std::make_tuple(base, d0, d1, stride_bytes, b0, b1, swz128);
    auto it = c->tmaps2.find(key);
    if (it != c->tmaps2.end()) return &it->second;
    CUtensorMap tm;
    cuuint64_t dim[2] = {(cuuint64_t)d0, (cuuint64_t)d1};
    cuuint64_t str[1] = {(cuuint64_t)stride_bytes};
    cuuint32_t box[2] = {b0, b1}, es[2] = {1, 1};
    CUresult rc = g_encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void *)base, dim, str, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) return nullptr;
    return &(c->tmaps2[key] = tm);
}

static bool wave_maps(Ctx *c, const WaveArgs &a, long rows_v, long rows_c, WaveMaps *m)
{
    const CUtensorMap *q = sheared_map(c, a.q, a.pv, rows_v);
    const CUtensorMap *x = sheared_map(c, a.ca, a.pc, rows_c);
    const CUtensorMap *y = sheared_map(c, a.cn, a.pc, rows_c);
    const CUtensorMap *d = sheared_map(c, a.cd, a.pc, rows_c);
    if (!q || !x || !y || !d) return false;
    m->q = *q; m->a1 = *x; m->a2 = *y; m->cd = *d;
    return true;
}

// Tiled (certified halo) or single-tile sweep of a level-shaped square [1, nl]^2 of an array with
// `rows` rows.
void launch_wave(Ctx *c, WaveArgs a, long rows_v, long rows_c, int warps, bool yform, int cls, double bytes)
{
    WaveMaps m;
    if (!wave_maps(c, a, rows_v, rows_c, &m)) { c->sticky = cudaErrorInvalidValue; return; }
    if (a.nr <= 0) { a.nr = a.nl; a.nr_out = a.nl; }
    const dim3 grid((a.nl + a.cols_out - 1) / a.cols_out, (a.nr_out + a.rows_out - 1) / a.rows_out);
    const size_t sm = wave_smem(warps, yform);
    ProfScope ps(c, cls, bytes);
#ifdef SPP_WAVE_PROF
    static long long *prof = nullptr;
    if (!prof) cudaMalloc(&prof, sizeof(long long) * (8 * 8 * 8192 + 2 * 8 * 160 * 8));
    cudaMemsetAsync(prof, 0, sizeof(long long) * (8 * 8 * 8192 + 2 * 8 * 160 * 8), c->st);
    a.prof = prof;
#endif
    if (yform) k_wave<true, false><<<grid, (2 * warps + 1) * 32, sm, c->st>>>(a, m);
    else k_wave<false, false><<<grid, (2 * warps + 1) * 32, sm, c->st>>>(a, m);
    c->launches++;
#ifdef SPP_WAVE_PROF
    wave_prof_dump(c, prof, "tiled", grid.x * grid.y, a.nl);
#endif
    dbg_sync(c, "k_wave tiled");
}

static int chain_warps(const Ctx *c) { return std::max(1, std::min(c->tune.sweep_warps, WMAXW)); }
// CTAs (row strips of 32 W rows) of an exact chained sweep over `rows` rows; the chain buffer is
// sized from this (capi.cu alloc_all)
long wave_chain_ctas(const Ctx *c, long rows) { const long r = 32L * chain_warps(c); return (rows + r - 1) / r; }

// Exact sweep: row strips of 32*W rows chained top-to-bottom across CTAs (cooperative launch).
void launch_wave_chain(Ctx *c, WaveArgs a, long rows_v, long rows_c, bool yform, int cls, double bytes)
{
    WaveMaps m;
    if (!wave_maps(c, a, rows_v, rows_c, &m)) { c->sticky = cudaErrorInvalidValue; return; }
    const int W = chain_warps(c);
    a.rows_out = 32 * W; a.halo_y = 0;
    a.cols_out = a.nl; a.halo_x = 0;
    if (a.nr <= 0) { a.nr = a.nl; a.nr_out = a.nl; }
    const int ncta = (int)wave_chain_ctas(c, a.nr_out);
    a.chain_flags = c->chain_flags;
    a.chain_buf = c->chain;
    a.chain_ld = c->chain_ld;
    {
        const cudaError_t e = cudaMemsetAsync(c->chain, 0xff, sizeof(double) * (size_t)ncta * c->chain_ld, c->st);   // kChainSentinel
        if (e != cudaSuccess && c->sticky == cudaSuccess) c->sticky = e;
    }
    const size_t sm = wave_smem(W, yform);
    void *args[] = {(void *)&a, (void *)&m};
    ProfScope ps(c, cls, bytes);
#ifdef SPP_WAVE_PROF
    static long long *prof = nullptr;
    if (!prof) cudaMalloc(&prof, sizeof(long long) * (8 * 8 * 8192 + 2 * 8 * 160 * 8));
    cudaMemsetAsync(prof, 0, sizeof(long long) * (8 * 8 * 8192 + 2 * 8 * 160 * 8), c->st);
    a.prof = prof;
#endif
    const cudaError_t le = yform
        ? cudaLaunchCooperativeKernel((void *)k_wave<true, true>, dim3(1, ncta), dim3(32 * (2 * W + 1)), args, sm, c->st)
        : cudaLaunchCooperativeKernel((void *)k_wave<false, true>, dim3(1, ncta), dim3(32 * (2 * W + 1)), args, sm, c->st);
    if (le != cudaSuccess && c->sticky == cudaSuccess) c->sticky = le;
    c->launches++;
#ifdef SPP_WAVE_PROF
    wave_prof_dump(c, prof, "chain", ncta, a.nl);
#endif
    dbg_sync(c, "k_wave chain");
}

// g = b + aW e'(i-1,j) + aS e'(i,j-1) with e' = e + P e_c (e_c may be null): the right-hand side
// of the y-form recurrence of a GS sweep from e' (the parallel W/S part), fused with the
// prolongation and coarse-grid correction; e' itself is never stored.

// One block-iteration = one row segment of 2*blockDim columns starting at the ghost column 0; each
// thread owns a column pair (i0, i0+1), i0 even: 16-byte loads of b, 1/D, aW and of the South
// row of e, one 16-byte store, and the interpolation's branch on the parity of i resolved at
// compile time (one node per thread had the lanes of a warp alternate between its branches).
// The arithmetic per node is unchanged.
template <bool UNI>
__global__ void __launch_bounds__(256) k_gs_prep(int nl, long pv, const double *__restrict__ e,
    const double *__restrict__ ec, long pcv, const double *__restrict__ b,
    const double *__restrict__ aW, const double *__restrict__ aS, double *g,
    const double *__restrict__ cd, long pc, int bscaled, int j0, int j1, Wts W)
{
    auto ld2 = [](const double *p) { return *reinterpret_cast<const double2 *>(p); };
    const int segw = 2 * blockDim.x;
    const int nseg = (nl + 1 + segw - 1) / segw;        // columns 0 .. nl
    const long nit = (long)(j1 - j0 + 1) * nseg;        // rows j0 .. j1 of the level
    for (long it = blockIdx.x; it < nit; it += gridDim.x) {
        const int j = (int)(it / nseg) + j0;
        const int i0 = (int)(it % nseg) * segw + 2 * threadIdx.x;
        if (i0 > nl) continue;
        const bool ok0 = i0 >= 1, ok1 = i0 + 1 <= nl;   // valid columns of the pair
        const long v = (long)j * pv + i0;
        const double2 es2 = ld2(e + v - pv);            // e(i0, j-1), e(i0+1, j-1)
        double ew0 = ok0 ? e[v - 1] : 0.0, ew1 = e[v];  // e(i0-1, j), e(i0, j)
        double es0 = es2.x, es1 = es2.y;
        if (ec) {
            ew0 += (i0 > 1) ? interp_p<UNI, true>(ec, pcv, i0 - 1, j, W) : 0.0;
            es0 += (j > 1) ? interp_p<UNI, false>(ec, pcv, i0, j - 1, W) : 0.0;
            ew1 += (i0 > 0) ? interp_p<UNI, false>(ec, pcv, i0, j, W) : 0.0;
            es1 += (j > 1) ? interp_p<UNI, true>(ec, pcv, i0 + 1, j - 1, W) : 0.0;
        }
        const double2 vb = ld2(b + v), vW = ld2(aW + i0);
        const double vS = aS[j];
        double2 out;
        if (!cd) {
            out.x = (vb.x + vW.x * ew0) + vS * es0;
            out.y = (vb.y + vW.y * ew1) + vS * es1;
        } else {
            const double2 dinv = ld2(cd + (long)j * pc + i0);   // z-form sweeps take g / D
            out.x = bscaled ? vb.x + (vW.x * ew0 + vS * es0) * dinv.x : ((vb.x + vW.x * ew0) + vS * es0) * dinv.x;
            out.y = bscaled ? vb.y + (vW.y * ew1 + vS * es1) * dinv.y : ((vb.y + vW.y * ew1) + vS * es1) * dinv.y;
        }
        if (ok0 && ok1) *reinterpret_cast<double2 *>(g + v) = out;
        else if (ok0) g[v] = out.x;
        else if (ok1) g[v + 1] = out.y;
    }
}

// q = b / D (z-form sweep from zero for a right-hand side nobody pre-scaled: test hooks)
__global__ void k_scale_cd(int nl, long pv, long pc, const double *__restrict__ b, const double *__restrict__ cd, double *q)
{
    const long tot = (long)nl * nl;
    for (GridWalk gw(tot, nl, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        q[(long)j * pv + i] = b[(long)j * pv + i] * cd[(long)j * pc + i];
    }
}

static inline int gblocks(long work) { long b = (work + 255) / 256; return (int)std::max(1L, std::min(b, 148L * 16)); }

// level l's g = b / D (z-form pre-smoothing rhs when no producer wrote it)
void launch_scale_cd(Ctx *c, int l, const double *b, double *q)
{
    Level &L = c->lev[l];
    k_scale_cd<<<gblocks((long)L.n * L.n), 256, 0, c->st>>>(L.n, L.pitch, L.cpitch, b, L.cd, q);
    c->launches++;
}

// One downstream GS sweep on level l: mode 0 from zero (q = b); mode 1 from e_old (+ P ec when
// ec != null): q = prep(e_old [+ P ec]).  z-form (c->mg_zform): z = q + (aE/D) z_E + (aN/D) z_N
// with q = rhs/D; inside the V-cycle the level right-hand sides are stored divided by D
// (bscaled), so mode 0 streams b itself; a caller's plain rhs is scaled here.  y-form:
// y = q + ya y_E + yn y_N, z = y/D at write-back.
// The parallel part of a GS sweep from e_old (+ P ec): q = prep(e_old [+ P ec]) into L.g on the
// level's rows (a row strip's own rows in a distributed solve).
void launch_gs_prep(Ctx *c, int l, const double *b, const double *eold, const double *ec, bool bscaled)
{
    Level &L = c->lev[l];
    const bool zf = c->mg_zform;
    const int j0 = L.sdist ? L.slo : 1, j1 = L.sdist ? L.shi : L.n;
    ProfScope ps(c, 5, (double)L.n * (j1 - j0 + 1) * (zf ? 32.0 : 24.0));
    auto kp = L.w.uni ? k_gs_prep<true> : k_gs_prep<false>;
    // a thread per column pair; a block no wider than a row needs (the small levels)
    // (the row's pairs spread evenly over its segments, as seg_shape does)
    const int prs = (L.n + 2) / 2, nsg = (prs + 255) / 256;
    const int nt = std::max(32, std::min(256, ((prs + nsg - 1) / nsg + 31) / 32 * 32));
    const long pairs = (long)(j1 - j0 + 1) * (((L.n + 1 + 2 * nt - 1) / (2 * nt)) * (long)nt);
    kp<<<(int)std::max(1L, std::min((pairs + nt - 1) / nt, 148L * 16)), nt, 0, c->st>>>(L.n, L.pitch, eold, ec,
        ec ? c->lev[l + 1].pitch : 0, b, L.aW, L.aS, L.g, zf ? L.cd : nullptr, L.cpitch, bscaled ? 1 : 0, j0, j1, L.w);
    c->launches++;
    dbg_sync(c, "k_gs_prep");
}

// The downstream recurrence of a GS sweep of level l for the right-hand side q (already in the
// sweep's form): tiled with certified halos, one exact CTA, or the exact chain; on a row strip
// the own rows plus L.shalo halo rows above.
void launch_gs_sweep(Ctx *c, int l, const double *q, double *enew)
{
    Level &L = c->lev[l];
    const bool zf = c->mg_zform;
    WaveArgs a{};
    a.nl = L.n; a.pv = L.pitch; a.pc = L.cpitch;
    if (zf) { a.ca = l == 0 ? c->ca : L.ya; a.cn = l == 0 ? c->cn : L.yn; }   // levels >= 1 keep aE/D, aN/D in ya, yn
    else { if (l == 0) ensure_y0(c); a.ca = L.ya; a.cn = L.yn; }
    a.cd = L.cd; a.z = enew; a.q = q;
    if (L.sdist) {                                  // row strip: own rows + halo rows above
        a.joff = L.slo - 1;
        a.nr_out = L.shi - L.slo + 1;
        a.nr = a.nr_out + L.shalo;
    }
    const double bytes = (double)L.n * (a.nr_out > 0 ? a.nr_out : L.n) * (zf ? 32.0 : 40.0);   // q, couplings (+ 1/D in y-form) read; z written
    const long rows_v = L.n + 2, rows_c = l == 0 ? c->N + 1 : L.n + 2;   // level 0 shares the global coefficients
    if (L.tile_warps == 0) { launch_wave_chain(c, a, rows_v, rows_c, !zf, 3, bytes); return; }
    a.rows_out = L.tile_rows; a.cols_out = L.tile_cols; a.halo_y = L.halo_y; a.halo_x = L.halo_x;
    launch_wave(c, a, rows_v, rows_c, L.tile_warps, !zf, 3, bytes);
}

// One downstream GS sweep on level l: mode 0 from zero (q = b); mode 1 from e_old (+ P ec when
// ec != null): q = prep(e_old [+ P ec]).  z-form (c->mg_zform): z = q + (aE/D) z_E + (aN/D) z_N
// with q = rhs/D; inside the V-cycle the level right-hand sides are stored divided by D
// (bscaled), so mode 0 streams b itself; a caller's plain rhs is scaled here.  y-form:
// y = q + ya y_E + yn y_N, z = y/D at write-back.
void launch_gs(Ctx *c, int l, int mode, const double *b, const double *eold, double *enew, const double *ec,
               bool bscaled)
{
    Level &L = c->lev[l];
    const bool zf = c->mg_zform;
    const double *q = b;
    if (mode == 0) {
        if (zf && !bscaled) { launch_scale_cd(c, l, b, L.g); q = L.g; }
    } else {
        launch_gs_prep(c, l, b, eold, ec, bscaled);
        q = L.g;
    }
    launch_gs_sweep(c, l, q, enew);
}

// ------------------------------------------------------------------------------------------
// Coarse V-cycle (levels with n <= kCoarseMaxN): one CTA runs the
// whole V(1,1) cycle of P:1205-1209 / P:1281-1283 for levels lc..L-1.  Every level's b, e and
// coefficients are staged into shared memory once (zero ghost ring), so no step waits on L2.
//   down: e_l = GS(b_l) from 0; rho = b_l - A_l e_l; b_{l+1} = S^-1 P^T S rho
//   coarsest: 4 GS sweeps from 0
//   up:   e_l += P e_{l+1}; e_l = GS(b_l) from e_l
// GS is the sequential downstream sweep (j desc, i desc; E/N new, W/S old) done in place as a
// one-warp wavefront: lane t owns row j = n - t and meets column i = n - (s - t) at step s, so
// its East neighbour is its own previous step, its North one lane t-1's previous step (through
// shared memory behind __syncwarp), and West / South are still old.  2n - 1 steps of a few
// shared-memory loads each; no block barrier inside a sweep.
// ------------------------------------------------------------------------------------------
constexpr int kCoarseMaxN = 32;     // one warp: one row per lane

struct CoarseLev {
    int n; int cpitch;
    const double *aE, *aN, *rr, *cd, *aW, *aS, *hb, *kb;
    Wts w;                          // interpolation weights from the next coarser level
};
struct CoarseArgs {
    int nlev;                       // levels lc .. lc+nlev-1 (the last is the coarsest)
    CoarseLev lv[8];
    const double *R; long rpitch;   // rhs of level lc (value layout)
    int rs;                         // R stored as R / D (z-form V-cycle)
    double *out; long opitch;       // result e of level lc (value layout)
};
// a level's shared-memory image: offsets into the block's shared array of (n+2)^2 arrays with
// stride st = n+2 and of 1D arrays of n+2 (offsets, not pointers: the accesses stay LDS/STS and
// the image copies into registers)
struct CSm { int b, e, aE, aN, cd, rr, aW, aS, hb, kb, n, st, ca, cn; };
extern __shared__ double coarse_sm[];

__device__ __forceinline__ void cgs_sweep(const CSm L, double *q)
{
    double *cs = coarse_sm;
    const int n = L.n, st = L.st;
    // the parallel part first (all threads): q = (b + aW e_W + aS e_S) / D from the old e, then
    // the z-form recurrence z = q + ca z_E + cn z_N (ca = aE/D, cn = aN/D) by one warp
    {
        const double *b = cs + L.b, *e = cs + L.e, *cd = cs + L.cd;
        for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
            const int j = k / n + 1, i = k % n + 1, s = j * st + i;
            q[s] = ((b[s] + cs[L.aW + i] * e[s - 1]) + cs[L.aS + j] * e[s - st]) * cd[s];
        }
    }
    __syncthreads();
    if (threadIdx.x < 32) {
        const int t = threadIdx.x;
        const bool act = t < n;
        const int j = n - t;
        const double *ca = cs + L.ca, *cn = cs + L.cn;
        double *e = cs + L.e;
        // one warp, lane t owns row j = n - t and meets column i = n - (s - t) at step s: East is
        // the lane's previous step (0 at the block edge), North lane t-1's previous step (shuffle;
        // lane 0: the ghost row).  Branch-free (idle lanes read a valid dummy node and keep their
        // value), the operands of the next step loaded after the step's shuffle.
        const int jj = act ? j : 1;
        auto ld = [&](int ii, double &Q, double &A, double &Nc) {
            const int ic = (ii >= 1 && ii <= n) ? ii : 1, o = jj * st + ic;
            Q = q[o]; A = ca[o]; Nc = cn[o];
        };
        double Q, A, Nc;
        ld(n + t, Q, A, Nc);
        double vlast = 0.0;
        for (int s = 0; s < 2 * n - 1; ++s) {
            const int i = n - (s - t);
            const bool ok = act && i >= 1 && i <= n;
            double vN = __shfl_up_sync(0xffffffffu, vlast, 1);
            if (t == 0) vN = 0.0;
            double Qn, An, Nn;
            ld(i - 1, Qn, An, Nn);
            const double z = fma(A, vlast, fma(Nc, vN, Q));
            vlast = ok ? z : vlast;
            if (ok) e[jj * st + i] = z;
            Q = Qn; A = An; Nc = Nn;
        }
    }
    __syncthreads();
}

#ifdef SPP_COARSE_PROF
__device__ int g_coarse_prof = 0;
#define CTP(k) do { if (threadIdx.x == 0) tp[k] = clock64(); } while (0)
#else
#define CTP(k)
#endif
__global__ void __launch_bounds__(256) k_coarse_vcycle(CoarseArgs a)
{
    double *cs = coarse_sm;
#ifdef SPP_COARSE_PROF
    long long tp[16] = {0};
#endif
    CTP(0);
    CSm S[8];
    int p = 0;
    for (int l = 0; l < a.nlev; ++l) {
        const int n = a.lv[l].n, st = n + 2, A = st * st;
        S[l] = CSm{p, p + A, p + 2 * A, p + 3 * A, p + 4 * A, p + 5 * A, p + 6 * A, p + 6 * A + st, p + 6 * A + 2 * st,
                   p + 6 * A + 3 * st, n, st, p + 6 * A + 4 * st, p + 7 * A + 4 * st};
        p += 8 * A + 4 * st;
    }
    double *rho = cs + p;
    // zero ghost rings: b, e of every level and rho (the coefficient images are fully staged)
    for (int l = 0; l < a.nlev; ++l)
        for (int k = threadIdx.x; k < 2 * S[l].st * S[l].st; k += blockDim.x) cs[S[l].b + k] = 0.0;
    for (int k = threadIdx.x; k < S[0].st * S[0].st; k += blockDim.x) rho[k] = 0.0;
    __syncthreads();
    CTP(1);
    // stage the coefficients and the rhs with asynchronous copies: every load in flight at once
    auto cp8 = [&](int dst, const double *src) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(cs + dst)), "l"(src)
                     : "memory");
    };
    for (int l = 0; l < a.nlev; ++l) {
        const CoarseLev &F = a.lv[l];
        const CSm M = S[l];
        const int n = F.n;
        for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
            const int j = k / n + 1, i = k % n + 1, q = j * F.cpitch + i, s = j * M.st + i;
            cp8(M.aE + s, F.aE + q); cp8(M.aN + s, F.aN + q); cp8(M.cd + s, F.cd + q); cp8(M.rr + s, F.rr + q);
            if (l == 0) cp8(M.b + s, a.R + (long)j * a.rpitch + i);
        }
        for (int k = threadIdx.x; k < n + 2; k += blockDim.x) {
            cp8(M.aW + k, F.aW + k); cp8(M.aS + k, F.aS + k); cp8(M.hb + k, F.hb + k); cp8(M.kb + k, F.kb + k);
        }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    CTP(2);
    if (a.rs) {                                        // level lc rhs stored as R / D -> R
        const CSm M = S[0];
        const int n = M.n;
        for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
            const int j = k / n + 1, i = k % n + 1, s = j * M.st + i;
            cs[M.b + s] *= ((cs[M.aW + i] + cs[M.aE + s]) + (cs[M.aS + j] + cs[M.aN + s])) + cs[M.rr + s];
        }
    }
    for (int l = 0; l < a.nlev; ++l) {                  // z-form couplings ca = aE/D, cn = aN/D
        const CSm M = S[l];
        for (int k = threadIdx.x; k < M.st * M.st; k += blockDim.x) {
            const int j = k / M.st, i = k % M.st;
            const bool in = i >= 1 && i <= M.n && j >= 1 && j <= M.n;
            cs[M.ca + k] = in ? cs[M.aE + k] * cs[M.cd + k] : 0.0;
            cs[M.cn + k] = in ? cs[M.aN + k] * cs[M.cd + k] : 0.0;
        }
    }
    __syncthreads();
    const int last = a.nlev - 1;
    // ---- down ----
    for (int l = 0; l < last; ++l) {
        const CSm F = S[l], C = S[l + 1];
        const Wts &W = a.lv[l].w;
        const int n = F.n, sf = F.st, sc = C.st;
        if (l == 0) CTP(3);
        cgs_sweep(F, rho);                                             // pre-smoothing from zero
        if (l == 0) CTP(4);
        {
            const double *e = cs + F.e, *b = cs + F.b;
            for (int k = threadIdx.x; k < n * n; k += blockDim.x) {    // S-scaled residual
                const int j = k / n + 1, i = k % n + 1;
                const int s = j * sf + i;
                const double ec = e[s];
                const double Ae = cs[F.aW + i] * (ec - e[s - 1]) + cs[F.aE + s] * (ec - e[s + 1]) +
                                  cs[F.aS + j] * (ec - e[s - sf]) + cs[F.aN + s] * (ec - e[s + sf]) + cs[F.rr + s] * ec;
                rho[s] = (cs[F.hb + i] * cs[F.kb + j]) * (b[s] - Ae);
            }
        }
        __syncthreads();
        const int nc = C.n;
        for (int k = threadIdx.x; k < nc * nc; k += blockDim.x) {      // b_c = S_c^-1 P^T (S rho)
            const int J = k / nc + 1, I = k % nc + 1;
            double acc = 0.0;
#pragma unroll
            for (int bb = -1; bb <= 1; ++bb) {
                const int j = 2 * J + bb;
                if (j < 1 || j > n) continue;
                const double *r = rho + j * sf + 2 * I;
                double rs = r[0];
                const bool u = W.uni;
                if (2 * I - 1 >= 1) rs = (u ? 0.5 : __ldg(W.xr + 2 * I - 1)) * r[-1] + rs;   // P^T: I is 2I-1's right parent
                if (2 * I + 1 <= n) rs = rs + (u ? 0.5 : __ldg(W.xl + 2 * I + 1)) * r[1];    //      and 2I+1's left parent
                acc += (bb == 0 ? 1.0 : (u ? 0.5 : (bb < 0 ? __ldg(W.yr + j) : __ldg(W.yl + j)))) * rs;
            }
            cs[C.b + J * sc + I] = acc / (cs[C.hb + I] * cs[C.kb + J]);
        }
        __syncthreads();
    }
    CTP(5);
    // ---- coarsest: four sweeps from zero ----
    for (int s4 = 0; s4 < 4; ++s4) cgs_sweep(S[last], rho);
    CTP(6);
    // ---- up ----
    for (int l = last - 1; l >= 0; --l) {
        const CSm F = S[l];
        const int n = F.n, sf = F.st, sc = S[l + 1].st;
        const double *ec = cs + S[l + 1].e;
        double *e = cs + F.e;
        const Wts &W = a.lv[l].w;
        for (int k = threadIdx.x; k < n * n; k += blockDim.x) {        // e += P e_c
            const int j = k / n + 1, i = k % n + 1;
            e[j * sf + i] += W.uni ? interp_w<true>(ec, sc, i, j, W) : interp_w<false>(ec, sc, i, j, W);
        }
        __syncthreads();
        if (l == 0) CTP(7);
        cgs_sweep(F, rho);                                             // post-smoothing
        if (l == 0) CTP(8);
    }
    {   // result of level lc
        const int n = S[0].n;
        for (int k = threadIdx.x; k < n * n; k += blockDim.x) {
            const int j = k / n + 1, i = k % n + 1;
            a.out[(long)j * a.opitch + i] = cs[S[0].e + j * S[0].st + i];
        }
    }
#ifdef SPP_COARSE_PROF
    CTP(9);
    if (threadIdx.x == 0 && atomicAdd(&g_coarse_prof, 1) < 4)
        printf("[coarse] n0=%d nlev=%d zero %lld stage %lld pre0 %lld down-rest %lld coarsest %lld up-rest %lld post0 %lld out %lld total %lld\n",
               a.lv[0].n, a.nlev, tp[1] - tp[0], tp[2] - tp[1], tp[4] - tp[3], tp[5] - tp[4], tp[6] - tp[5], tp[7] - tp[6],
               tp[8] - tp[7], tp[9] - tp[8], tp[9] - tp[0]);
#endif
}

static size_t coarse_smem(const Ctx *c, int lc)
{
    size_t tot = 0;
    for (int l = lc; l < c->L; ++l) {
        const size_t st = (size_t)c->lev[l].n + 2;
        tot += 8 * st * st + 4 * st;
    }
    tot += (size_t)(c->lev[lc].n + 2) * (c->lev[lc].n + 2);
    return tot * sizeof(double);
}

// V-cycle of levels lc..L-1 in one launch; result in lev[lc].q.  Returns false when the levels
// do not fit (the caller then recurses level by level).
bool launch_coarse_vcycle(Ctx *c, int lc, const double *R, bool rs)
{
    if (c->L - lc > 8 || c->lev[lc].n > std::min(c->tune.coarse_max, kCoarseMaxN)) return false;
    const size_t sm = coarse_smem(c, lc);
    if (sm > 200 * 1024) return false;
    CoarseArgs a{};
    a.nlev = c->L - lc;
    for (int l = lc; l < c->L; ++l) {
        const Level &L = c->lev[l];
        a.lv[l - lc] = CoarseLev{L.n, (int)L.cpitch, L.aE, L.aN, L.rr, L.cd, L.aW, L.aS, L.hb, L.kb, L.w};
    }
    a.R = R; a.rpitch = c->lev[lc].pitch; a.rs = rs ? 1 : 0;
    a.out = c->lev[lc].q; a.opitch = c->lev[lc].pitch;
    double nn = 0;
    for (int l = lc; l < c->L; ++l) nn += (double)c->lev[l].n * c->lev[l].n;
    ProfScope ps(c, 10, nn * 96.0);   // b read; aE, aN, 1/D, r read by two sweeps + residual; e written
    k_coarse_vcycle<<<1, 256, sm, c->st>>>(a);
    c->launches++;
    return true;
}

// ------------------------------------------------------------------------------------------
// Residual + restriction:  rho = R - A_l e  on the fine level, then
//   b_c(I,J) = S_c^{-1} sum_{a,b in {-1,0,1}} w_a w_b S_f rho(2I+a, 2J+b),  w_0 = 1, w_{+-1} = 1/2,
// S = diag(hbar_i kbar_j).  One CTA per RT x RT coarse tile: the S-scaled residual of the
// (2RT+1)^2 fine nodes it needs is formed once into shared memory, then gathered.  rho is never
// written to HBM.
// (The V-cycle itself restricts the residual of its pre-smoothing through k_restrict_low below.)
// ------------------------------------------------------------------------------------------
template <int RT, bool UNI>
__global__ void __launch_bounds__(256, 7) k_resid_restrict(int nf, long pv, long pc, const double *__restrict__ e,
    const double *__restrict__ R, const double *__restrict__ aE, const double *__restrict__ aN,
    const double *__restrict__ rr, const double *__restrict__ aW, const double *__restrict__ aS,
    const double *__restrict__ hbf, const double *__restrict__ kbf, int nc, long pvc,
    const double *__restrict__ hbc, const double *__restrict__ kbc, double *bc,
    const double *__restrict__ cdc, long pcc, int rs_in, int scale_out, int jc0, int jc1, Wts W)
{
    constexpr int RFW = 2 * RT + 1;
    __shared__ double s[RFW * RFW];
    // coarse rows jc0 .. jc1 (a row strip's rows of level l+1; 1 .. nc on one GPU)
    const int I0 = (int)blockIdx.x * RT + 1, J0 = (int)blockIdx.y * RT + jc0;
    const int fi0 = 2 * I0 - 1, fj0 = 2 * J0 - 1;
#pragma unroll 4
    for (int p = threadIdx.x; p < RFW * RFW; p += blockDim.x) {
        const int di = p % RFW, dj = p / RFW;
        const int i = fi0 + di, j = fj0 + dj;
        double v = 0.0;
        if (i <= nf && j <= nf) {
            const long g = (long)j * pv + i, q = (long)j * pc + i;
            const double ec = e[g];
            const double vW = aW[i], vE = aE[q], vS = aS[j], vN = aN[q], vr = rr[q];
            const double Ae = vW * (ec - e[g - 1]) + vE * (ec - e[g + 1]) + vS * (ec - e[g - pv]) +
                              vN * (ec - e[g + pv]) + vr * ec;
            const double Rv = rs_in ? R[g] * (((vW + vE) + (vS + vN)) + vr) : R[g];   // R stored as R/D (z-form)
            v = (hbf[i] * kbf[j]) * (Rv - Ae);
        }
        s[p] = v;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < RT * RT; p += blockDim.x) {
        const int I = I0 + p % RT, J = J0 + p / RT;
        if (I > nc || J > jc1) continue;
        const int li = 2 * (I - I0) + 1, lj = 2 * (J - J0) + 1;
        double acc = 0.0;
        // P^T with the fine level's geometric weights (R21): coarse I is the right parent of fine
        // 2I-1 and the left parent of 2I+1 (1/2 each on a Shishkin corner)
        const double wl = UNI ? 0.5 : __ldg(W.xr + 2 * I - 1), wr = UNI ? 0.5 : __ldg(W.xl + 2 * I + 1);
        const double wd = UNI ? 0.5 : __ldg(W.yr + 2 * J - 1), wu = UNI ? 0.5 : __ldg(W.yl + 2 * J + 1);
#pragma unroll
        for (int bb = -1; bb <= 1; ++bb) {
            const double *srow = s + (lj + bb) * RFW + li;
            const double rs = (wl * srow[-1] + srow[0]) + wr * srow[1];
            acc += (bb == 0 ? 1.0 : (bb < 0 ? wd : wu)) * rs;
        }
        const double bv = acc / (hbc[I] * kbc[J]);
        bc[(long)J * pvc + I] = scale_out ? bv * cdc[(long)J * pcc + I] : bv;   // z-form: stored as b_c / D_c
    }
}

// The V-cycle's restriction of the residual of its pre-smoothing.  e is the sweep from zero on R
// (P:1205-1209), so D e = R + aE e_E + aN e_N and the residual is exactly its lower part,
//   rho = R - A_l e = aW e(i-1,j) + aS e(i,j-1)
// (the identity holds in exact arithmetic; computed this way it has no cancellation): the kernel
// reads e alone, 8 B per fine node instead of 40 (R, e, aE, aN, r).  One thread per
// coarse node: the 4 x 4 block of e it needs (fine rows 2J-2 .. 2J+1, columns 2I-2 .. 2I+1) by
// eight 16-byte loads -- neighbouring threads read neighbouring 32 bytes -- instead of a shared-
// memory tile of 33 x 33 fine residuals per 16 x 16 coarse nodes with a barrier between.  The
// arithmetic is the tile kernel's, expression for expression.
template <bool UNI>
__global__ void __launch_bounds__(256) k_restrict_low(int nf, long pv, const double *__restrict__ e,
    const double *__restrict__ aW, const double *__restrict__ aS, const double *__restrict__ hbf,
    const double *__restrict__ kbf, int nc, long pvc, const double *__restrict__ hbc, const double *__restrict__ kbc,
    double *bc, const double *__restrict__ cdc, long pcc, int scale_out, int jc0, Wts W)
{
    const int I = (int)(blockIdx.x * blockDim.x + threadIdx.x) + 1, J = (int)blockIdx.y + jc0;
    if (I > nc) return;
    const int i0 = 2 * I - 2;
    double ev[4][4];                                   // e(i0 + c, 2J - 2 + r)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const double *p = e + (long)(2 * J - 2 + r) * pv + i0;
        const double2 a = *reinterpret_cast<const double2 *>(p), b = *reinterpret_cast<const double2 *>(p + 2);
        ev[r][0] = a.x; ev[r][1] = a.y; ev[r][2] = b.x; ev[r][3] = b.y;
    }
    double sres[3][3];                                 // S-scaled residual at fine (i0+1+di, 2J-1+dj)
#pragma unroll
    for (int dj = 0; dj < 3; ++dj)
#pragma unroll
        for (int di = 0; di < 3; ++di) {
            const int i = i0 + 1 + di, j = 2 * J - 1 + dj;
            sres[dj][di] = (i <= nf && j <= nf) ? (hbf[i] * kbf[j]) * (aW[i] * ev[dj + 1][di] + aS[j] * ev[dj][di + 1]) : 0.0;
        }
    const double wl = UNI ? 0.5 : __ldg(W.xr + 2 * I - 1), wr = UNI ? 0.5 : __ldg(W.xl + 2 * I + 1);
    const double wd = UNI ? 0.5 : __ldg(W.yr + 2 * J - 1), wu = UNI ? 0.5 : __ldg(W.yl + 2 * J + 1);
    double acc = 0.0;
#pragma unroll
    for (int bb = -1; bb <= 1; ++bb) {
        const double *srow = sres[bb + 1];
        const double rs = (wl * srow[0] + srow[1]) + wr * srow[2];
        acc += (bb == 0 ? 1.0 : (bb < 0 ? wd : wu)) * rs;
    }
    const double bv = acc / (hbc[I] * kbc[J]);
    bc[(long)J * pvc + I] = scale_out ? bv * cdc[(long)J * pcc + I] : bv;   // z-form: stored as b_c / D_c
}

// R == nullptr: e is the pre-smoothing sweep from zero (k_restrict_low); R is not read
void launch_resid_restrict(Ctx *c, int l, const double *R, const double *e, bool rs_in, bool scale_out)
{
    Level &F = c->lev[l], &C = c->lev[l + 1];
    const bool low = R == nullptr;
    ProfScope ps(c, 4, (double)F.n * F.n * (low ? 8.0 : 40.0) + 8.0 * C.n * (double)C.n);
    // coarse tile edge: enough CTAs to fill the GPU on the small levels, and several waves of
    // CTAs on the large ones (one wave plus a small remainder leaves most SMs idle in the tail)
    const int RTn = C.n >= 128 ? 16 : 8;
    // coarse rows: this rank's strip of level l+1 when level l runs on strips
    const int jc0 = F.sdist ? C.slo : 1, jc1 = F.sdist ? C.shi : C.n;
    if (low) {                                          // thread per coarse node, rows jc0 .. jc1
        const int t = std::min(256, (C.n + 31) / 32 * 32);
        const dim3 g2((C.n + t - 1) / t, jc1 - jc0 + 1);
        auto kr = F.w.uni ? k_restrict_low<true> : k_restrict_low<false>;
        kr<<<g2, t, 0, c->st>>>(F.n, F.pitch, e, F.aW, F.aS, F.hb, F.kb, C.n, C.pitch, C.hb, C.kb, C.b, C.cd, C.cpitch,
                                scale_out ? 1 : 0, jc0, F.w);
        c->launches++;
        return;
    }
    const dim3 grid((C.n + RTn - 1) / RTn, (jc1 - jc0 + RTn) / RTn);
#define SPP_RR(T) (F.w.uni ? k_resid_restrict<T, true> : k_resid_restrict<T, false>)<<<grid, T >= 32 ? 256 : (T >= 16 ? 256 : 128), 0, c->st>>>(F.n, F.pitch, \
        F.cpitch, e, R, F.aE, F.aN, F.rr, F.aW, F.aS, F.hb, F.kb, C.n, C.pitch, C.hb, C.kb, C.b, C.cd, C.cpitch, \
        rs_in ? 1 : 0, scale_out ? 1 : 0, jc0, jc1, F.w)
    if (RTn == 32) SPP_RR(32);
    else if (RTn == 16) SPP_RR(16);
    else SPP_RR(8);
#undef SPP_RR
    c->launches++;
}

// ------------------------------------------------------------------------------------------
// Outer corner iteration update: z_new = z + e (z == nullptr: z = 0),
// rho = b_C - A_CC z_new (difference form), partial ||S_0 rho||_2^2 per block (fixed grid of
// kRedBlocks blocks; the host sums the partials in a fixed order).  z_new is a different buffer
// from z (neighbour reads of z).
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kRedThreads) k_cycle_update(int nl, long pv, long pc, const double *__restrict__ z,
    const double *__restrict__ e, double *znew, const double *__restrict__ b, const double *__restrict__ aE,
    const double *__restrict__ aN, const double *__restrict__ rr, const double *__restrict__ aW,
    const double *__restrict__ aS, const double *__restrict__ hb, const double *__restrict__ kb, double *rho,
    double *part, const MGState *ms, const double *__restrict__ cd, int scale_rho, int jz0, int jz1, int j0, int j1)
{
    __shared__ double sm[32];
    if (ms) { z = ms->zcur; znew = ms->znext; }        // corner graph: buffers from the device state
    double acc = 0.0;
    // z' = z + e on rows jz0 .. jz1; rho and the norm on the owned rows j0 .. j1 (a row strip
    // also carries z' on its one-row halos; everything 1 .. nl on one GPU).
    // One block-iteration = one row segment of 2*blockDim columns starting at the ghost column 0,
    // each thread a column pair (i0, i0+1), i0 even, with 16-byte loads and stores (the pitches
    // are multiples of 16 doubles).  Ghost columns (0, nl+1) are written as the zeros they are.
    auto ld2 = [](const double *p) { return *reinterpret_cast<const double2 *>(p); };
    const int segw = 2 * blockDim.x;
    const int nseg = (nl + 2 + segw - 1) / segw;       // columns 0 .. nl+1
    const long nit = (long)(jz1 - jz0 + 1) * nseg;
    for (long it = blockIdx.x; it < nit; it += gridDim.x) {
        const int j = (int)(it / nseg) + jz0;
        const int i0 = (int)(it % nseg) * segw + 2 * threadIdx.x;
        if (i0 > nl) continue;
        const long g = (long)j * pv + i0, q = (long)j * pc + i0;
        const bool ok0 = i0 >= 1, ok1 = i0 + 1 <= nl;  // valid columns of the pair
        double2 c = ld2(e + g);
        if (z) { const double2 t = ld2(z + g); c.x += t.x; c.y += t.y; }
        *reinterpret_cast<double2 *>(znew + g) = c;
        if (j < j0 || j > j1) continue;
        double2 s = ld2(e + g - pv), n = ld2(e + g + pv);
        double w = e[g - 1], ea = e[g + 2];
        if (z) {
            const double2 zs = ld2(z + g - pv), zn = ld2(z + g + pv);
            s.x += zs.x; s.y += zs.y; n.x += zn.x; n.y += zn.y;
            w += z[g - 1]; ea += z[g + 2];
        }
        const double2 vE = ld2(aE + q), vN = ld2(aN + q), vr = ld2(rr + q), vb = ld2(b + g);
        const double2 vW = ld2(aW + i0);
        const double vS = aS[j];
        const double Az0 = vW.x * (c.x - w) + vE.x * (c.x - c.y) + vS * (c.x - s.x) + vN.x * (c.x - n.x) + vr.x * c.x;
        const double Az1 = vW.y * (c.y - c.x) + vE.y * (c.y - ea) + vS * (c.y - s.y) + vN.y * (c.y - n.y) + vr.y * c.y;
        const double r0 = ok0 ? vb.x - Az0 : 0.0, r1 = ok1 ? vb.y - Az1 : 0.0;
        double2 out = make_double2(r0, r1);
        if (scale_rho) { const double2 vd = ld2(cd + q); out.x *= vd.x; out.y *= vd.y; }   // rho/D in z-form
        *reinterpret_cast<double2 *>(rho + g) = out;
        const double2 vh = ld2(hb + i0);
        const double kj = kb[j];
        const double t0 = (vh.x * kj) * r0, t1 = (vh.y * kj) * r1;
        acc += t0 * t0;
        acc += t1 * t1;
    }
    double v = acc;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
    if (lane == 0) sm[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s2 = 0.0;
        for (int k = 0; k < nwp; ++k) s2 += sm[k];
        part[blockIdx.x] = s2;
    }
    zero_tail(part);
}

void launch_cycle_update(Ctx *c, const double *z, const double *e, double *znew, const double *b, double *rho,
                         double *part, const MGState *ms)
{
    Level &L = c->lev[0];
    const double nn = (double)L.n * L.n;
    ProfScope ps(c, 6, nn * ((z ? 64.0 : 56.0) + (c->mg_zform ? 8.0 : 0.0)));
    // a row strip updates z on its one-row halos too (their e came from the neighbours)
    const int j0 = L.sdist ? L.slo : 1, j1 = L.sdist ? L.shi : L.n;
    const int jz0 = std::max(1, j0 - (L.sdist ? 1 : 0)), jz1 = std::min(L.n, j1 + (L.sdist ? 1 : 0));
    int nb = 0, nt = 0;
    seg_shape(L.n, jz1 - jz0 + 1, &nb, &nt);
    k_cycle_update<<<nb, nt, 0, c->st>>>(L.n, L.pitch, L.cpitch, z, e, znew, b,
                                                          L.aE, L.aN, L.rr, L.aW, L.aS, L.hb, L.kb, rho, part, ms, L.cd,
                                                          c->mg_zform ? 1 : 0, jz0, jz1, j0, j1);
    c->launches++;
}

// ------------------------------------------------------------------------------------------
// Setup: the contraction factors of the downstream recurrence z = q/D + ca z_E + cn z_N (z-form,
// ca = aE/D, cn = aN/D) over level l, couplings to the block boundary (i = nl East, j = nl North;
// they multiply a zero inflow) excluded.  Three partial maxima per block:
//   rho     = max (ca + cn)                 (y-form bound)
//   gamma_y = max cn / (1 - ca)             (row decay of a north-boundary error)
//   gamma_x = max ca / (1 - cn)             (column decay of an east-boundary error)
// gamma_y: with M_j = max_i |e(i,j)| of an error e = ca e_E + cn e_N that vanishes on the east
// edge, the node attaining M_j gives M_j <= ca M_j + cn M_{j+1}, so M_j <= gamma_y M_{j+1};
// gamma_x likewise per column.  Both are <= rho (cn/(1-ca) <= ca + cn iff ca (1 - ca - cn) >= 0).
__global__ void k_level_rho(int nl, long pc, const double *aE, const double *aN, const double *cd, double *part,
                            double *partgy, double *partgx)
{
    __shared__ double sm[3][32];
    double mx = 0.0, gy = 0.0, gx = 0.0;
    const long tot = (long)nl * nl;
    for (GridWalk gw(tot, nl, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        const long q = (long)j * pc + i;
        const double ca = (i < nl ? aE[q] : 0.0) * cd[q], cn = (j < nl ? aN[q] : 0.0) * cd[q];
        mx = fmax(mx, ca + cn);
        gy = fmax(gy, cn / (1.0 - ca));
        gx = fmax(gx, ca / (1.0 - cn));
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        gy = fmax(gy, __shfl_xor_sync(0xffffffffu, gy, d));
        gx = fmax(gx, __shfl_xor_sync(0xffffffffu, gx, d));
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nwp = blockDim.x >> 5;
    if (lane == 0) { sm[0][wid] = mx; sm[1][wid] = gy; sm[2][wid] = gx; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, c2 = 0.0;
        for (int k = 0; k < nwp; ++k) { a = fmax(a, sm[0][k]); b = fmax(b, sm[1][k]); c2 = fmax(c2, sm[2][k]); }
        part[blockIdx.x] = a; partgy[blockIdx.x] = b; partgx[blockIdx.x] = c2;
    }
    zero_tail(part);
    zero_tail(partgy);
    zero_tail(partgx);
}

// ya = aE / D_E = aE(i,j) cd(i+1,j), yn = aN / D_N = aN(i,j) cd(i,j+1) on [1, nl]^2 (the ghost
// ring of cd is zero, so the couplings to the block boundary vanish).
__global__ void k_ycoef(int nl, long pc, const double *aE, const double *aN, const double *cd, double *ya, double *yn)
{
    const long tot = (long)nl * nl;
    for (GridWalk gw(tot, nl, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        const long q = (long)j * pc + i;
        ya[q] = aE[q] * cd[q + 1];
        yn[q] = aN[q] * cd[q + pc];
    }
}

void launch_ycoef(Ctx *c, int nl, long pc, const double *aE, const double *aN, const double *cd, double *ya, double *yn)
{
    k_ycoef<<<gblocks((long)nl * nl), 256, 0, c->st>>>(nl, pc, aE, aN, cd, ya, yn);
    c->launches++;
}

// The global grid's y-form couplings, formed on first use when the setup skipped them (the
// Jacobi-mode z-form solve never reads them).  Bit for bit k_coef_2d's: aE (1/D_E) with 1/D_E
// from the same formula, and the zero ghost ring of cd at the block edges.
void ensure_y0(Ctx *c)
{
    if (c->y0_ok) return;
    launch_ycoef(c, c->N - 1, c->P, c->aE, c->aN, c->cd, c->ya, c->yn);
    c->y0_ok = 1;
}

// Tile plan of a sweep over `rows` output rows x n columns of a level with certified halo
// `halo`.  whole: the block is the whole level (no rows above it);
// otherwise it is a row strip of a distributed solve whose top tile recomputes `halo` rows of the
// strip above.  A tile's sweep takes about (chunks + 5 (W - 1)) chunk-times: each of its W warps
// starts 5 chunks after the one above (62-column lane skew + one chunk of granularity), and a warp
// sweeps (tile columns + halo + 62) / 16 chunks.  Picks the warps per tile (3..Wt; the halo rows
// are part of the tile) and the column tiling with the smallest such time among the plans that
// run as one wave of one CTA per SM.  Returns false when no plan exists.
bool plan_tiles(const Ctx *c, int n, int rows, int halo, int halox, bool whole, Level &L)
{
    const Tune &T = c->tune;
    const int Wt = std::max(1, std::min(T.gs_warps, c->mg_zform ? WMAXW : 4));   // 5 warps only fit in z-form
    const int lag = T.gs_lag;
    auto cost = [lag](int W, int cols) { return (cols + WLAG * 31 + WCW - 1) / WCW + lag * (W - 1); };
    int bestW = 0, bestRows = 0, bestCols = 0, bestT = 1 << 30, bestN = 1 << 30;
    if (whole && n <= 32 * Wt) {                               // candidate: one exact CTA
        bestW = (n + 31) / 32; bestRows = n; bestCols = n; bestT = cost(bestW, n); bestN = 1;
    }
    for (int W = std::min(2, Wt); W <= Wt; ++W) {
        const int rows_out = 32 * W - halo;
        if (rows_out < 16 || (whole && rows_out >= n)) continue;
        const int nrt = (rows + rows_out - 1) / rows_out;
        if (nrt > c->sm_count) continue;
        const int maxct = std::max(1, std::min(c->sm_count / nrt, n / 64));
        for (int nct = 1; nct <= maxct; ++nct) {
            int tc = (n + nct - 1) / nct;
            tc = (tc + 15) / 16 * 16;
            if (T.gs_tile_cols > 0) tc = std::min(n, T.gs_tile_cols);
            const bool full = tc >= n;
            const int t = cost(W, (full ? n : tc + halox));
            const int ncta = nrt * ((n + tc - 1) / tc);
            if (t < bestT || (t == bestT && ncta < bestN)) {
                bestT = t; bestN = ncta; bestW = W; bestRows = rows_out; bestCols = full ? n : tc;
            }
        }
    }
    if (bestW == 0) return false;
    L.tile_warps = bestW;
    L.tile_rows = bestRows;
    L.tile_cols = bestCols;
    const bool exact1 = whole && bestRows >= n;
    L.halo_y = exact1 ? 0 : halo;
    L.halo_x = bestCols >= n ? 0 : halox;
    if (getenv("SPP_DEBUG_TILES"))
        fprintf(stderr, "[spp] level n=%d rows=%d%s halo=%d,%d: warps %d tile %dx%d (+%d,%d) cost %d chunks, %d CTAs\n",
                n, rows, whole ? "" : " (strip)", halo, halox, L.tile_warps, L.tile_rows, L.tile_cols, L.halo_y, L.halo_x,
                bestT, bestN);
    return true;
}

// Tile plans in two halves around one host synchronisation (batched with the line chains' by
// setup_2d_ctx): the contraction factors of every level and their read-back into c->rho_h, then
// the certified halos and tiles.
cudaError_t setup_mg_tiles_launch(Ctx *c)
{
    const size_t S = (size_t)c->L * kRedBlocks;
    for (int l = 0; l < c->L; ++l) {
        double *p = c->part + (size_t)l * kRedBlocks;
        k_level_rho<<<kRedBlocks, kRedThreads, 0, c->st>>>(c->lev[l].n, c->lev[l].cpitch, c->lev[l].aE,
                                                           c->lev[l].aN, c->lev[l].cd, p, p + S, p + 2 * S);
        c->launches++;
    }
    c->rho_h.assign(3 * S, 0.0);
    SPP_CUDA_TRY(cudaMemcpyAsync(c->rho_h.data(), c->part, sizeof(double) * 3 * S, cudaMemcpyDeviceToHost, c->st));
    return cudaSuccess;
}

cudaError_t setup_mg_tiles_plan(Ctx *c)
{
    const Tune &T = c->tune;
    const int Wt = std::max(1, std::min(T.gs_warps, c->mg_zform ? WMAXW : 4));   // 5 warps only fit in z-form
    const size_t S = (size_t)c->L * kRedBlocks;
    const std::vector<double> &h = c->rho_h;
    for (int l = 0; l < c->L; ++l) {
        Level &L = c->lev[l];
        double rho = 0.0, gy = 0.0, gx = 0.0;
        for (int k = 0; k < kRedBlocks; ++k) {
            rho = std::fmax(rho, h[(size_t)l * kRedBlocks + k]);
            gy = std::fmax(gy, h[S + (size_t)l * kRedBlocks + k]);
            gx = std::fmax(gx, h[2 * S + (size_t)l * kRedBlocks + k]);
        }
        L.contraction = rho;
        // certified halos: the truncation error of a tile whose rows
        // above / columns right of its output are recomputed from zero inflow is <= (g_y^hy +
        // g_x^hx) max|z|; hy, hx = smallest multiples of 8 with each term <= 0.5e-17.  In y-form
        // (y = D z, other couplings) the rho bound rho^h <= 1e-17 is used for both.
        auto depth = [&](double g, double target) {
            if (!(g < 1.0)) return -1;
            if (g <= 0.0) return 8;
            for (int d = 8; d <= T.gs_max_halo; d += 8)
                if (d * std::log(g) <= std::log(target)) return d;
            return -1;
        };
        int hy, hx;
        if (c->mg_zform && !T.rho_halo) { hy = depth(gy, 0.5e-17); hx = depth(gx, 0.5e-17); }
        else hy = hx = depth(rho, 1e-17);
        const int halo = (hy < 0 || hx < 0) ? -1 : hy;
        L.halo_cert = halo;
        L.halo_certx = halo < 0 ? -1 : hx;
        const int n = L.n;
        if (halo < 0 || halo + 16 > 32 * Wt) {
            if (n <= 32 * Wt) {                                // one CTA, exact
                L.tile_warps = (n + 31) / 32;
                L.tile_rows = n; L.tile_cols = n; L.halo_x = 0; L.halo_y = 0;
            } else L.tile_warps = 0;                           // no certified halo: exact chain
            continue;
        }
        if (!plan_tiles(c, n, n, hy, hx, true, L)) L.tile_warps = 0;   // no tiling: exact chain
    }
    return cudaSuccess;
}

cudaError_t setup_mg_tiles(Ctx *c)
{
    SPP_CUDA_TRY(setup_mg_tiles_launch(c));
    SPP_CUDA_TRY(cudaStreamSynchronize(c->st));
    return setup_mg_tiles_plan(c);
}

}  // namespace spp
