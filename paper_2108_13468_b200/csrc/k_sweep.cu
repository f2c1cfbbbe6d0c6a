// k_sweep.cu -- downstream triangular sweep on a rectangle (sm_100a).
//
//   z(i,j) = s(i,j) q(i,j) + ca(i,j) z(i+1,j) + cn(i,j) z(i,j+1),  j = jhi..jlo, i = ihi..ilo
//
// This one recurrence is (a) the M_II solve of the block preconditioner (P:1041-1056:
// "downstream Gauss-Seidel approximation that sweeps from the upper-right corner of the
// interior region to the bottom-left corner"; q = D v or v, ca = aE/D, cn = aN/D) and (b) the
// E/N-implicit half of one downstream point Gauss-Seidel sweep of the corner multigrid
// (P:1205-1209), whose W/S "old" terms are folded into q by the caller.
//
// Parallel schedule: one lane per row, one warp per 32 rows, the
// warp walks the columns right-to-left with lane t one step behind lane t-1, so the North
// value arrives by __shfl_up_sync from the lane above and the East value is the lane's own
// previous result.  Warps of a CTA are chained through a shared-memory edge ring with
// two-way progress counters.  Rows are loaded by each lane in chunks of CH columns into a
// register double buffer (the loads of chunk c+1 are in flight while chunk c is computed).
//   EXACT mode: CTAs are chained through global progress flags (cooperative launch, so all
//               CTAs are resident): the sweep equals the sequential one.
//   HALO mode:  CTAs are independent; each recomputes `halo` rows above its output rows
//               (and `halo_x` columns to the right of its output columns) from zero inflow.
//               The inflow error decays at least like rho^d, rho = max (ca + cn) < 1 (all
//               coefficients are positive), so the halo is chosen per level with
//               rho^halo < 1e-20.
#include "spp_internal.cuh"

namespace spp {

constexpr int CH = 8;      // columns per chunk
constexpr int EB = 64;     // shared-memory edge ring (columns)
constexpr int WMAX = 16;   // warps per CTA

struct SweepTile {         // column tiling (HALO mode); 0 => whole width
    int cols_out, halo_x;
};

__device__ __forceinline__ int ld_acquire_gpu(const int *p)
{
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int *p, int v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <bool HAS_S>
__device__ __forceinline__ void load_chunk(int s0, int lane, bool rvalid, int ncols, int ihi,
                                           const double *qrow, const double *srow,
                                           const double *arow, const double *nrow,
                                           double (&Q)[CH], double (&S)[CH], double (&A)[CH],
                                           double (&Nn)[CH])
{
#pragma unroll
    for (int k = 0; k < CH; ++k) {
        const int idx = s0 + k - lane;
        const bool ok = rvalid && idx >= 0 && idx < ncols;
        const int col = ihi - idx;
        Q[k] = ok ? __ldg(qrow + col) : 0.0;
        if (HAS_S) S[k] = ok ? __ldg(srow + col) : 0.0;
        A[k] = ok ? __ldg(arow + col) : 0.0;
        Nn[k] = ok ? __ldg(nrow + col) : 0.0;
    }
}

template <bool HAS_S, bool EXACT>
__global__ void __launch_bounds__(WMAX * 32) k_sweep(SweepArgs a, SweepTile tile)
{
    __shared__ double edge[WMAX][EB];
    __shared__ int prod[WMAX], cons[WMAX];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x < WMAX) { prod[threadIdx.x] = 0; cons[threadIdx.x] = 0; }
    __syncthreads();

    // ---- rows of this CTA (blockIdx.x counts row blocks from the top) ----
    const int out_top = a.jhi - (int)blockIdx.x * a.rows_out;
    const int out_bot = max(a.jlo, out_top - a.rows_out + 1);
    const int top = EXACT ? out_top : min(a.jhi, out_top + a.halo);
    // ---- columns of this CTA (blockIdx.y counts column tiles from the right) ----
    int out_right = a.ihi, out_left = a.ilo, right = a.ihi;
    if (!EXACT && tile.cols_out > 0) {
        out_right = a.ihi - (int)blockIdx.y * tile.cols_out;
        out_left = max(a.ilo, out_right - tile.cols_out + 1);
        right = min(a.ihi, out_right + tile.halo_x);
    }
    const int ncols = right - out_left + 1;
    const int wtop = top - w * 32;
    if (wtop < out_bot) return;                       // no rows for this warp
    const int nwa = min(nw, (top - out_bot) / 32 + 1);
    const int row = wtop - lane;
    const bool rvalid = row >= out_bot;
    const bool wrow = rvalid && row <= out_top;       // output row
    const int rr = rvalid ? row : wtop;
    const double *qrow = a.q + (long)rr * a.qp;
    const double *srow = HAS_S ? a.s + (long)rr * a.sp : nullptr;
    const double *arow = a.ca + (long)rr * a.cp;
    const double *nrow = a.cn + (long)rr * a.cp;
    double *zrow = a.z + (long)rr * a.zp;
    const bool chained_in = EXACT && w == 0 && blockIdx.x > 0;
    const bool has_consumer = (w + 1 < nwa);
    const bool publish = EXACT && (w == nwa - 1) && (blockIdx.x + 1 < gridDim.x);
    const int nsteps = ncols + 31;

    double qc[CH], sc[CH], ac[CH], nc[CH], qn[CH], sn[CH], an[CH], nn[CH];
    load_chunk<HAS_S>(0, lane, rvalid, ncols, right, qrow, srow, arow, nrow, qc, sc, ac, nc);
    double zprev = 0.0;

    for (int s0 = 0; s0 < nsteps; s0 += CH) {
        // issue the next chunk's loads early
        load_chunk<HAS_S>(s0 + CH, lane, rvalid, ncols, right, qrow, srow, arow, nrow, qn, sn, an, nn);
        // prefetch further ahead into L2
        {
            const int idx = s0 + 8 * CH - lane;
            if (rvalid && idx >= 0 && idx < ncols && ((idx & 15) < CH)) {
                const int col = right - idx;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(qrow + col));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(arow + col));
                asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + col));
                if (HAS_S) asm volatile("prefetch.global.L2 [%0];" ::"l"(srow + col));
            }
        }
        // ---- North inflow of lane 0 for this chunk ----
        double ein[CH];
#pragma unroll
        for (int k = 0; k < CH; ++k) ein[k] = 0.0;
        const int need = min(ncols, s0 + CH);
        if (w > 0) {
            if (lane == 0) {
                while (*((volatile int *)&prod[w - 1]) < need) { }
                __threadfence_block();
#pragma unroll
                for (int k = 0; k < CH; ++k)
                    ein[k] = *((volatile double *)&edge[w - 1][(s0 + k) & (EB - 1)]);
                __threadfence_block();
                *((volatile int *)&cons[w]) = need;
            }
        } else if (chained_in) {
            if (lane == 0) {
                while (ld_acquire_gpu(a.flags + blockIdx.x - 1) < need) { }
                const double *zab = a.z + (long)(out_top + 1) * a.zp;
#pragma unroll
                for (int k = 0; k < CH; ++k) {
                    const int idx = s0 + k;
                    ein[k] = (idx < ncols) ? __ldcg(zab + right - idx) : 0.0;
                }
            }
        }
        // ---- back-pressure: do not overwrite edge slots the consumer has not read ----
        if (has_consumer && lane == 31) {
            const int lim = s0 + CH - 31 - EB;
            if (lim > 0) {
                while (*((volatile int *)&cons[w + 1]) < lim) { }
            }
        }
        __syncwarp();
        // ---- CH wavefront steps ----
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            const int idx = s0 + k - lane;
            double zN = __shfl_up_sync(0xffffffffu, zprev, 1);
            if (lane == 0) zN = ein[k];
            const double sq = HAS_S ? sc[k] * qc[k] : qc[k];
            double z = fma(nc[k], zN, fma(ac[k], zprev, sq));
            const bool ok = rvalid && idx >= 0 && idx < ncols;
            z = ok ? z : 0.0;
            if (ok && wrow && (right - idx) <= out_right) zrow[right - idx] = z;
            if (lane == 31 && ok && has_consumer) edge[w][idx & (EB - 1)] = z;
            zprev = z;
        }
        // ---- publish lane 31 progress ----
        const int done = min(ncols, max(0, s0 + CH - 31));
        if (lane == 31) {
            if (has_consumer) {
                __threadfence_block();
                *((volatile int *)&prod[w]) = done;
            }
            if (publish) st_release_gpu(a.flags + blockIdx.x, done);
        }
#pragma unroll
        for (int k = 0; k < CH; ++k) {
            qc[k] = qn[k]; ac[k] = an[k]; nc[k] = nn[k];
            if (HAS_S) sc[k] = sn[k];
        }
    }
}

// Launch.  exact: chained CTAs (cooperative launch); otherwise HALO mode with a.halo rows.
void launch_sweep(Ctx *c, const SweepArgs &a0, bool exact, int cls, double bytes)
{
    SweepArgs a = a0;
    const int rows = a.jhi - a.jlo + 1;
    if (rows <= 0 || a.ihi < a.ilo) return;
    ProfScope ps(c, cls, bytes);
    SweepTile tile{0, 0};
    if (exact) {
        // warps per CTA: at most WMAX; CTAs chained through global flags.
        int nwarps = (rows + 31) / 32;
        int wpc = nwarps < WMAX ? nwarps : WMAX;
        a.rows_out = wpc * 32;
        a.halo = 0;
        int nblk = (rows + a.rows_out - 1) / a.rows_out;
        cudaMemsetAsync(a.flags, 0, sizeof(int) * (nblk + 1), c->st);
        dim3 grid(nblk), block(wpc * 32);
        void *args[] = {(void *)&a, (void *)&tile};
        if (a.s)
            cudaLaunchCooperativeKernel((void *)k_sweep<true, true>, grid, block, args, 0, c->st);
        else
            cudaLaunchCooperativeKernel((void *)k_sweep<false, true>, grid, block, args, 0, c->st);
    } else {
        int hw = (a.halo + 31) / 32;
        int ow = a.rows_out / 32;
        if (ow + hw > WMAX) ow = WMAX - hw;
        a.rows_out = ow * 32;
        int nblk = (rows + a.rows_out - 1) / a.rows_out;
        dim3 grid(nblk, 1), block((ow + hw) * 32);
        if (a.s)
            k_sweep<true, false><<<grid, block, 0, c->st>>>(a, tile);
        else
            k_sweep<false, false><<<grid, block, 0, c->st>>>(a, tile);
    }
    c->launches++;
}

}  // namespace spp
