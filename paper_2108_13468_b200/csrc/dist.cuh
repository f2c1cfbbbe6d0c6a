// dist.cuh -- row-strip decomposition of the 2D solve over P ranks.
//
// Rank r owns the interior rows [J[r], J[r+1]) of every global grid function (the strip
// boundary J[Pb] = n+1 splits the bottom half C u Y from the top half X u I), and the rows
// [Cb[r], Cb[r+1]) of the corner block for the corner multigrid, whose first D levels run as
// row strips on every rank (levels >= D run whole on every rank after one all-gather).  Every
// array keeps the single-GPU layout (a strip's rows, and its halos, sit at their global
// positions), so the single-GPU kernels run on a strip through their row-range arguments.
//
// The exchange steps are lists of Xfer blocks, generated from the geometry alone (identical on
// every rank) and executed either by a loopback transport (P strips on one device: cudaMemcpy2D
// between the strips' buffers) or by NCCL (grouped ncclSend / ncclRecv on the context's stream).
#pragma once
#include <vector>

#include "spp_internal.cuh"

namespace spp {

enum Role : int {
    R_V = 0, R_Z, R_U, R_W, R_CHAIN, R_LB, R_LE, R_LQ, R_LG, R_LRHO, R_BC, R_ZC, R_ZC2, R_PART, R_CBUF, R_F,
    R_NROLES
};

// A block of `rows` rows x `width` elements with row stride `pitch` (the same on both sides),
// from rank src's buffer (role, slot) at element offset soff to rank dst's at doff.
struct Xfer {
    int src, dst, role, slot;
    long soff, doff, width, rows, pitch;
};

// Geometry of a distributed solve: identical on every rank.
struct Geom {
    int N = 0, n = 0, m = 0, P = 1, Pb = 0, D = 0, L = 0;
    long pitch = 0;                       // global grid pitch
    std::vector<int> J;                   // rank r owns global interior rows [J[r], J[r+1])
    std::vector<int> Cb;                  // rank r owns corner (level-0) rows [Cb[r], Cb[r+1])
    std::vector<int> nl;                  // unknowns per axis of each corner level
    std::vector<long> lpitch;             // value pitch of each corner level
    std::vector<int> halo;                // certified halo of each strip level (l < D)
    std::vector<int> xstart;              // top rank: first line of its X warm-up (-1: none)
    std::vector<int> ylo, yhi, ystart;    // bottom rank: owned Y lines and warm-up start (yhi < ylo: none)
    std::vector<int> ncta;                // top rank: CTA strips of its M_II chain
    long chain_ld = 0;
    int ext_slot = 0, mii_cols = 0;
    bool top(int r) const { return r >= Pb; }
    int lrow0(int l, int r) const { return r == 0 ? 1 : (Cb[r] >> l); }        // first row at level l
    int lrow1(int l, int r) const { return r == P - 1 ? nl[l] + 1 : (Cb[r + 1] >> l); }   // one past the last
    int shalo(int l, int r) const { return std::max(0, std::min(halo[l], nl[l] + 1 - lrow1(l, r))); }
};

// schedule generators (dist.cu); every function appends the blocks of one exchange step
void xf_vec_halo(const Geom &g, std::vector<Xfer> &v, int role, int slot);
void xf_mii(const Geom &g, std::vector<Xfer> &v, int t, int zslot);
void xf_xhalo(const Geom &g, std::vector<Xfer> &v, int vslot, int zslot);
void xf_yin(const Geom &g, std::vector<Xfer> &v, int vslot, int zslot);
void xf_yout(const Geom &g, std::vector<Xfer> &v, int zslot);
void xf_rown1(const Geom &g, std::vector<Xfer> &v, int zslot);
void xf_partials(const Geom &g, std::vector<Xfer> &v, int slot, int count);
void xf_corner_in(const Geom &g, std::vector<Xfer> &v);
void xf_corner_out(const Geom &g, std::vector<Xfer> &v, int zrole);
void xf_mg_rhs(const Geom &g, std::vector<Xfer> &v, int l, int role, int slot);
void xf_mg_e(const Geom &g, std::vector<Xfer> &v, int l);
void xf_mg_pm1(const Geom &g, std::vector<Xfer> &v, int l, int role, int slot);
void xf_mg_g(const Geom &g, std::vector<Xfer> &v, int l);
void xf_mg_gather(const Geom &g, std::vector<Xfer> &v, int l, int role, int slot);

struct Dist {
    Geom g;
    int me = -1;                          // NCCL: this process's rank; loopback: -1 (every strip local)
    std::vector<Ctx *> cx;                // loopback: every strip's context; NCCL: {this rank's}
    void *comm = nullptr;                 // ncclComm_t (NCCL mode)
    cudaStream_t st = nullptr;
    double *stage = nullptr; size_t stage_cap = 0;   // NCCL pack / unpack staging
    int64_t nxfer = 0; double xbytes = 0; int64_t nexch = 0;   // statistics
    Ctx *ctx_of(int r) const { return me < 0 ? cx[r] : (r == me ? cx[0] : nullptr); }
};

spp_status exchange_rows(Dist *d, const std::vector<Xfer> &xs);
spp_status solve_dist(Ctx *c, const double *f, double *u, spp_mem mem, double *hist, int hcap, spp_stats *st);
spp_status setup_dist(Ctx *c, const double *c1, const double *c2, const double *r, spp_mem mem);
void destroy_dist(Ctx *c);

}  // namespace spp
