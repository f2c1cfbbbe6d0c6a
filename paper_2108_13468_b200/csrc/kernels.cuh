// kernels.cuh -- declarations of the kernels shared between translation units.
#pragma once
#include "spp_internal.cuh"

namespace spp {

__global__ void k_coef_1d(int N, double eps, const double *wx, const double *wy, double *aW, double *aS);
__global__ void __launch_bounds__(256, 6) k_coef_2d(int N, long P, double eps, const double *wx, const double *wy,
                          const double *c1, const double *c2, const double *r, const double *aW,
                          const double *aS, double *aE, double *aN, double *rr, double *ca,
                          double *cn, double *cd, double *ya, double *yn, int want_y, int *bad);
__global__ void k_coef_level(int N, int nl, int step, long Pl, double eps, const double *lwx, const double *lwy,
                             const double *c1, const double *c2,
                             const double *r, double *aW, double *aS, double *hb, double *kb,
                             double *aE, double *aN, double *rr, double *ca, double *cn, double *cd);
__global__ void k_level0_1d(int N, const double *wx, const double *wy, const double *aW,
                            const double *aS, double *lW, double *lS, double *hb, double *kb);
__global__ void k_pack(int m, long P, const double *src, double *dst, int j0, int nrows);
__global__ void k_unpack(int m, long P, const double *src, double *dst, int j0, int nrows);
__global__ void k_spmv(int m, long P, const double *z, const double *aE, const double *aN,
                       const double *rr, const double *aW, const double *aS, int weighted, double *w,
                       const double *v0, double *part, int j0, int nrows);
__global__ void k_resid_stats(int m, long P, const double *f, const double *Au, const double *aE,
                              const double *aN, const double *rr, const double *aW, const double *aS,
                              double *part4, long pstride, int j0, int nrows);
__global__ void k_rhs(int m, long P, const double *f, const double *aE, const double *aN,
                      const double *rr, const double *aW, const double *aS, int weighted,
                      double *out, double *part, int j0, int nrows, const double *Au = nullptr);
__global__ void k_scale(long n2, double *x, double alpha);
__global__ void k_mgs(long n2, double *w, const double *x, const double *part_in, double *hslot,
                      const double *y, double *part_out, int nparts);
__global__ void k_normalize(long n2, const double *w, const double *part_in, double *hslot, double *v, int nparts);
__global__ void k_update_x(long n2, int k, const double *const *Z, const double *y, double *x, int accumulate);
__global__ void k_corner_rhs(int N, long P, long P0, const double *v, const double *z,
                             const double *aE, const double *aN, const double *rr, const double *aW,
                             const double *aS, const double *hb, const double *kb, int weighted,
                             double *bc, double *part, double *bc2, const double *cd, int scale2, int j0, int j1);
__global__ void k_mg_resid(int nl, long Pv, long Pc, double *z, const double *e, const double *b,
                           const double *aE, const double *aN, const double *rr, const double *aW,
                           const double *aS, const double *hb, const double *kb, double *rho,
                           double *part);
__global__ void k_prolong_add(int nl, long Pv, double *e, const double *ec, long Pcv, Wts W);
__global__ void k_corner_out(int n, long P0, const double *zc, long P, double *z, const MGState *ms, int j0, int j1);
__global__ void k_pack_level(int nl, long Pv, const double *src, double *dst);
__global__ void k_unpack_level(int nl, long Pv, const double *src, double *dst);

void launch_lines(Ctx *c, const double *v, double *z);

// 1D solver (k_1d.cu)
spp_status setup_1d(Ctx *c, const double *cc, const double *r, spp_mem mem);
spp_status solve_1d_abi(Ctx *c, const double *f, double *u, spp_mem mem, double *hist, int hcap,
                        spp_stats *st);

// Batched 1D solves: nprob independent problems, one CTA each.
struct Batch1 {
    cudaStream_t st = nullptr;
    spp_options opt{};
    int nprob = 0, maxit = 0;
    std::vector<int> n;                  // N per problem
    std::vector<double> eps, h, H;       // mesh widths per problem (h = tau/(N/2), H = (1-tau)/(N/2))
    std::vector<long long> xo, so;       // offsets of the interior samples / scratch block
    long long total = 0, scratch_len = 0;
    std::vector<int> order;              // problems sorted by launch shape
    std::vector<int> gstart, gcount, gK, gT;
    double *scratch = nullptr;           // per-problem workspace blocks
    double *dpar = nullptr;              // eps, h, H, res0, res (5 * nprob)
    long long *doff = nullptr;           // xo, so (2 * nprob)
    int *dint = nullptr;                 // n, order, iters, conv, bad (5 * nprob)
    double *stage = nullptr;             // host-residency staging: f, u (2 * total)
    int64_t launches = 0;
    float setup_ms = 0.f;
    std::string err;
};
cudaError_t batch1d_alloc(Batch1 *b);
cudaError_t batch1d_setup(Batch1 *b, const double *c, const double *r);   // device c, r
cudaError_t batch1d_solve(Batch1 *b, const double *f, double *u);         // device f, u

}  // namespace spp
