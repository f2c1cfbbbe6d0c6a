// dist.cu -- the 2D solve on row strips over P ranks: the exchange
// schedule (pure functions of the geometry), the two transports (loopback between P strips on
// one device; NCCL grouped send/recv between processes) and the distributed FGMRES iteration,
// block preconditioner (eq:2D blocks) and corner multigrid.
//
// What crosses a strip boundary, per FGMRES iteration (everything else is strip-local):
//   SpMV: one row of z on each side; MGS dots and norms: the
//   per-strip partial sums, all-gathered and summed in one fixed order on every rank;
//   M_II: the exact downstream sweep runs top strip first, each strip's chained
//   sweep taking the bottom row of the strip above as its North inflow;
//   M_XX: the certified warm-up lines of a strip's first chunk come from above;
//   M_YY: the vertical lines cross the bottom strips, so each bottom rank solves a
//   column block of whole lines (its v block gathered from the other bottom strips, the result
//   scattered back);
//   corner: b_C is redistributed to the corner partition, whose strips
//   run the first D levels' smoothing with the certified halo rows of the strip above as their
//   halo, residual/restriction and prolongation with one- and two-row halos, and the levels
//   >= D whole on every rank after one all-gather of their right-hand side.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "dist.cuh"
#include "kernels.cuh"

namespace spp {

// ===================================================================================== schedule
// rows [a, b) x columns [c0, c0+w) of (role, slot), row stride pitch, needed by rank dst: one block
// from every other rank r owning rows [lo[r], hi[r]) of that range
static void need_rows(std::vector<Xfer> &v, int dst, const std::vector<int> &lo, const std::vector<int> &hi, int role,
                      int slot, int a, int b, long pitch, long c0, long w)
{
    for (int r = 0; r < (int)lo.size(); ++r) {
        if (r == dst) continue;
        const int s0 = std::max(a, lo[r]), s1 = std::min(b, hi[r]);
        if (s0 >= s1) continue;
        const long off = (long)s0 * pitch + c0;
        v.push_back({r, dst, role, slot, off, off, w, (long)(s1 - s0), pitch});
    }
}
static void gowners(const Geom &g, std::vector<int> &lo, std::vector<int> &hi)
{
    lo.assign(g.J.begin(), g.J.end() - 1);
    hi.assign(g.J.begin() + 1, g.J.end());
}
static void lowners(const Geom &g, int l, std::vector<int> &lo, std::vector<int> &hi)
{
    lo.resize(g.P); hi.resize(g.P);
    for (int r = 0; r < g.P; ++r) { lo[r] = g.lrow0(l, r); hi[r] = g.lrow1(l, r); }
}

// one row of (role, slot) on each side of every strip (SpMV, true-residual stencil)
void xf_vec_halo(const Geom &g, std::vector<Xfer> &v, int role, int slot)
{
    std::vector<int> lo, hi;
    gowners(g, lo, hi);
    for (int d = 0; d < g.P; ++d) {
        need_rows(v, d, lo, hi, role, slot, g.J[d] - 1, g.J[d], g.pitch, 0, g.pitch);
        need_rows(v, d, lo, hi, role, slot, g.J[d + 1], g.J[d + 1] + 1, g.pitch, 0, g.pitch);
    }
}

// M_II hand-off: top strip t's bottom row (its chain buffer's last slot) -> strip t-1's inflow
void xf_mii(const Geom &g, std::vector<Xfer> &v, int t, int zslot)
{
    (void)zslot;
    if (t <= g.Pb) return;
    v.push_back({t, t - 1, R_CHAIN, 0, (long)(g.ncta[t] - 1) * g.chain_ld, (long)g.ext_slot * g.chain_ld,
                 (long)g.mii_cols, 1, g.chain_ld});
}

// M_XX warm-up of the top strips: v (columns 1..n) and the I neighbour z(n+1, j) of the warm-up
// rows above the strip
void xf_xhalo(const Geom &g, std::vector<Xfer> &v, int vslot, int zslot)
{
    std::vector<int> lo, hi;
    gowners(g, lo, hi);
    for (int t = g.Pb; t < g.P; ++t) {
        if (g.xstart[t] < 0) continue;
        const int a = g.J[t + 1], b = g.N - g.xstart[t];   // line l <-> row N-1-l
        need_rows(v, t, lo, hi, R_V, vslot, a, b, g.pitch, 1, g.n);
        need_rows(v, t, lo, hi, R_Z, zslot, a, b, g.pitch, g.n + 1, 1);
    }
}

// M_YY: bottom rank b solves lines [ylo, yhi] (column i = N-1-l) from ystart: v on every bottom
// row of those columns and the I neighbour z(i, n+1)
void xf_yin(const Geom &g, std::vector<Xfer> &v, int vslot, int zslot)
{
    std::vector<int> lo, hi;
    gowners(g, lo, hi);
    for (int b = 0; b < g.Pb; ++b) {
        if (g.yhi[b] < g.ylo[b]) continue;
        const long c0 = g.N - 1 - g.yhi[b], w = g.yhi[b] - g.ystart[b] + 1;
        need_rows(v, b, lo, hi, R_V, vslot, 1, g.n + 1, g.pitch, c0, w);
        need_rows(v, b, lo, hi, R_Z, zslot, g.n + 1, g.n + 2, g.pitch, c0, w);
    }
}

// M_YY results: owner b's solved columns, every other bottom strip's rows
void xf_yout(const Geom &g, std::vector<Xfer> &v, int zslot)
{
    for (int b = 0; b < g.Pb; ++b) {
        if (g.yhi[b] < g.ylo[b]) continue;
        const long c0 = g.N - 1 - g.yhi[b], w = g.yhi[b] - g.ylo[b] + 1;
        for (int s = 0; s < g.Pb; ++s) {
            if (s == b) continue;
            const long off = (long)g.J[s] * g.pitch + c0;
            v.push_back({b, s, R_Z, zslot, off, off, w, (long)(g.J[s + 1] - g.J[s]), g.pitch});
        }
    }
}

// the X row next to the corner, z(i, n+1) for i <= n: top strip Pb -> bottom strip Pb-1 (corner rhs)
void xf_rown1(const Geom &g, std::vector<Xfer> &v, int zslot)
{
    if (g.Pb < 1 || g.Pb >= g.P) return;
    const long off = (long)(g.n + 1) * g.pitch + 1;
    v.push_back({g.Pb, g.Pb - 1, R_Z, zslot, off, off, (long)g.n, 1, g.pitch});
}

// all-gather of `count` consecutive partial-sum slots: segment r of every slot to every rank
void xf_partials(const Geom &g, std::vector<Xfer> &v, int slot, int count)
{
    const long ps = (long)g.P * kRedBlocks;
    for (int r = 0; r < g.P; ++r)
        for (int s = 0; s < g.P; ++s) {
            if (s == r) continue;
            const long off = slot * ps + (long)r * kRedBlocks;
            v.push_back({r, s, R_PART, 0, off, off, (long)kRedBlocks, (long)count, ps});
        }
}

// b_C (and its first V-cycle input b_C/D) from the global row owners to the corner partition
void xf_corner_in(const Geom &g, std::vector<Xfer> &v)
{
    std::vector<int> lo, hi;
    gowners(g, lo, hi);
    for (int r = 0; r < g.P; ++r) {
        need_rows(v, r, lo, hi, R_BC, 0, g.lrow0(0, r), g.lrow1(0, r), g.lpitch[0], 0, g.lpitch[0]);
        need_rows(v, r, lo, hi, R_LRHO, 0, g.lrow0(0, r), g.lrow1(0, r), g.lpitch[0], 0, g.lpitch[0]);
    }
}

// the corner result z_C from the corner partition back to the global row owners
void xf_corner_out(const Geom &g, std::vector<Xfer> &v, int zrole)
{
    std::vector<int> lo, hi;
    lowners(g, 0, lo, hi);
    for (int s = 0; s < g.Pb; ++s)
        need_rows(v, s, lo, hi, zrole, 0, g.J[s], g.J[s + 1], g.lpitch[0], 0, g.lpitch[0]);
}

// level-l right-hand side of a strip's sweep: the halo rows above (recomputed from zero inflow,
// certified) and the row below (the restriction's bottom fine row)
void xf_mg_rhs(const Geom &g, std::vector<Xfer> &v, int l, int role, int slot)
{
    std::vector<int> lo, hi;
    lowners(g, l, lo, hi);
    for (int r = 0; r < g.P; ++r) {
        const int a = g.lrow1(l, r);
        need_rows(v, r, lo, hi, role, slot, a, a + g.shalo(l, r), g.lpitch[l], 0, g.lpitch[l]);
        const int b = g.lrow0(l, r);
        need_rows(v, r, lo, hi, role, slot, b - 1, b, g.lpitch[l], 0, g.lpitch[l]);
    }
}

// pre-smoothed e of level l: two rows below (residual of the restriction's bottom fine row) and
// one above
void xf_mg_e(const Geom &g, std::vector<Xfer> &v, int l)
{
    std::vector<int> lo, hi;
    lowners(g, l, lo, hi);
    for (int r = 0; r < g.P; ++r) {
        const int b = g.lrow0(l, r), a = g.lrow1(l, r);
        need_rows(v, r, lo, hi, R_LE, l, b - 2, b, g.lpitch[l], 0, g.lpitch[l]);
        need_rows(v, r, lo, hi, R_LE, l, a, a + 1, g.lpitch[l], 0, g.lpitch[l]);
    }
}

// one row on each side at level l (the coarse correction for the prolongation; the corner
// iterate's update)
void xf_mg_pm1(const Geom &g, std::vector<Xfer> &v, int l, int role, int slot)
{
    std::vector<int> lo, hi;
    lowners(g, l, lo, hi);
    for (int r = 0; r < g.P; ++r) {
        const int b = g.lrow0(l, r), a = g.lrow1(l, r);
        need_rows(v, r, lo, hi, role, slot, b - 1, b, g.lpitch[l], 0, g.lpitch[l]);
        need_rows(v, r, lo, hi, role, slot, a, a + 1, g.lpitch[l], 0, g.lpitch[l]);
    }
}

// post-smoothing right-hand side g: the halo rows above
void xf_mg_g(const Geom &g, std::vector<Xfer> &v, int l)
{
    std::vector<int> lo, hi;
    lowners(g, l, lo, hi);
    for (int r = 0; r < g.P; ++r) {
        const int a = g.lrow1(l, r);
        need_rows(v, r, lo, hi, R_LG, l, a, a + g.shalo(l, r), g.lpitch[l], 0, g.lpitch[l]);
    }
}

// every strip's rows of level l to every rank (the levels that run whole)
void xf_mg_gather(const Geom &g, std::vector<Xfer> &v, int l, int role, int slot)
{
    std::vector<int> lo, hi;
    lowners(g, l, lo, hi);
    for (int r = 0; r < g.P; ++r) need_rows(v, r, lo, hi, role, slot, 1, g.nl[l] + 1, g.lpitch[l], 0, g.lpitch[l]);
}

// ===================================================================================== transport
struct NcclApi {
    ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
    ncclResult_t (*gstart)();
    ncclResult_t (*gend)();
    const char *(*errstr)(ncclResult_t);
    ncclResult_t (*uid)(ncclUniqueId *);
    ncclResult_t (*init)(ncclComm_t *, int, ncclUniqueId, int);
    ncclResult_t (*destroy)(ncclComm_t);
    ncclResult_t (*count)(const ncclComm_t, int *);
    ncclResult_t (*urank)(const ncclComm_t, int *);
    ncclResult_t (*asyncerr)(ncclComm_t, ncclResult_t *);     // optional (failure detection)
};

// NCCL is resolved at run time: SPP_NCCL_LIB if set (the binding points it at torch's libnccl),
// else the libnccl.so.2 already loaded in the process, else the one the loader finds.
static const NcclApi *nccl_api(std::string *why)
{
    static NcclApi api;
    static int state = 0;               // 0 unknown, 1 ok, -1 missing
    static std::string err;
    if (state == 0) {
        void *h = nullptr;
        const char *env = getenv("SPP_NCCL_LIB");
        if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        bool ok = h != nullptr;
#define SPP_SYM(field, name)                                             \
        if (ok) {                                                        \
            *(void **)&api.field = dlsym(h, name);                       \
            if (!api.field) { ok = false; err = std::string("missing ") + name; } \
        }
        SPP_SYM(send, "ncclSend") SPP_SYM(recv, "ncclRecv") SPP_SYM(gstart, "ncclGroupStart")
        SPP_SYM(gend, "ncclGroupEnd") SPP_SYM(errstr, "ncclGetErrorString") SPP_SYM(uid, "ncclGetUniqueId")
        SPP_SYM(init, "ncclCommInitRank") SPP_SYM(destroy, "ncclCommDestroy") SPP_SYM(count, "ncclCommCount")
        SPP_SYM(urank, "ncclCommUserRank")
#undef SPP_SYM
        if (ok) *(void **)&api.asyncerr = dlsym(h, "ncclCommGetAsyncError");
        if (!h) err = std::string("cannot load libnccl.so.2: ") + (dlerror() ? dlerror() : "?");
        state = ok ? 1 : -1;
    }
    if (state < 0) { if (why) *why = err; return nullptr; }
    return &api;
}

static double *role_ptr(Ctx *c, int role, int slot)
{
    switch (role) {
    case R_V: return c->V[slot];
    case R_Z: return c->Z[slot];
    case R_U: return c->U;
    case R_W: return c->w;
    case R_CHAIN: return c->chain;
    case R_LB: return c->lev[slot].b;
    case R_LE: return c->lev[slot].e;
    case R_LQ: return c->lev[slot].q;
    case R_LG: return c->lev[slot].g;
    case R_LRHO: return c->lev[slot].rho;
    case R_BC: return c->Bc;
    case R_ZC: return c->Zc;
    case R_ZC2: return c->Zc2;
    case R_PART: return c->part;
    case R_CBUF: return c->cbuf;
    case R_F: return c->F;
    default: return nullptr;
    }
}

static spp_status dfail(Dist *d, spp_status code, const std::string &msg)
{
    for (Ctx *c : d->cx) c->err = msg;
    fprintf(stderr, "[spp] %s\n", msg.c_str());
    return code;
}

// Execute one exchange step.  Loopback: device copies between the strips' buffers (one stream).
// NCCL: one group of ncclSend / ncclRecv (matched in list order, which every rank generates
// identically) on the context's stream; non-contiguous blocks go through a staging buffer.
spp_status exchange_rows(Dist *d, const std::vector<Xfer> &xs)
{
    d->nexch++;
    if (xs.empty()) return SPP_OK;
    double bytes = 0;
    for (const Xfer &x : xs)
        if (d->me < 0 || x.src == d->me || x.dst == d->me) bytes += 8.0 * x.width * x.rows;
    ProfScope ps(d->cx[0], 11, bytes);
    if (d->me < 0) {
        for (const Xfer &x : xs) {
            double *sp = role_ptr(d->cx[x.src], x.role, x.slot) + x.soff;
            double *dp = role_ptr(d->cx[x.dst], x.role, x.slot) + x.doff;
            const cudaError_t e = cudaMemcpy2DAsync(dp, x.pitch * sizeof(double), sp, x.pitch * sizeof(double),
                                                    x.width * sizeof(double), x.rows, cudaMemcpyDeviceToDevice, d->st);
            if (e != cudaSuccess) return dfail(d, SPP_E_CUDA, std::string("loopback exchange: ") + cudaGetErrorString(e));
            d->nxfer++;
            d->xbytes += 8.0 * x.width * x.rows;
        }
        return SPP_OK;
    }
    std::string why;
    const NcclApi *api = nccl_api(&why);
    if (!api) return dfail(d, SPP_E_NCCL, "NCCL unavailable: " + why);
    Ctx *c = d->cx[0];
    const int me = d->me;
    auto contig = [](const Xfer &x) { return x.rows == 1 || x.width == x.pitch; };
    size_t need = 0;
    for (const Xfer &x : xs)
        if ((x.src == me || x.dst == me) && !contig(x)) need += (size_t)x.width * x.rows;
    if (need > d->stage_cap) {
        if (d->stage) cudaFree(d->stage);
        d->stage = nullptr;
        d->stage_cap = 0;
        if (cudaMalloc(&d->stage, need * sizeof(double)) != cudaSuccess) return dfail(d, SPP_E_NOMEM, "NCCL staging");
        d->stage_cap = need;
    }
    std::vector<double *> buf(xs.size(), nullptr);
    size_t o = 0;
    for (size_t k = 0; k < xs.size(); ++k) {
        const Xfer &x = xs[k];
        if (x.src != me && x.dst != me) continue;
        double *base = role_ptr(c, x.role, x.slot) + (x.src == me ? x.soff : x.doff);
        if (contig(x)) { buf[k] = base; continue; }
        buf[k] = d->stage + o;
        o += (size_t)x.width * x.rows;
        if (x.src == me)
            cudaMemcpy2DAsync(buf[k], x.width * sizeof(double), base, x.pitch * sizeof(double), x.width * sizeof(double),
                              x.rows, cudaMemcpyDeviceToDevice, d->st);
    }
    ncclResult_t rc = api->gstart();
    for (size_t k = 0; k < xs.size() && rc == ncclSuccess; ++k) {
        const Xfer &x = xs[k];
        const size_t cnt = (size_t)x.width * x.rows;
        if (x.src == me) rc = api->send(buf[k], cnt, ncclDouble, x.dst, (ncclComm_t)d->comm, d->st);
        else if (x.dst == me) rc = api->recv(buf[k], cnt, ncclDouble, x.src, (ncclComm_t)d->comm, d->st);
        if (x.src == me || x.dst == me) { d->nxfer++; d->xbytes += 8.0 * cnt; }
    }
    const ncclResult_t rc2 = api->gend();
    if (rc == ncclSuccess) rc = rc2;
    if (rc != ncclSuccess) return dfail(d, SPP_E_NCCL, std::string("NCCL exchange: ") + api->errstr(rc));
    if (api->asyncerr) {                               // a failure NCCL has already seen (dead peer, network)
        ncclResult_t ar = ncclSuccess;
        if (api->asyncerr((ncclComm_t)d->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
            return dfail(d, SPP_E_NCCL, std::string("NCCL asynchronous error: ") + api->errstr(ar));
    }
    for (size_t k = 0; k < xs.size(); ++k) {
        const Xfer &x = xs[k];
        if (x.dst != me || contig(x)) continue;
        double *base = role_ptr(c, x.role, x.slot) + x.doff;
        cudaMemcpy2DAsync(base, x.pitch * sizeof(double), buf[k], x.width * sizeof(double), x.width * sizeof(double),
                          x.rows, cudaMemcpyDeviceToDevice, d->st);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return dfail(d, SPP_E_CUDA, std::string("NCCL exchange staging: ") + cudaGetErrorString(e));
    (void)c;
    return SPP_OK;
}

#define DTRY(expr)                               \
    do {                                         \
        const spp_status _s = (expr);            \
        if (_s != SPP_OK) return _s;             \
    } while (0)
#define DCUDA(d, expr)                                                                      \
    do {                                                                                    \
        const cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) return dfail(d, SPP_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

// ===================================================================================== geometry
static inline double *pslot(Ctx *c, int k) { return c->part + (size_t)k * c->nparts * kRedBlocks; }
static inline double *pseg(Ctx *c, int k) { return pslot(c, k) + (size_t)c->rank * kRedBlocks; }

// Wait for a stream on the host.  Loopback: a plain synchronise.  NCCL: the stream holds
// sends / receives that never complete when a peer has died or left the collective order, so
// poll it, ask NCCL for an asynchronous error now and then, and give up after
// SPP_NCCL_TIMEOUT_S seconds (default 600) with SPP_E_NCCL instead of hanging (SURVEY 5,
// failure detection; no recovery: the caller destroys the context).
static spp_status dist_wait(Dist *d, cudaStream_t st)
{
    if (d->me < 0) { DCUDA(d, cudaStreamSynchronize(st)); return SPP_OK; }
    const NcclApi *api = nccl_api(nullptr);
    static const double limit = [] { const char *e = getenv("SPP_NCCL_TIMEOUT_S"); const double v = e ? atof(e) : 0.0; return v > 0.0 ? v : 600.0; }();
    const auto t0 = std::chrono::steady_clock::now();
    for (unsigned long spins = 1;; ++spins) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) return SPP_OK;
        if (e != cudaErrorNotReady) return dfail(d, SPP_E_CUDA, std::string("stream wait: ") + cudaGetErrorString(e));
        if ((spins & 0xfff) != 0) continue;
        if (api && api->asyncerr) {
            ncclResult_t ar = ncclSuccess;
            if (api->asyncerr((ncclComm_t)d->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
                return dfail(d, SPP_E_NCCL, std::string("NCCL asynchronous error: ") + api->errstr(ar));
        }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit)
            return dfail(d, SPP_E_NCCL, "timeout waiting for an exchange (SPP_NCCL_TIMEOUT_S): a peer is gone or out of step");
    }
}

static spp_status fetch_sum_all(Dist *d, Ctx *c, int k, double *out)
{
    const int cnt = c->nparts * kRedBlocks;
    DCUDA(d, cudaMemcpyAsync(c->hpin, pslot(c, k), sizeof(double) * cnt, cudaMemcpyDeviceToHost, c->st));
    DTRY(dist_wait(d, c->st));
    double s = 0.0;
    for (int i = 0; i < cnt; ++i) s += c->hpin[i];
    *out = s;
    return SPP_OK;
}

// Geometry + the strips' level plans, after the (replicated) setup.  Identical on every rank:
// it depends on the partition, the level sizes, the certified halos and the line contractions.
static spp_status dist_finish(Dist *d)
{
    Geom &g = d->g;
    Ctx *c = d->cx[0];
    const int P = g.P, n = c->n, N = c->N;
    g.N = N; g.n = n; g.m = N - 1; g.L = c->L; g.pitch = c->P;
    g.nl.resize(c->L); g.lpitch.resize(c->L);
    for (int l = 0; l < c->L; ++l) { g.nl[l] = c->lev[l].n; g.lpitch[l] = c->lev[l].pitch; }
    // strip levels: the first D levels whose certified halo exists and whose strips tile
    int Dreq = c->tune.dist_levels;
    int D = std::max(0, std::min(Dreq, c->L - 1));
    for (;;) {
        bool ok = D >= 1 && (n >> D) >= P;
        for (int l = 0; ok && l < D; ++l) ok = c->lev[l].halo_cert >= 0;
        if (ok) {
            std::vector<int> Cb(P + 1);
            Cb[0] = 1; Cb[P] = n + 1;
            for (int r = 1; r < P; ++r) Cb[r] = (int)std::lround((double)r * (n >> D) / P) << D;
            g.Cb = Cb;
            g.D = D;
            g.halo.assign(D, 0);
            for (int l = 0; l < D; ++l) g.halo[l] = c->lev[l].halo_cert;
            for (int l = 0; ok && l < D; ++l)
                for (int r = 0; ok && r < P; ++r) {
                    Level tmp = c->lev[l];
                    ok = plan_tiles(c, g.nl[l], g.lrow1(l, r) - g.lrow0(l, r), g.halo[l], c->lev[l].halo_certx, false, tmp);
                }
        }
        if (ok) break;
        if (--D < 1)
            return dfail(d, SPP_E_ARG, "row strips: the corner multigrid has no level with a certified halo that "
                                       "tiles into strips (corner too small for this many ranks?)");
    }
    // line chains: every rank's chunk extents (the same plan each rank's setup_lines made)
    g.xstart.assign(P, -1); g.ylo.assign(P, 0); g.yhi.assign(P, -1); g.ystart.assign(P, 0);
    g.ncta.assign(P, 0);
    for (int r = 0; r < P; ++r) {
        if (g.top(r)) {
            const int lo = N - g.J[r + 1], hi = N - 1 - g.J[r];
            const auto ch = plan_chain_chunks(0, c->kx, lo, hi, c->sm_count);
            int st = lo;
            for (const auto &k : ch) st = std::min(st, k.start);
            g.xstart[r] = st < lo ? st : -1;
            g.ncta[r] = (int)wave_chain_ctas(c, g.J[r + 1] - g.J[r]);
        } else {
            const int nl = n - 1;
            const int lo = (int)((long)nl * r / g.Pb), hi = (int)((long)nl * (r + 1) / g.Pb) - 1;
            g.ylo[r] = lo; g.yhi[r] = hi;
            const auto ch = plan_chain_chunks(1, c->ky, lo, hi, c->sm_count);
            int st = lo;
            for (const auto &k : ch) st = std::min(st, k.start);
            g.ystart[r] = st;
        }
    }
    g.chain_ld = c->chain_ld;
    g.ext_slot = (int)wave_chain_ctas(c, n) + 1;
    g.mii_cols = n - 1;
    // per local strip: its levels' rows and tile plans
    for (int r = 0; r < P; ++r) {
        Ctx *cr = d->ctx_of(r);
        if (!cr) continue;
        for (int l = 0; l < cr->L; ++l) {
            Level &Lv = cr->lev[l];
            if (l <= D) { Lv.slo = g.lrow0(l, r); Lv.shi = g.lrow1(l, r) - 1; }
            else { Lv.slo = 1; Lv.shi = Lv.n; }
            Lv.sdist = l < D;
            Lv.shalo = l < D ? g.shalo(l, r) : 0;
            if (l < D) plan_tiles(cr, Lv.n, Lv.shi - Lv.slo + 1, g.halo[l], Lv.halo_certx, false, Lv);
        }
    }
    return SPP_OK;
}

// ===================================================================================== setup
// Coefficients: every rank holds its own rows of c1, c2, r; they are all-gathered into each
// rank's staging buffer and the setup (coefficients, line factors, multigrid levels, halo
// certificates) runs replicated, so every rank plans with the same numbers.
spp_status setup_dist(Ctx *c0, const double *c1, const double *c2, const double *r, spp_mem mem)
{
    Dist *d = c0->dist;
    Geom &g = d->g;
    const int m = c0->m;
    const size_t mm = (size_t)m * m;
    if (d->me < 0) {                                   // loopback: the caller's arrays are whole
        for (Ctx *c : d->cx) DTRY(setup_2d_ctx(c, c1, c2, r, mem));
        return dist_finish(d);
    }
    Ctx *c = d->cx[0];
    const int me = d->me;
    const size_t own = (size_t)(g.J[me + 1] - g.J[me]) * m, off = (size_t)(g.J[me] - 1) * m;
    const cudaMemcpyKind kind = mem == SPP_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const double *src[3] = {c1, c2, r};
    for (int a = 0; a < 3; ++a)
        DCUDA(d, cudaMemcpyAsync(c->cbuf + a * mm + off, src[a], sizeof(double) * own, kind, c->st));
    std::vector<Xfer> xs;
    for (int s = 0; s < g.P; ++s)
        for (int t = 0; t < g.P; ++t) {
            if (s == t) continue;
            const long cnt = (long)(g.J[s + 1] - g.J[s]) * m, o = (long)(g.J[s] - 1) * m;
            for (int a = 0; a < 3; ++a) xs.push_back({s, t, R_CBUF, 0, o + (long)(a * mm), o + (long)(a * mm), cnt, 1, cnt});
        }
    DTRY(exchange_rows(d, xs));
    DTRY(setup_2d_ctx(c, c->cbuf, c->cbuf + mm, c->cbuf + 2 * mm, SPP_DEVICE));
    return dist_finish(d);
}

// ===================================================================================== preconditioner
static void launch_mii_dist(Ctx *c, const Geom &g, int t, const double *v, double *z)
{
    WaveArgs a{};
    a.nl = g.n - 1; a.pv = c->P; a.pc = c->P; a.ioff = g.n; a.joff = g.J[t] - 1;
    a.nr = a.nr_out = g.J[t + 1] - g.J[t];
    a.q = v; a.z = z; a.cd = c->cd;
    const bool scaled = !c->weighted;
    if (scaled) { ensure_y0(c); a.ca = c->ya; a.cn = c->yn; }    // D z = v + aE z_E + aN z_N (y-form)
    else { a.ca = c->ca; a.cn = c->cn; }           // z = (D v)/D + ca z_E + cn z_N (z-form)
    a.ext_in = t < g.P - 1 ? c->chain + (long)g.ext_slot * c->chain_ld : nullptr;
    a.chain_last = t > g.Pb ? 1 : 0;
    launch_wave_chain(c, a, c->N + 1, c->N + 1, scaled, 1, (double)a.nl * a.nr * (scaled ? 40.0 : 32.0));
}

// V-cycle on the strips (levels < D) or whole on every rank (levels >= D); the result in
// lev[l].q (own rows for a strip level), as the single-GPU vcycle returns it.
static spp_status vcycle_dist(Dist *d, int l, bool rs)
{
    const Geom &g = d->g;
    const int P = g.P;
    const int Rrole = l == 0 ? R_LRHO : R_LB;
    std::vector<Xfer> xs;
    if (l >= g.D) {
        xf_mg_gather(g, xs, l, Rrole, l);
        DTRY(exchange_rows(d, xs));
        for (int r = 0; r < P; ++r)
            if (Ctx *c = d->ctx_of(r)) vcycle(c, l, l == 0 ? c->lev[0].rho : c->lev[l].b, rs);
        return SPP_OK;
    }
    xf_mg_rhs(g, xs, l, Rrole, l);
    DTRY(exchange_rows(d, xs));
    for (int r = 0; r < P; ++r)                        // pre-smoothing from zero
        if (Ctx *c = d->ctx_of(r)) {
            Level &L = c->lev[l];
            launch_gs(c, l, 0, l == 0 ? L.rho : L.b, nullptr, L.e, nullptr, rs);
        }
    xs.clear();
    xf_mg_e(g, xs, l);
    DTRY(exchange_rows(d, xs));
    const bool zf = d->cx[0]->mg_zform;
    for (int r = 0; r < P; ++r)                        // residual + restriction onto the strip's coarse rows
        if (Ctx *c = d->ctx_of(r)) {
            Level &L = c->lev[l];
            launch_resid_restrict(c, l, nullptr, L.e, false, zf);   // L.e: the sweep from zero above
        }
    DTRY(vcycle_dist(d, l + 1, zf));
    if (l + 1 < g.D) {
        xs.clear();
        xf_mg_pm1(g, xs, l + 1, R_LQ, l + 1);
        DTRY(exchange_rows(d, xs));
    }
    for (int r = 0; r < P; ++r)                        // prolongation + the post-sweep's W/S part
        if (Ctx *c = d->ctx_of(r)) {
            Level &L = c->lev[l];
            launch_gs_prep(c, l, l == 0 ? L.rho : L.b, L.e, c->lev[l + 1].q, rs);
        }
    xs.clear();
    xf_mg_g(g, xs, l);
    DTRY(exchange_rows(d, xs));
    for (int r = 0; r < P; ++r)
        if (Ctx *c = d->ctx_of(r)) launch_gs_sweep(c, l, c->lev[l].g, c->lev[l].q);
    return SPP_OK;
}

// z = M^{-1} v on the strips (eq:2D blocks, I -> Y -> X -> C); v = V[k], z = Z[k].
static spp_status precond_dist(Dist *d, int k, int *cycles, int *cap)
{
    const Geom &g = d->g;
    const int P = g.P, n = g.n;
    std::vector<Xfer> xs;
    // M_II, top strip first (each strip's chain takes the bottom row of the strip above)
    for (int t = P - 1; t >= g.Pb; --t) {
        if (Ctx *c = d->ctx_of(t)) launch_mii_dist(c, g, t, c->V[k], c->Z[k]);
        if (t > g.Pb) {
            xs.clear();
            xf_mii(g, xs, t, k);
            DTRY(exchange_rows(d, xs));
        }
    }
    // M_XX warm-up rows and M_YY column blocks, then both chains
    xs.clear();
    xf_xhalo(g, xs, k, k);
    xf_yin(g, xs, k, k);
    DTRY(exchange_rows(d, xs));
    for (int r = 0; r < P; ++r)
        if (Ctx *c = d->ctx_of(r)) launch_lines(c, c->V[k], c->Z[k]);
    xs.clear();
    xf_yout(g, xs, k);
    xf_rown1(g, xs, k);
    DTRY(exchange_rows(d, xs));
    // corner right-hand side on the bottom strips' rows, ||S_0 b_C||^2
    for (int r = 0; r < P; ++r) {
        Ctx *c = d->ctx_of(r);
        if (!c) continue;
        Level &L0 = c->lev[0];
        if (g.top(r)) {
            DCUDA(d, cudaMemsetAsync(pseg(c, 1), 0, sizeof(double) * kRedBlocks, c->st));
            continue;
        }
        const int j0 = g.J[r], j1 = g.J[r + 1] - 1;
        int nb = 0, nt = 0;
        seg_shape(n, j1 - j0 + 1, &nb, &nt);
        k_corner_rhs<<<nb, nt, 0, c->st>>>(c->N, c->P, L0.pitch, c->V[k], c->Z[k],
            c->aE, c->aN, c->rr, c->aW, c->aS, L0.hb, L0.kb, c->weighted, c->Bc, pseg(c, 1), L0.rho, c->cd, c->mg_zform,
            j0, j1);
        c->launches++;
    }
    xs.clear();
    xf_partials(g, xs, 1, 1);
    xf_corner_in(g, xs);
    DTRY(exchange_rows(d, xs));
    Ctx *lead = d->cx[0];
    double b0sq = 0.0;
    DTRY(fetch_sum_all(d, lead, 1, &b0sq));
    // stationary V-cycle iteration (reading R6): exactly corner_solve's decisions
    const double b0 = std::sqrt(b0sq);
    double res = b0;
    int cyc = 0;
    *cap = 0;
    const int fixed = lead->opt.mg_fixed_cycles;
    for (;;) {
        if (fixed > 0) { if (cyc >= fixed) break; }
        else {
            if (res <= lead->opt.mg_reduction * b0) break;
            if (cyc >= lead->opt.mg_max_cycles) { *cap = 1; break; }
        }
        DTRY(vcycle_dist(d, 0, lead->mg_zform));
        xs.clear();
        xf_mg_pm1(g, xs, 0, R_LQ, 0);
        DTRY(exchange_rows(d, xs));
        for (int r = 0; r < P; ++r)
            if (Ctx *c = d->ctx_of(r)) {
                const double *zprev = cyc == 0 ? nullptr : ((cyc - 1) & 1 ? c->Zc2 : c->Zc);
                double *zn = (cyc & 1) ? c->Zc2 : c->Zc;
                launch_cycle_update(c, zprev, c->lev[0].q, zn, c->Bc, c->lev[0].rho, pseg(c, 0));
            }
        xs.clear();
        xf_partials(g, xs, 0, 1);
        DTRY(exchange_rows(d, xs));
        ++cyc;
        if (fixed <= 0) {
            double s = 0.0;
            DTRY(fetch_sum_all(d, lead, 0, &s));
            res = std::sqrt(s);
        }
    }
    *cycles = cyc;
    // z_C back to the bottom strips
    const int zrole = cyc == 0 ? -1 : (((cyc - 1) & 1) ? R_ZC2 : R_ZC);
    if (zrole >= 0) {
        xs.clear();
        xf_corner_out(g, xs, zrole);
        DTRY(exchange_rows(d, xs));
    }
    for (int r = 0; r < g.Pb; ++r)
        if (Ctx *c = d->ctx_of(r)) {
            const double *zc = zrole < 0 ? nullptr : role_ptr(c, zrole, 0);
            const int j0 = g.J[r], j1 = g.J[r + 1] - 1;
            k_corner_out<<<red_grid((long)n * (j1 - j0 + 1)), 256, 0, c->st>>>(n, c->lev[0].pitch, zc, c->P, c->Z[k],
                                                                               nullptr, j0, j1);
            c->launches++;
        }
    return SPP_OK;
}

// ===================================================================================== FGMRES
// The single-GPU solve_2d on strips: the same steps in the same order; every reduction is the
// all-gathered per-strip partials summed in one fixed order, so every rank takes the same
// decisions.
spp_status solve_dist(Ctx *c0, const double *f, double *u, spp_mem mem, double *hist, int hcap, spp_stats *st)
{
    Dist *d = c0->dist;
    const Geom &g = d->g;
    const int P = g.P, m = g.m, maxit = c0->opt.max_iters;
    Ctx *lead = d->cx[0];
    const int64_t l0 = [&] { int64_t s = 0; for (Ctx *c : d->cx) s += c->launches; return s; }();
    cudaEvent_t e0, e1;
    DCUDA(d, cudaEventCreate(&e0));
    DCUDA(d, cudaEventCreate(&e1));
    DCUDA(d, cudaEventRecord(e0, d->st));
    auto own = [&](int r, int &j0, int &nr) { j0 = g.J[r]; nr = g.J[r + 1] - g.J[r]; };
    const int weighted = lead->weighted, stop = lead->opt.stop;
    for (int r = 0; r < P; ++r)
        if (Ctx *c = d->ctx_of(r)) {
            int j0, nr;
            own(r, j0, nr);
            const double *fr = f + (d->me < 0 ? (size_t)(j0 - 1) * m : 0);
            if (mem == SPP_HOST) {
                DCUDA(d, cudaMemcpyAsync(c->cbuf, fr, sizeof(double) * (size_t)nr * m, cudaMemcpyHostToDevice, c->st));
                fr = c->cbuf;
            }
            k_pack<<<red_grid((long)nr * m), 256, 0, c->st>>>(m, c->P, fr, c->F, j0, nr);
            DCUDA(d, ensure_vectors(c, 1));
            k_rhs<<<red_grid((long)m * nr), kRedThreads, 0, c->st>>>(m, c->P, c->F, c->aE, c->aN, c->rr, c->aW, c->aS,
                                                                    weighted, c->V[0], pseg(c, 0), j0, nr);
            DCUDA(d, cudaMemsetAsync(c->U, 0, sizeof(double) * c->G, c->st));
            c->launches += 2;
        }
    std::vector<Xfer> xs;
    xf_partials(g, xs, 0, 1);
    DTRY(exchange_rows(d, xs));
    double bsq = 0.0;
    DTRY(fetch_sum_all(d, lead, 0, &bsq));
    const double beta = std::sqrt(bsq);
    if (!std::isfinite(beta)) return dfail(d, SPP_E_NONFINITE, "||W f|| is not finite (NaN/Inf in the right-hand side)");
    std::vector<double> H((size_t)(maxit + 1) * (maxit + 1), 0.0), cs(maxit + 1), sn(maxit + 1), gg(maxit + 2, 0.0),
        yv(maxit + 1);
    if (hist && hcap > 0) hist[0] = beta;
    int iters = 0, converged = 0, mg_tot = 0, mg_min = 1 << 30, mg_max = 0, caps = 0;
    double resf = beta;
    const double target = (stop == SPP_STOP_ABS_L2) ? lead->opt.tol : lead->opt.tol * beta;
    // flat own-row ranges of the Krylov vectors
    auto flat = [&](int r, long &off, long &cnt) { off = (long)g.J[r] * g.pitch; cnt = (long)(g.J[r + 1] - g.J[r]) * g.pitch; };
    if (beta == 0.0) converged = 1;
    else {
        for (int r = 0; r < P; ++r)
            if (Ctx *c = d->ctx_of(r)) {
                long off, cnt;
                flat(r, off, cnt);
                k_scale<<<red_grid(cnt / 2), 256, 0, c->st>>>(cnt, c->V[0] + off, 1.0 / beta);
                c->launches++;
            }
        gg[0] = beta;
        for (int k = 0; k < maxit; ++k) {
            for (Ctx *c : d->cx) DCUDA(d, ensure_vectors(c, k + 1));
            int cyc = 0, cap = 0;
            DTRY(precond_dist(d, k, &cyc, &cap));
            if (cap && lead->opt.mg_strict) return dfail(d, SPP_E_MG_CAP, "corner multigrid hit the cycle cap");
            mg_tot += cyc; mg_min = std::min(mg_min, cyc); mg_max = std::max(mg_max, cyc); caps += cap;
            // w = W A z_k on the strips (one-row halos of z_k), with <w, v_0>
            xs.clear();
            xf_vec_halo(g, xs, R_Z, k);
            DTRY(exchange_rows(d, xs));
            for (int r = 0; r < P; ++r)
                if (Ctx *c = d->ctx_of(r)) {
                    int j0, nr;
                    own(r, j0, nr);
                    ProfScope ps(c, 0, 48.0 * m * nr);
                    k_spmv<<<red_grid((long)m * nr), kRedThreads, 0, c->st>>>(m, c->P, c->Z[k], c->aE, c->aN, c->rr,
                        c->aW, c->aS, weighted, c->w, c->V[0], pseg(c, 0), j0, nr);
                    c->launches++;
                }
            xs.clear();
            xf_partials(g, xs, 0, 1);
            DTRY(exchange_rows(d, xs));
            // modified Gram-Schmidt, one all-gather per dot product
            for (int j = 1; j <= k + 1; ++j) {
                for (int r = 0; r < P; ++r)
                    if (Ctx *c = d->ctx_of(r)) {
                        long off, cnt;
                        flat(r, off, cnt);
                        const double *y = j <= k ? c->V[j] + off : c->w + off;
                        ProfScope ps(c, 7, 32.0 * cnt);
                        k_mgs<<<red_grid(cnt), kRedThreads, 0, c->st>>>(cnt, c->w + off, c->V[j - 1] + off, pslot(c, j - 1),
                                                                       c->dscal + (j - 1), y, pseg(c, j), P);
                        c->launches++;
                    }
                if (j == k + 1) break;
                xs.clear();
                xf_partials(g, xs, j, 1);
                DTRY(exchange_rows(d, xs));
            }
            // the last step above subtracted h_k v_k and formed ||w||^2 partials
            xs.clear();
            xf_partials(g, xs, k + 1, 1);
            DTRY(exchange_rows(d, xs));
            for (int r = 0; r < P; ++r)
                if (Ctx *c = d->ctx_of(r)) {
                    long off, cnt;
                    flat(r, off, cnt);
                    k_normalize<<<red_grid(cnt), kRedThreads, 0, c->st>>>(cnt, c->w + off, pslot(c, k + 1),
                                                                         c->dscal + k + 1, c->V[k + 1] + off, P);
                    c->launches++;
                }
            DCUDA(d, cudaMemcpyAsync(lead->hpin, lead->dscal, sizeof(double) * (k + 2), cudaMemcpyDeviceToHost, lead->st));
            DTRY(dist_wait(d, lead->st));
            double *h = &H[(size_t)k * (maxit + 1)];
            for (int j = 0; j <= k + 1; ++j) {
                h[j] = lead->hpin[j];
                if (!std::isfinite(h[j]))
                    return dfail(d, SPP_E_NONFINITE, "Hessenberg entry is not finite (NaN/Inf guard, SURVEY 5)");
            }
            for (int i = 0; i < k; ++i) {               // Givens (Saad 2003), as solve_2d
                const double t = cs[i] * h[i] + sn[i] * h[i + 1];
                h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
                h[i] = t;
            }
            const double den = std::hypot(h[k], h[k + 1]);
            if (den == 0.0) { cs[k] = 1.0; sn[k] = 0.0; }
            else { cs[k] = h[k] / den; sn[k] = h[k + 1] / den; }
            const bool brk = h[k + 1] == 0.0;
            h[k] = den; h[k + 1] = 0.0;
            gg[k + 1] = -sn[k] * gg[k];
            gg[k] = cs[k] * gg[k];
            const double res = std::fabs(gg[k + 1]);
            iters = k + 1;
            resf = res;
            if (hist && k + 1 < hcap) hist[k + 1] = res;
            if (brk) { converged = res <= target; break; }
            if (lead->opt.fixed_iters > 0) {
                if (k + 1 >= lead->opt.fixed_iters) { converged = res <= target; break; }
            } else if (res <= target) { converged = 1; break; }
        }
        for (int i = iters - 1; i >= 0; --i) {
            double t = gg[i];
            for (int j = i + 1; j < iters; ++j) t -= H[(size_t)j * (maxit + 1) + i] * yv[j];
            yv[i] = t / H[(size_t)i * (maxit + 1) + i];
        }
        for (int r = 0; r < P; ++r)
            if (Ctx *c = d->ctx_of(r)) {
                long off, cnt;
                flat(r, off, cnt);
                const double **hz = (const double **)(c->hpin + 8 * kRedBlocks * c->nparts);
                double *hy = (double *)(hz + maxit + 8);
                for (int j = 0; j < iters; ++j) { hz[j] = c->Z[j] + off; hy[j] = yv[j]; }
                const double **dptr = (const double **)(c->dscal + maxit + 8);
                double *dy = c->dscal + 2 * maxit + 16;
                DCUDA(d, cudaMemcpyAsync(dptr, hz, sizeof(double *) * iters, cudaMemcpyHostToDevice, c->st));
                DCUDA(d, cudaMemcpyAsync(dy, hy, sizeof(double) * iters, cudaMemcpyHostToDevice, c->st));
                k_update_x<<<red_grid(cnt / 2), 256, 0, c->st>>>(cnt, iters, dptr, dy, c->U + off, 0);
                c->launches++;
            }
    }
    for (Ctx *c : d->cx)
        if (c->sticky != cudaSuccess) { const cudaError_t se = c->sticky; c->sticky = cudaSuccess; DCUDA(d, se); }
    DCUDA(d, cudaEventRecord(e1, d->st));
    if (u) {
        for (int r = 0; r < P; ++r)
            if (Ctx *c = d->ctx_of(r)) {
                int j0, nr;
                own(r, j0, nr);
                double *ur = u + (d->me < 0 ? (size_t)(j0 - 1) * m : 0);
                if (mem == SPP_HOST) {
                    k_unpack<<<red_grid((long)nr * m), 256, 0, c->st>>>(m, c->P, c->U, c->cbuf, j0, nr);
                    DCUDA(d, cudaMemcpyAsync(ur, c->cbuf, sizeof(double) * (size_t)nr * m, cudaMemcpyDeviceToHost, c->st));
                } else {
                    k_unpack<<<red_grid((long)nr * m), 256, 0, c->st>>>(m, c->P, c->U, ur, j0, nr);
                }
                c->launches++;
            }
    }
    DCUDA(d, cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (st) {                                          // true residuals (after the timed region)
        memset(st, 0, sizeof(*st));
        xs.clear();
        xf_vec_halo(g, xs, R_U, 0);
        DTRY(exchange_rows(d, xs));
        for (int r = 0; r < P; ++r)
            if (Ctx *c = d->ctx_of(r)) {
                int j0, nr;
                own(r, j0, nr);
                k_spmv<<<kRedBlocks, kRedThreads, 0, c->st>>>(m, c->P, c->U, c->aE, c->aN, c->rr, c->aW, c->aS, 0, c->w,
                                                              nullptr, nullptr, j0, nr);
                k_resid_stats<<<kRedBlocks, kRedThreads, 0, c->st>>>(m, c->P, c->F, c->w, c->aE, c->aN, c->rr, c->aW,
                    c->aS, pseg(c, 0), (long)P * kRedBlocks, j0, nr);
            }
        xs.clear();
        xf_partials(g, xs, 0, 4);
        DTRY(exchange_rows(d, xs));
        double s4[4];
        for (int a = 0; a < 4; ++a) DTRY(fetch_sum_all(d, lead, a, &s4[a]));
        st->true_res_l2_rel = s4[2] > 0 ? std::sqrt(s4[0] / s4[2]) : 0.0;
        st->true_res_jacobi_rel = s4[3] > 0 ? std::sqrt(s4[1] / s4[3]) : 0.0;
        st->iters = iters; st->converged = converged;
        st->mg_cycles_total = mg_tot; st->mg_cycles_min = iters ? mg_min : 0; st->mg_cycles_max = mg_max;
        st->mg_cap_hits = caps; st->applies = iters;
        int64_t l1 = 0;
        for (Ctx *c : d->cx) l1 += c->launches;
        st->kernel_launches = (int32_t)(l1 - l0);
        st->res0 = beta; st->res_final = resf;
        st->setup_s = lead->setup_ms * 1e-3; st->solve_s = ms * 1e-3;
    }
    for (Ctx *c : d->cx) prof_collect(c);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return dfail(d, SPP_E_CUDA, std::string("solve: ") + cudaGetErrorString(e));
    return converged ? SPP_OK : SPP_NOT_CONVERGED;
}

void destroy_dist(Ctx *c)
{
    Dist *d = c->dist;
    if (!d) return;
    if (d->stage) cudaFree(d->stage);
    delete d;
}

// ===================================================================================== partition
// Default row strips: ceil(P/2) strips share the bottom half (rows 1..n) and the rest the top
// half (rows n+1..N-1), as evenly as possible; P = 1: one strip.
bool strip_partition(int N, int P, std::vector<int> &J)
{
    const int n = N / 2;
    J.assign(P + 1, 0);
    if (P == 1) { J[0] = 1; J[1] = N; return true; }
    const int Pb = (P + 1) / 2, Pt = P - Pb;
    if (Pb > n || Pt > n - 1) return false;
    for (int b = 0; b <= Pb; ++b) J[b] = 1 + (int)((long)n * b / Pb);
    // top strips: every strip that hands its bottom row to the strip below (all but the lowest)
    // spans a multiple of 32 rows (check_partition); the lowest takes the remainder
    const int s = std::max(32, (int)std::lround((double)(n - 1) / Pt / 32.0) * 32);
    if ((long)(Pt - 1) * s >= n - 1) return false;
    J[P] = N;
    for (int t = P - 1; t > Pb; --t) J[t] = J[t + 1] - s;
    return true;
}

// Check a partition gathered from the ranks: contiguous, covering 1..N-1, every strip non-empty,
// a boundary at n+1 (P > 1).  Sets Pb.
bool check_partition(int N, const std::vector<int> &J, int *Pb, std::string *why)
{
    const int P = (int)J.size() - 1, n = N / 2;
    if (J.front() != 1 || J.back() != N) { *why = "strips must cover rows 1..N-1"; return false; }
    int pb = -1;
    for (int r = 0; r < P; ++r) {
        if (J[r + 1] <= J[r]) { *why = "strip " + std::to_string(r) + " is empty or out of order"; return false; }
        if (J[r] == n + 1) pb = r;
    }
    if (P > 1 && pb < 1) { *why = "a strip boundary must sit at row n+1 = N/2+1 (the X/I | C/Y split)"; return false; }
    // the M_II relay publishes the bottom row of a strip's last CTA strip, lane 31 of its last
    // warp: every top strip with a strip below it in the top half spans whole warps (32 rows)
    for (int r = pb + 1; P > 1 && r < P; ++r)
        if ((J[r + 1] - J[r]) % 32 != 0) {
            *why = "top strip " + std::to_string(r) + " spans " + std::to_string(J[r + 1] - J[r]) +
                   " rows: every top strip above the lowest must span a multiple of 32 rows";
            return false;
        }
    *Pb = P > 1 ? pb : 1;
    return true;
}

}  // namespace spp

// ===================================================================================== ABI helpers
using namespace spp;
extern "C" {

spp_status spp_nccl_unique_id(uint8_t *id)
{
    std::string why;
    const NcclApi *api = nccl_api(&why);
    if (!id) return SPP_E_ARG;
    if (!api) { fprintf(stderr, "[spp] %s\n", why.c_str()); return SPP_E_NCCL; }
    ncclUniqueId u;
    if (api->uid(&u) != ncclSuccess) return SPP_E_NCCL;
    memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return SPP_OK;
}

spp_status spp_nccl_comm_create(const uint8_t *id, int32_t nranks, int32_t rank, void **comm)
{
    std::string why;
    const NcclApi *api = nccl_api(&why);
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return SPP_E_ARG;
    if (!api) { fprintf(stderr, "[spp] %s\n", why.c_str()); return SPP_E_NCCL; }
    ncclUniqueId u;
    memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    const ncclResult_t rc = api->init(&c, nranks, u, rank);
    if (rc != ncclSuccess) { fprintf(stderr, "[spp] ncclCommInitRank: %s\n", api->errstr(rc)); return SPP_E_NCCL; }
    *comm = (void *)c;
    return SPP_OK;
}

void spp_nccl_comm_destroy(void *comm)
{
    const NcclApi *api = nccl_api(nullptr);
    if (api && comm) api->destroy((ncclComm_t)comm);
}

// Host-only exchange schedule of one FGMRES iteration (k = 0, one corner cycle) for a synthetic
// geometry: N, the partition J (nranks+1), D strip levels with certified halo `halo` each, and a
// line-chain warm-up of `warm` lines.  Writes 11 int64 per block (step, src, dst, role, slot,
// soff, doff, width, rows, pitch, 0) for the blocks rank `rank` sends or receives (rank < 0: all)
// and returns the number of blocks (or a negative status).  Test hook for the multi-process
// orchestration (tests/test_multiproc.py); the solve uses the same generators.
int32_t spp_dist_plan(int32_t N, int32_t nranks, const int32_t *j, int32_t D, int32_t halo, int32_t warm, int32_t rank,
                      int64_t *out, int32_t cap)
{
    if (!j || nranks < 2 || N < 16 || (N % 2) || D < 1) return SPP_E_ARG;
    Geom g;
    g.N = N; g.n = N / 2; g.m = N - 1; g.P = nranks;
    g.J.assign(j, j + nranks + 1);
    std::string why;
    if (!check_partition(N, g.J, &g.Pb, &why)) return SPP_E_ARG;
    g.pitch = round_up(N + 1, 16);
    const int n = g.n;
    for (int nl = n; nl >= 4; nl /= 2) { g.nl.push_back(nl); g.lpitch.push_back(round_up(nl + 2, 16)); }
    g.L = (int)g.nl.size();
    if (D > g.L - 1 || (n >> D) < nranks) return SPP_E_ARG;
    g.D = D;
    g.halo.assign(D, halo);
    g.Cb.assign(nranks + 1, 0);
    g.Cb[0] = 1; g.Cb[nranks] = n + 1;
    for (int r = 1; r < nranks; ++r) g.Cb[r] = (int)std::lround((double)r * (n >> D) / nranks) << D;
    g.xstart.assign(nranks, -1); g.ylo.assign(nranks, 0); g.yhi.assign(nranks, -1); g.ystart.assign(nranks, 0);
    g.ncta.assign(nranks, 0);
    for (int r = 0; r < nranks; ++r) {
        if (g.top(r)) {
            const int lo = N - g.J[r + 1];
            g.xstart[r] = lo > 0 && warm > 0 ? std::max(0, lo - warm) : -1;
            g.ncta[r] = (g.J[r + 1] - g.J[r] + 63) / 64;
        } else {
            const int nl = n - 1;
            g.ylo[r] = (int)((long)nl * r / g.Pb); g.yhi[r] = (int)((long)nl * (r + 1) / g.Pb) - 1;
            g.ystart[r] = std::max(0, g.ylo[r] - warm);
        }
    }
    g.chain_ld = n + 32; g.ext_slot = (n + 63) / 64 + 1; g.mii_cols = n - 1;
    std::vector<std::vector<Xfer>> steps;
    auto step = [&](auto fn) { std::vector<Xfer> v; fn(v); steps.push_back(v); };
    for (int t = nranks - 1; t > g.Pb; --t) step([&](std::vector<Xfer> &v) { xf_mii(g, v, t, 0); });
    step([&](std::vector<Xfer> &v) { xf_xhalo(g, v, 0, 0); xf_yin(g, v, 0, 0); });
    step([&](std::vector<Xfer> &v) { xf_yout(g, v, 0); xf_rown1(g, v, 0); });
    step([&](std::vector<Xfer> &v) { xf_partials(g, v, 1, 1); xf_corner_in(g, v); });
    for (int l = 0; l < D; ++l) {
        step([&](std::vector<Xfer> &v) { xf_mg_rhs(g, v, l, l == 0 ? R_LRHO : R_LB, l); });
        step([&](std::vector<Xfer> &v) { xf_mg_e(g, v, l); });
    }
    step([&](std::vector<Xfer> &v) { xf_mg_gather(g, v, D, R_LB, D); });
    for (int l = D - 1; l >= 0; --l) {
        if (l + 1 < D) step([&](std::vector<Xfer> &v) { xf_mg_pm1(g, v, l + 1, R_LQ, l + 1); });
        step([&](std::vector<Xfer> &v) { xf_mg_g(g, v, l); });
    }
    step([&](std::vector<Xfer> &v) { xf_mg_pm1(g, v, 0, R_LQ, 0); });
    step([&](std::vector<Xfer> &v) { xf_partials(g, v, 0, 1); });
    step([&](std::vector<Xfer> &v) { xf_corner_out(g, v, R_ZC); });
    step([&](std::vector<Xfer> &v) { xf_vec_halo(g, v, R_Z, 0); });
    step([&](std::vector<Xfer> &v) { xf_partials(g, v, 0, 1); });
    step([&](std::vector<Xfer> &v) { xf_partials(g, v, 1, 1); });
    int32_t cnt = 0;
    for (size_t s = 0; s < steps.size(); ++s)
        for (const Xfer &x : steps[s]) {
            if (rank >= 0 && x.src != rank && x.dst != rank) continue;
            if (out && cnt < cap) {
                int64_t *o = out + 11 * (size_t)cnt;
                o[0] = (int64_t)s; o[1] = x.src; o[2] = x.dst; o[3] = x.role; o[4] = x.slot; o[5] = x.soff;
                o[6] = x.doff; o[7] = x.width; o[8] = x.rows; o[9] = x.pitch; o[10] = 0;
            }
            ++cnt;
        }
    return cnt;
}

}  // extern "C"
