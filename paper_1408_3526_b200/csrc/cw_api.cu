// cw_api.cu -- C ABI of the B200 whitening pipeline (include/cw_b200.h).
//
// Host side of the drop-in: owns the per-stream device state (observer
// state, smoothing state T^, raw-frame delay ring, outputs), folds the
// reference's constant tables into float tables for the fused kernel, and
// launches one cw_frame_kernel per frame.  Reference counterparts are cited
// per function; there is no CPU compute path: every frame runs on the GPU
// or the call fails with CW_ERR_CUDA.
#include "cw_inst.cuh"
#include "cw_generic.cuh"
#include "cw_jit.cuh"
#include "../../include/cw_b200.h"

#ifdef _OPENMP
#include <omp.h>
#endif
#include <cuda.h>  // CUstream / CUdeviceptr types of the stream memory operation entry point
#include <nvtx3/nvToolsExt.h>  // header-only NVTX ranges (visible in nsys / ncu --nvtx)

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace cwb;

// kernel instances, one translation unit each (cw_inst.cu)
#define CW_DECLARE(a, b, c, d, e, n) LaunchFn CW_INST_FN(a, b, c, d, e, n)();
CW_INSTANCES(CW_DECLARE)
#undef CW_DECLARE

namespace {

thread_local std::string g_create_error;
void (*g_phase_clocks)(unsigned long long *) = nullptr;  // CW_PHASE_TIMING: the last created pipeline's unit

// Compiled geometries: the default (4,4,2,3,3) and the SURVEY §8d C5 sweep.
// Symmetric lag grids of 9/17/33 entries get fully unrolled contraction
// kernels; any other grid runs the runtime-loop instance (NL = 0), which
// also carries the geometry's naive-spectrum kernel.  Each instance is its
// own translation unit (cw_inst.cu, compiled once per CW_INSTANCES entry).

bool find_inst(int kx, int ky, int kz, int bx, int by, int nl_sym, LaunchFn *out)
{
    bool geo = false;
    LaunchFn base{}, sym{};
    bool have_sym = false;
#define CW_FIND(a, b, c, d, e, n)                                   \
    if (kx == a && ky == b && kz == c && bx == d && by == e) {      \
        geo = true;                                                 \
        if (n == 0) base = CW_INST_FN(a, b, c, d, e, n)();          \
        else if (n == nl_sym) {                                     \
            sym = CW_INST_FN(a, b, c, d, e, n)();                   \
            have_sym = true;                                        \
        }                                                           \
    }
    CW_INSTANCES(CW_FIND)
#undef CW_FIND
    if (!geo) return false;
    if (have_sym) {  // the naive kernel lives in the NL = 0 unit
        sym.launch_naive = base.launch_naive;
        sym.naive_kernel = base.naive_kernel;
        sym.naive_smem = base.naive_smem;
        *out = sym;
    } else {
        *out = base;
    }
    return true;
}

}  // namespace

struct cw_handle {
    int kx, ky, kz, bx, by, mhx, mhy, mhz;
    int mx, my, mz;
    int W, H, NXB, halo, row_off;
    int device;
    int nlx, nly;
    double alpha;
    std::vector<double> lag_x, lag_y;
    LaunchFn fn;
    Tables tab;
    int grid;
    int sms = 0;
    cudaStream_t own = nullptr;
    void *d_raw = nullptr;  // PGM16 upload staging (cw_submit_raw), allocated on first use
    float *d_state = nullptr, *d_that = nullptr, *d_coef = nullptr, *d_frames = nullptr;
    float *d_res = nullptr, *d_pred = nullptr;  // 2 output sets each
    uint8_t *d_vidx = nullptr;
    // runtime-geometry path (cw_generic.cuh) for parameters without a
    // compiled fused instance; velocity indices are uint16 pairs when a lag
    // grid has more than 256 entries
    bool generic = false;
    int kind = 0;  // 0: compiled fused instance, 1: run-time compiled fused instance, 2: runtime-geometry kernels
    int idx_bytes = 1;
    GenTables gt{};
    void *d_gtab = nullptr;
    float2 *d_xf = nullptr;
    int nxf = 0;  // x-stage frames allocated
    // fused kernel work split (FrameArgs.work): static fraction + dynamic chunks
    unsigned int *d_work = nullptr;
    unsigned char *d_rank = nullptr;  // compact instances: rank u16 [nl], then (ix, iy) u8 pairs [nl]
    double dyn_static = 0.92;  // measured on C3 (tools/ab_kernel.py): 0.92 / 2 rows, ~1% faster than all-static
    int dyn_chunk = 2;
    // frame chaining (FrameArgs::done): per-CTA completion flags of the fused
    // kernel; with `chain` the split is static and every fused launch is a
    // programmatic dependent launch, so consecutive frames overlap
    unsigned int *d_done = nullptr;
    unsigned int seq = 0;
    bool chain = true;         // CW_CHAIN=0 turns it off
    bool last_static = false;  // the last fused launch used the static split
    // chained cw_submit: cuStreamWriteValue32 (driver entry point; null: not
    // available -> event waits) and its flags [0] upload, [1] download,
    // [2] ring-slot copy of a resident frame (copy engine)
    CUresult (*write_value)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    unsigned int *d_flags = nullptr;
    // per ring slot: tag (frame + 1) of the flagged copy that filled it, 0 if
    // it was filled in stream order; the next kernel's slot gets next_ring_tag
    std::vector<unsigned int> ring_tag;
    unsigned int next_ring_tag = 0;
    int nslots = 0;  // frame ring slots: max(mhat_z + 2, Mz + 1) (async upload spare; naive window)
    bool naive = false;  // spectrum backend: false = recursive (observer), true = naive window DFT
    int naive_grid = 0;
    // async submit/wait (cw_submit): upload / download streams and per-frame events
    cudaStream_t up = nullptr, down = nullptr;
    static constexpr int NEV = 8;
    cudaEvent_t ev_up[NEV] = {}, ev_k[NEV] = {}, ev_down[NEV] = {};
    cudaEvent_t ev_join = nullptr;  // cw_join
    int ready_of[NEV] = {};
    long long fidx_of[NEV] = {};
    bool dl_flagged[NEV] = {};  // chained cw_submit: the frame's download is followed by a flag write
    bool dl_any[NEV] = {};      // the frame's outputs were downloaded on `down` (its output set is busy)
    // detection epilogue: 2 device sets (double-buffered like the outputs),
    // NEV pinned host mirrors (one per outstanding frame)
    float det_tau = 0.f;
    int det_cap = 0;
    bool det_on = false;
    unsigned char *d_det = nullptr, *h_det = nullptr;
    // pageable frames given to cw_push are staged here (pinned, multithreaded copy)
    float *h_stage = nullptr;
    cudaEvent_t ev_stage = nullptr;  // the last upload from h_stage
    size_t det_bytes = 0;
    size_t state_floats = 0, that_floats = 0;  // floats (pairs x 2)
    long long frames_seen = 0;
    bool have_that = false;
    int forced_ix = -1, forced_iy = -1;
    // optional per-launch timing: events recorded around each frame kernel
    bool timing = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::string err;
};

// frame chaining applies to the fused kernel with the recursive backend;
// the in-kernel ring fill needs the delayed frame two launches back or more
static bool chained(const cw_handle *h) { return h->chain && !h->generic && !h->naive && h->mhz >= 2; }

#ifndef CW_RESIDENT_CE
#define CW_RESIDENT_CE 1  // resident frames' ring copies on the copy engine (0: in the kernel prologue)
#endif

static int fail(cw_handle *h, int code, const std::string &msg)
{
    if (h)
        h->err = msg;
    else
        g_create_error = msg;
    return code;
}

// Binds the handle's device for the duration of an ABI call and restores the
// caller's current device on exit: streams, events and lazily allocated
// buffers belong to h->device, and a launch into a stream of another device
// fails, so every call that launches, copies, allocates or waits binds it
// (pipelines on several GPUs may be driven from one thread).
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(const cw_handle *h) : DeviceGuard(h ? h->device : -1) {}
    explicit DeviceGuard(int device)
    {
        if (device >= 0 && cudaGetDevice(&prev) == cudaSuccess && prev != device)
            cudaSetDevice(device);
        else
            prev = -1;
    }
    ~DeviceGuard()
    {
        if (prev >= 0)
            cudaSetDevice(prev);
    }
};

#define CW_CUDA(h, expr)                                                                  \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess)                                                            \
            return fail((h), CW_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(_e)); \
    } while (0)

// detection buffer: 64-byte header + one f64 sum of squares per (row, block)
static size_t det_head_bytes(const cw_handle *h) { return 64 + 8 * (size_t)h->H * h->NXB; }

// validate(): the subset of params.py:114-158 that the device path relies on
// (the Python host layer runs the full rule set with the reference messages).
static int check_params(const cw_params *p, int W, int H, std::string *msg)
{
    char buf[256];
    if (p->kx < 1 || p->ky < 1 || p->kz < 1) {
        *msg = "half-window sizes must be >= 1";
        return CW_ERR_PARAM;
    }
    if (p->bx < 0 || p->bx >= p->kx || p->by < 0 || p->by >= p->ky) {
        *msg = "bandwidth must satisfy B < K";
        return CW_ERR_PARAM;
    }
    const int m[3] = {2 * p->kx + 1, 2 * p->ky + 1, 2 * p->kz + 1};
    for (int i = 0; i < 3; i++)
        if (p->mhat[i] < 0 || p->mhat[i] > m[i] - 1) {
            snprintf(buf, sizeof buf, "group delay component %d outside window [0, %d]", p->mhat[i], m[i] - 1);
            *msg = buf;
            return CW_ERR_PARAM;
        }
    if (!(p->alpha > 0.0 && p->alpha < 1.0)) {
        *msg = "smoothing pole must be in (0,1)";
        return CW_ERR_PARAM;
    }
    if (p->n_lag_x < 1 || p->n_lag_y < 1 || p->n_lag_x > 65535 || p->n_lag_y > 65535 || !p->lag_x || !p->lag_y) {
        *msg = "lag grids must hold 1..65535 entries";
        return CW_ERR_UNSUPPORTED;
    }
    if (W < m[0] || H < m[1]) {
        snprintf(buf, sizeof buf, "image %dx%d smaller than analysis window %dx%d", W, H, m[0], m[1]);
        *msg = buf;
        return CW_ERR_PARAM;
    }
    return CW_OK;
}

// Float tables for the fused kernel (double-precision construction).
//  x/y phase tables: spectrum.py:65-74; autocorr tables: flow.py:87-97;
//  pick gains: flow.py:147-163; pick tie order: _kernels.py:286-298.
static void build_tables(cw_handle *h)
{
    Tables &t = h->tab;
    std::memset(&t, 0, sizeof t);
    const double PI = 3.14159265358979323846;
    const int Mx = h->mx, My = h->my, Mz = h->mz;
    for (int k = 0; k <= h->kx; k++)
        for (int m = 0; m < Mx; m++) {
            t.exc[k][m] = (float)std::cos(2 * PI * k * m / Mx);
            t.exs[k][m] = (float)std::sin(2 * PI * k * m / Mx);
            t.ex2[k][m] = make_float2(t.exc[k][m], t.exs[k][m]);
        }
    for (int k = 0; k <= h->ky; k++) {
        for (int m = 0; m < My; m++) {
            t.eyc[k][m] = (float)std::cos(2 * PI * k * m / My);
            t.eys[k][m] = (float)std::sin(2 * PI * k * m / My);
        }
        t.twc[k] = (float)std::cos(2 * PI * k / My);
        t.tws[k] = (float)std::sin(2 * PI * k / My);
        t.tw2[k] = make_float2(t.twc[k], t.tws[k]);
        t.twn2[k] = make_float2(-t.tws[k], t.twc[k]);
    }
    // S = norm * z+; the three unscaled Hann passes each scale by 4, so
    // P = |C|^2 = norm^2 / 4^6 |C_unscaled|^2: fold into the kz collapse.
    const double norm = 1.0 / std::sqrt((double)Mx * My * Mz);
    const double pscale = norm * norm / 4096.0;
    for (int i = 0; i < Mz; i++) {
        const int kz = i - h->kz;
        t.wc[i] = (float)std::cos(2 * PI * kz / Mz);
        t.ws[i] = (float)std::sin(2 * PI * kz / Mz);
        t.azc[i] = (float)(pscale * std::cos(2 * PI * kz / Mz));
        t.azs[i] = (float)(-pscale * std::sin(2 * PI * kz / Mz));
        t.w2[i] = make_float2(t.wc[i], t.ws[i]);
        t.wn2[i] = make_float2(-t.ws[i], t.wc[i]);
        t.az2[i] = make_float2(t.azc[i], t.azs[i]);
    }
    std::vector<double> gx(h->nlx), gy(h->nly);
    for (int i = 0; i < h->nlx; i++)
        gx[i] = 0.375 / (0.25 + 0.125 * std::cos(2 * PI * h->lag_x[i] / Mx));
    for (int i = 0; i < h->nly; i++)
        gy[i] = 0.375 / (0.25 + 0.125 * std::cos(2 * PI * h->lag_y[i] / My));
    // stage 1: e^{-j 2 pi kx lx / Mx} = cos - j sin, gx folded
    for (int l = 0; l < h->nlx; l++) {
        t.s1v[l].gain = (float)gx[l];
        for (int k = 1; k <= h->kx; k++) {
            const double th = 2 * PI * k * h->lag_x[l] / Mx;
            t.s1v[l].cs[k - 1].x = (float)(gx[l] * std::cos(th));
            t.s1v[l].cs[k - 1].y = (float)(gx[l] * std::sin(th));
        }
    }
    // stage 2: R = B0 + 2 sum_ky (cos phi Re B + sin phi Im B), gy folded
    for (int l = 0; l < h->nly; l++) {
        t.s2v[l].gain = (float)gy[l];
        for (int k = 1; k <= h->ky; k++) {
            const double ph = 2 * PI * k * h->lag_y[l] / My;
            t.s2v[l].cs[k - 1].x = (float)(2.0 * gy[l] * std::cos(ph));
            t.s2v[l].cs[k - 1].y = (float)(2.0 * gy[l] * std::sin(ph));
        }
    }
    // rank: sort by (lag_x^2 + lag_y^2, ix, iy) -- the reference tie order
    std::vector<int> order(h->nlx * h->nly);
    for (int i = 0; i < (int)order.size(); i++)
        order[i] = i;  // i = iy * nlx + ix
    auto n2 = [&](int i) {
        const int ix = i % h->nlx, iy = i / h->nlx;
        return h->lag_x[ix] * h->lag_x[ix] + h->lag_y[iy] * h->lag_y[iy];
    };
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        const double na = n2(a), nb = n2(b);
        if (na != nb)
            return na < nb;
        const int ax = a % h->nlx, bx = b % h->nlx;
        if (ax != bx)
            return ax < bx;
        return a / h->nlx < b / h->nlx;
    });
    for (int rk = 0; rk < (int)order.size(); rk++) {
        const int i = order[rk];
        t.rank[i] = (uint16_t)rk;
        t.rix[rk] = (uint8_t)(i % h->nlx);
        t.riy[rk] = (uint8_t)(i / h->nlx);
    }
    t.norm = (float)norm;
    t.inv_mz = (float)(1.0 / Mz);
    // +-lag pairing needs an odd grid symmetric about an exact 0
    auto symmetric = [](const std::vector<double> &g) {
        const int n = (int)g.size();
        if (n % 2 == 0 || g[n / 2] != 0.0)
            return 0;
        for (int i = 0; i < n / 2; i++)
            if (g[i] != -g[n - 1 - i])
                return 0;
        return 1;
    };
    t.sym_x = symmetric(h->lag_x);
    t.sym_y = symmetric(h->lag_y);
    t.alpha = (float)h->alpha;
    t.beta = (float)(1.0 - h->alpha);
    t.nlx = h->nlx;
    t.nly = h->nly;
}

// Device tables of the runtime-geometry path (cw_generic.cuh): built in
// double, stored as float (spectrum.py:65-74, flow.py:87-97, flow.py:147-163,
// _kernels.py:286-298, design.py:256-274).
static int build_generic(cw_handle *h, const float *bank, const int64_t *retained, int nret)
{
    const double PI = 3.14159265358979323846;
    const int Mx = h->mx, My = h->my, Mz = h->mz, nlx = h->nlx, nly = h->nly, nl = nlx * nly;
    const int nb = Mx * My * Mz;
    const double nbd = (double)nb, norm = 1.0 / std::sqrt(nbd);
    std::vector<float2> ex(Mx * Mx), ey(My * My), ez(Mz * Mz), w(Mz), az(Mz), axl((size_t)nlx * Mx),
        ayl((size_t)nly * My), coef((size_t)nl * nret);
    auto cis = [](double th, double scale) { return make_float2((float)(scale * std::cos(th)), (float)(scale * std::sin(th))); };
    for (int k = 0; k < Mx; k++)
        for (int m = 0; m < Mx; m++)
            ex[k * Mx + m] = cis(2 * PI * (k - h->kx) * m / Mx, 1.0);
    for (int k = 0; k < My; k++)
        for (int m = 0; m < My; m++)
            ey[k * My + m] = cis(2 * PI * (k - h->ky) * m / My, 1.0);
    for (int k = 0; k < Mz; k++) {
        for (int m = 0; m < Mz; m++)
            ez[k * Mz + m] = cis(2 * PI * (k - h->kz) * m / Mz, 1.0);
        w[k] = cis(2 * PI * (k - h->kz) / Mz, 1.0);
        az[k] = cis(-2 * PI * (k - h->kz) / Mz, 1.0 / nbd);
    }
    for (int l = 0; l < nlx; l++) {
        const double g = 0.375 / (0.25 + 0.125 * std::cos(2 * PI * h->lag_x[l] / Mx));
        for (int k = 0; k < Mx; k++)
            axl[(size_t)l * Mx + k] = cis(-2 * PI * (k - h->kx) * h->lag_x[l] / Mx, g);
    }
    for (int l = 0; l < nly; l++) {
        const double g = 0.375 / (0.25 + 0.125 * std::cos(2 * PI * h->lag_y[l] / My));
        for (int k = 0; k < My; k++)
            ayl[(size_t)l * My + k] = cis(-2 * PI * (k - h->ky) * h->lag_y[l] / My, g);
    }
    std::vector<int> order(nl);
    for (int i = 0; i < nl; i++)
        order[i] = i;
    auto n2 = [&](int i) { return h->lag_x[i % nlx] * h->lag_x[i % nlx] + h->lag_y[i / nlx] * h->lag_y[i / nlx]; };
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        const double na = n2(a), nb2 = n2(b);
        if (na != nb2)
            return na < nb2;
        if (a % nlx != b % nlx)
            return a % nlx < b % nlx;
        return a / nlx < b / nlx;
    });
    std::vector<uint32_t> rank(nl), rix(nl), riy(nl);
    for (int rk = 0; rk < nl; rk++) {
        rank[order[rk]] = rk;
        rix[rk] = order[rk] % nlx;
        riy[rk] = order[rk] / nlx;
    }
    std::vector<int32_t> ret(nret);
    for (int j = 0; j < nret; j++) {
        if (retained[j] < 0 || retained[j] >= nb)
            return CW_ERR_VALUE;
        ret[j] = (int32_t)retained[j];
    }
    for (size_t i = 0; i < (size_t)nl * nret; i++)
        coef[i] = make_float2((float)(norm * bank[2 * i]), (float)(norm * bank[2 * i + 1]));
    // one device block, 16-byte aligned pieces
    std::vector<unsigned char> blob;
    std::vector<size_t> off;
    auto put = [&](const void *src, size_t bytes) {
        off.push_back(blob.size());
        blob.insert(blob.end(), (const unsigned char *)src, (const unsigned char *)src + bytes);
        blob.resize((blob.size() + 15) / 16 * 16);
    };
    put(ex.data(), ex.size() * 8);
    put(ey.data(), ey.size() * 8);
    put(ez.data(), ez.size() * 8);
    put(w.data(), w.size() * 8);
    put(az.data(), az.size() * 8);
    put(axl.data(), axl.size() * 8);
    put(ayl.data(), ayl.size() * 8);
    put(rank.data(), rank.size() * 4);
    put(rix.data(), rix.size() * 4);
    put(riy.data(), riy.size() * 4);
    put(coef.data(), coef.size() * 8);
    put(ret.data(), ret.size() * 4);
    CW_CUDA(h, cudaMalloc(&h->d_gtab, blob.size()));
    CW_CUDA(h, cudaMemcpy(h->d_gtab, blob.data(), blob.size(), cudaMemcpyHostToDevice));
    const unsigned char *b = static_cast<const unsigned char *>(h->d_gtab);
    GenTables &t = h->gt;
    t.ex = reinterpret_cast<const float2 *>(b + off[0]);
    t.ey = reinterpret_cast<const float2 *>(b + off[1]);
    t.ez = reinterpret_cast<const float2 *>(b + off[2]);
    t.w = reinterpret_cast<const float2 *>(b + off[3]);
    t.az = reinterpret_cast<const float2 *>(b + off[4]);
    t.axl = reinterpret_cast<const float2 *>(b + off[5]);
    t.ayl = reinterpret_cast<const float2 *>(b + off[6]);
    t.rank = reinterpret_cast<const uint32_t *>(b + off[7]);
    t.rix = reinterpret_cast<const uint32_t *>(b + off[8]);
    t.riy = reinterpret_cast<const uint32_t *>(b + off[9]);
    t.coef = reinterpret_cast<const float2 *>(b + off[10]);
    t.ret = reinterpret_cast<const int32_t *>(b + off[11]);
    return CW_OK;
}

// x-stage planes for nf frames (1: recursive backend, Mz: naive)
static int ensure_xf(cw_handle *h, int nf)
{
    if (h->nxf >= nf)
        return CW_OK;
    cudaFree(h->d_xf);
    h->d_xf = nullptr;
    h->nxf = 0;
    const size_t bytes = (size_t)nf * h->mx * h->W * h->H * sizeof(float2);
    CW_CUDA(h, cudaMalloc(&h->d_xf, bytes));
    CW_CUDA(h, cudaMemset(h->d_xf, 0, bytes));
    h->nxf = nf;
    return CW_OK;
}

// PEF coefficients on the stored half space (pipeline.py:269-282,
// _kernels.py:330-342): pred = Re sum_k c(k) S(k) over the retained band,
// folded so that the kernel computes sum_j coef[j] * z+[j] with
// S = norm * z+, pairing k with -k: Re(c S) + Re(c' conj S)
//   = S.re (c.re + c'.re) + S.im (c'.im - c.im).
static int build_coef(cw_handle *h, const float *bank, const int64_t *retained, int nret,
                      std::vector<float> *out)
{
    const int Mx = h->mx, My = h->my, Mz = h->mz, KX = h->kx, KY = h->ky, KZ = h->kz;
    const int BX = h->bx, BY = h->by;
    const int WX = 2 * BX + 1;
    // map reference flat bin -> coefficient position j
    std::vector<int> pos(Mx * My * Mz, -1);
    for (int j = 0; j < nret; j++) {
        if (retained[j] < 0 || retained[j] >= Mx * My * Mz)
            return CW_ERR_VALUE;
        pos[retained[j]] = j;
    }
    auto flat = [&](int kz, int ky, int kx) { return ((kz + KZ) * My + (ky + KY)) * Mx + (kx + KX); };
    // the kernel holds z+ = Mz xhat+ (unnormalised DFT), S = norm * z+
    const double cS = 1.0 / std::sqrt((double)Mx * My * Mz);
    // float2 pairs per velocity, in the kernel's retained z+ order:
    // row 0: DC (kz = 0 real + zero pad, kz = 1..KZ), kx = 1..BX (all kz);
    // rows ky = 1..BY: kx = -BX..BX (all kz)
    // rows padded to even pair counts (zero pad pairs) for the kernel's
    // 16-byte two-pair loads (Geo::RETPP)
    const int P0 = (KZ + 1) + BX * Mz, PN = WX * Mz;
    const int P0p = (P0 + 1) / 2 * 2, PNp = (PN + 1) / 2 * 2;
    const int NRET = 2 * (P0p + BY * PNp);
    out->assign((size_t)h->nlx * h->nly * NRET, 0.f);
    for (int v = 0; v < h->nlx * h->nly; v++) {
        const float *bk = bank + (size_t)v * nret * 2;
        auto coef = [&](int kz, int ky, int kx, double *re, double *im) -> bool {
            const int j = pos[flat(kz, ky, kx)];
            if (j < 0)
                return false;
            *re = bk[2 * j];
            *im = bk[2 * j + 1];
            return true;
        };
        float *o = out->data() + (size_t)v * NRET;
        int w = 0;
        // pred += p.x z.r + p.y z.i = Re(k z), k = (p.x, -p.y); a kernel that
        // reads the stored (rotated) state z = w z+ instead of z+ gets
        // k conj(w(kz)) (fold_w)
        const double PI = 3.14159265358979323846;
        auto put = [&](int kz, double px, double py) {
            if (h->fn.pef_l2 && kz != 0) {
                const double wr = std::cos(2 * PI * kz / Mz), wi = std::sin(2 * PI * kz / Mz);
                const double kr = px, ki = -py;  // k conj(w)
                const double nr = kr * wr + ki * wi, ni = ki * wr - kr * wi;
                px = nr;
                py = -ni;
            }
            o[w++] = (float)px;
            o[w++] = (float)py;
        };
        auto pair = [&](int kz, int ky, int kx) -> bool {
            double cr, ci, dr, di;
            if (!coef(kz, ky, kx, &cr, &ci) || !coef(-kz, -ky, -kx, &dr, &di))
                return false;
            put(kz, cS * (cr + dr), cS * (di - ci));
            return true;
        };
        // row 0: DC bin (kz = 0 real, kz = 1..KZ), then kx = 1..BX, all kz
        double cr, ci;
        if (!coef(0, 0, 0, &cr, &ci))
            return CW_ERR_VALUE;
        o[w++] = (float)(cS * cr);
        o[w++] = 0.f;  // pad: the DC kz = 0 state is real
        for (int kz = 1; kz <= KZ; kz++)
            if (!pair(kz, 0, 0))
                return CW_ERR_VALUE;
        for (int kx = 1; kx <= BX; kx++)
            for (int kz = -KZ; kz <= KZ; kz++)
                if (!pair(kz, 0, kx))
                    return CW_ERR_VALUE;
        w = 2 * P0p;  // pad pair stays zero
        for (int ky = 1; ky <= BY; ky++) {
            for (int kx = -BX; kx <= BX; kx++)
                for (int kz = -KZ; kz <= KZ; kz++)
                    if (!pair(kz, ky, kx))
                        return CW_ERR_VALUE;
            w = 2 * (P0p + ky * PNp);
        }
        if (w != NRET)
            return CW_ERR_VALUE;
    }
    return CW_OK;
}

extern "C" {

int32_t cw_abi_version(void) { return CW_ABI_VERSION; }

const char *cw_last_error(const cw_handle *h) { return h ? h->err.c_str() : g_create_error.c_str(); }

int cw_create(const cw_params *p, int32_t width, int32_t height, int32_t device, const float *bank_c64,
              const int64_t *retained, int32_t n_retained, int32_t halo_rows, int32_t row_offset,
              cw_handle **out)
{
    if (!out || !p)
        return fail(nullptr, CW_ERR_VALUE, "null argument");
    *out = nullptr;
    std::string msg;
    int rc = check_params(p, width, height, &msg);
    if (rc != CW_OK)
        return fail(nullptr, rc, msg);
    // symmetric odd grids with an exact 0 get the unrolled +-lag kernels
    auto sym = [](const double *g, int n) {
        if (n % 2 == 0 || g[n / 2] != 0.0)
            return false;
        for (int i = 0; i < n / 2; i++)
            if (g[i] != -g[n - 1 - i])
                return false;
        return true;
    };
    const int nl_sym = (p->n_lag_x == p->n_lag_y && sym(p->lag_x, p->n_lag_x) && sym(p->lag_y, p->n_lag_y))
                           ? p->n_lag_x
                           : 0;
    // the fused kernel when a compiled instance covers the geometry and the
    // lag grids fit its tables; the runtime-geometry path otherwise (or when
    // CW_FORCE_GENERIC=1, for testing it on the compiled geometries)
    LaunchFn fn{};
    const char *force = std::getenv("CW_FORCE_GENERIC"), *nojit = std::getenv("CW_NO_JIT");
    const bool force_generic = force && force[0] == '1';
    int kind = 0;
    bool have = !force_generic && p->n_lag_x <= MAXL && p->n_lag_y <= MAXL &&
                find_inst(p->kx, p->ky, p->kz, p->bx, p->by, nl_sym, &fn);
    if (!have && !force_generic && !(nojit && nojit[0] == '1') &&
        jit_supported(p->kx, p->ky, p->kz, p->bx, p->by, p->n_lag_x, p->n_lag_y)) {
        std::string jerr;  // no NVRTC / compile failure: the runtime-geometry kernels run instead
        have = jit_instance(p->kx, p->ky, p->kz, p->bx, p->by, nl_sym, &fn, &jerr);
        kind = 1;
    }
    const bool generic = !have;
    if (generic)
        kind = 2;
    const int nret_expect = (2 * p->kz + 1) * (2 * p->bx + 1) * (2 * p->by + 1);
    if (n_retained != nret_expect || !bank_c64 || !retained)
        return fail(nullptr, CW_ERR_VALUE, "bank does not match the retained band of these parameters");
    if (halo_rows < 0 || halo_rows >= height || row_offset < 0)
        return fail(nullptr, CW_ERR_VALUE, "bad strip geometry");

    cw_handle *h = new cw_handle();
    h->kx = p->kx;
    h->ky = p->ky;
    h->kz = p->kz;
    h->bx = p->bx;
    h->by = p->by;
    h->mhx = p->mhat[0];
    h->mhy = p->mhat[1];
    h->mhz = p->mhat[2];
    h->mx = 2 * p->kx + 1;
    h->my = 2 * p->ky + 1;
    h->mz = 2 * p->kz + 1;
    h->W = width;
    h->H = height;
    h->NXB = (width + 31) / 32;
    h->halo = halo_rows;
    h->row_off = row_offset;
    h->device = device;
    h->nlx = p->n_lag_x;
    h->nly = p->n_lag_y;
    h->alpha = p->alpha;
    h->lag_x.assign(p->lag_x, p->lag_x + p->n_lag_x);
    h->lag_y.assign(p->lag_y, p->lag_y + p->n_lag_y);
    h->fn = fn;
    h->generic = generic;
    h->kind = kind;
    h->idx_bytes = (h->nlx > 256 || h->nly > 256) ? 2 : 1;
    std::vector<float> coef;
    if (!generic) {
        g_phase_clocks = fn.phase_clocks;
        build_tables(h);
        rc = build_coef(h, bank_c64, retained, n_retained, &coef);
        if (rc != CW_OK) {
            delete h;
            return fail(nullptr, rc, "bank/retained layout inconsistent with the parameters");
        }
        if (coef.size() != (size_t)h->nlx * h->nly * 2 * fn.retp) {  // host layout == kernel's padded rows
            delete h;
            return fail(nullptr, CW_ERR_UNSUPPORTED, "PEF coefficient layout does not match the kernel instance");
        }
    }

    auto cleanup_fail = [&](int code, const std::string &m) {
        std::string keep = h->err.empty() ? m : h->err;
        cw_destroy(h);
        return fail(nullptr, code, keep);
    };
    DeviceGuard dg(-1);  // restores the caller's current device on return
    if (cudaGetDevice(&dg.prev) != cudaSuccess || cudaSetDevice(device) != cudaSuccess)
        return cleanup_fail(CW_ERR_CUDA, "cudaSetDevice failed (no CUDA device?)");
    if (cudaStreamCreateWithFlags(&h->own, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup_fail(CW_ERR_CUDA, "cudaStreamCreate failed");
    int occ = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (!generic) {
        if (cudaFuncSetAttribute(fn.kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fn.smem) != cudaSuccess)
            return cleanup_fail(CW_ERR_CUDA, "cannot reserve shared memory for the frame kernel");
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn.kernel, fn.threads, fn.smem);
        if (occ < 1 || sms < 1)
            return cleanup_fail(CW_ERR_CUDA, "frame kernel cannot be resident on this device");
        const long long units = (long long)h->NXB * (height - halo_rows);
        long long slots = (long long)occ * sms;
        if (const char *e = std::getenv("CW_GRID_X"))  // experiment knob: CTAs per resident slot
            slots = std::max<long long>(1, (long long)(std::atof(e) * (double)slots));
        h->grid = (int)std::min<long long>(slots, std::max<long long>(1, units / 2));
    }
    h->sms = std::max(1, sms);

    const size_t pix_packets = (size_t)height * h->NXB;
    const size_t HW = (size_t)width * height;
    if (generic) {  // [plane][pixel] float2: full spectrum z+, T^ (My x Mx)
        h->state_floats = HW * h->mx * h->my * h->mz * 2;
        h->that_floats = HW * h->mx * h->my * 2;
        if (build_generic(h, bank_c64, retained, n_retained) != CW_OK || ensure_xf(h, 1) != CW_OK)
            return cleanup_fail(CW_ERR_NOMEM, "runtime-geometry tables / buffers: " + h->err);
    } else {
        h->state_floats = pix_packets * fn.nsp * 32 * 2;
        h->that_floats = pix_packets * fn.ntp * 32 * 2;
    }
    if (cudaMalloc(&h->d_state, h->state_floats * 4) != cudaSuccess ||
        cudaMalloc(&h->d_that, h->that_floats * 4) != cudaSuccess ||
        (!generic && cudaMalloc(&h->d_coef, coef.size() * 4) != cudaSuccess) ||
        cudaMalloc(&h->d_frames, HW * 4 * std::max(h->mhz + 2, h->mz + 1)) != cudaSuccess ||
        cudaMalloc(&h->d_res, HW * 4 * 2) != cudaSuccess || cudaMalloc(&h->d_pred, HW * 4 * 2) != cudaSuccess ||
        cudaMalloc(&h->d_vidx, HW * 2 * 2 * h->idx_bytes) != cudaSuccess)
        return cleanup_fail(CW_ERR_NOMEM, "device allocation failed");
    cudaMemsetAsync(h->d_state, 0, h->state_floats * 4, h->own);
    cudaMemsetAsync(h->d_that, 0, h->that_floats * 4, h->own);
    h->nslots = std::max(h->mhz + 2, h->mz + 1);
    h->ring_tag.assign(h->nslots, 0u);
    cudaMemsetAsync(h->d_frames, 0, HW * 4 * h->nslots, h->own);
    cudaMemsetAsync(h->d_res, 0, HW * 4 * 2, h->own);
    cudaMemsetAsync(h->d_pred, 0, HW * 4 * 2, h->own);
    cudaMemsetAsync(h->d_vidx, 0, HW * 2 * 2 * h->idx_bytes, h->own);
    if (cudaStreamCreateWithFlags(&h->up, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->down, cudaStreamNonBlocking) != cudaSuccess)
        return cleanup_fail(CW_ERR_CUDA, "cudaStreamCreate failed");
    for (int i = 0; i < cw_handle::NEV; i++)
        if (cudaEventCreateWithFlags(&h->ev_up[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_k[i], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev_down[i], cudaEventDisableTiming) != cudaSuccess)
            return cleanup_fail(CW_ERR_CUDA, "cudaEventCreate failed");
    if (cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess)
        return cleanup_fail(CW_ERR_CUDA, "cudaEventCreate failed");
    if (!generic)
        cudaMemcpyAsync(h->d_coef, coef.data(), coef.size() * 4, cudaMemcpyHostToDevice, h->own);
    if (const char *e = std::getenv("CW_DYN_STATIC"))  // tuning knobs (tools/ab_kernel.py)
        h->dyn_static = std::atof(e);
    if (const char *e = std::getenv("CW_DYN_CHUNK"))
        h->dyn_chunk = std::max(1, std::atoi(e));
    if (const char *e = std::getenv("CW_CHAIN"))
        h->chain = std::atoi(e) != 0;
    if (cudaMalloc(&h->d_work, 2 * sizeof(unsigned int)) != cudaSuccess ||
        cudaMalloc(&h->d_done, sizeof(unsigned int) * std::max(1, h->grid)) != cudaSuccess)
        return cleanup_fail(CW_ERR_NOMEM, "device allocation failed");
    cudaMemsetAsync(h->d_done, 0, sizeof(unsigned int) * std::max(1, h->grid), h->own);
    {
        void *fp = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (!std::getenv("CW_NO_MEMOPS") &&  // (test knob: the event-wait fallback)
            cudaGetDriverEntryPoint("cuStreamWriteValue32", &fp, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess && fp && cudaMalloc(&h->d_flags, 3 * sizeof(unsigned int)) == cudaSuccess) {
            h->write_value = reinterpret_cast<decltype(h->write_value)>(fp);
            cudaMemsetAsync(h->d_flags, 0, 3 * sizeof(unsigned int), h->own);
        }
        cudaGetLastError();
    }
    if (!generic && fn.compact) {  // the rank tables the compact instance reads from global memory
        const int nl = h->nlx * h->nly;
        std::vector<unsigned char> rk((size_t)nl * 4);
        std::memcpy(rk.data(), h->tab.rank, (size_t)nl * 2);
        for (int i = 0; i < nl; i++) {
            rk[(size_t)nl * 2 + 2 * i] = h->tab.rix[i];
            rk[(size_t)nl * 2 + 2 * i + 1] = h->tab.riy[i];
        }
        if (cudaMalloc(&h->d_rank, rk.size()) != cudaSuccess ||
            cudaMemcpy(h->d_rank, rk.data(), rk.size(), cudaMemcpyHostToDevice) != cudaSuccess)
            return cleanup_fail(CW_ERR_NOMEM, "device allocation failed");
    }
    cudaMemsetAsync(h->d_work, 0, 2 * sizeof(unsigned int), h->own);
    if (cudaStreamSynchronize(h->own) != cudaSuccess)
        return cleanup_fail(CW_ERR_CUDA, "device initialisation failed");
    *out = h;
    return CW_OK;
}

void cw_destroy(cw_handle *h)
{
    DeviceGuard dg(h);
    if (!h)
        return;
    if (h->own)
        cudaStreamSynchronize(h->own);
    cudaFree(h->d_state);
    cudaFree(h->d_that);
    cudaFree(h->d_coef);
    cudaFree(h->d_frames);
    cudaFree(h->d_raw);
    cudaFree(h->d_res);
    cudaFree(h->d_pred);
    cudaFree(h->d_vidx);
    cudaFree(h->d_gtab);
    cudaFree(h->d_work);
    cudaFree(h->d_done);
    cudaFree(h->d_flags);
    cudaFree(h->d_rank);
    cudaFree(h->d_xf);
    cudaFree(h->d_det);
    if (h->h_det)
        cudaFreeHost(h->h_det);
    if (h->ev_stage) {
        cudaEventSynchronize(h->ev_stage);
        cudaEventDestroy(h->ev_stage);
    }
    if (h->h_stage)
        cudaFreeHost(h->h_stage);
    for (cudaEvent_t e : h->ev_pool)
        cudaEventDestroy(e);
    for (int i = 0; i < cw_handle::NEV; i++) {
        if (h->ev_up[i]) cudaEventDestroy(h->ev_up[i]);
        if (h->ev_k[i]) cudaEventDestroy(h->ev_k[i]);
        if (h->ev_down[i]) cudaEventDestroy(h->ev_down[i]);
    }
    if (h->ev_join) {
        cudaEventDestroy(h->ev_join);
    }
    if (h->up) {
        cudaStreamSynchronize(h->up);
        cudaStreamDestroy(h->up);
    }
    if (h->down) {
        cudaStreamSynchronize(h->down);
        cudaStreamDestroy(h->down);
    }
    if (h->own)
        cudaStreamDestroy(h->own);
    delete h;
}

int cw_set_forced_velocity(cw_handle *h, int32_t ix, int32_t iy)
{
    if (!h)
        return CW_ERR_VALUE;
    if (ix < 0 || iy < 0) {
        h->forced_ix = h->forced_iy = -1;
        return CW_OK;
    }
    if (ix >= h->nlx || iy >= h->nly)
        return fail(h, CW_ERR_PARAM, "forced velocity index outside the grid");
    h->forced_ix = ix;
    h->forced_iy = iy;
    return CW_OK;
}

int64_t cw_frames_seen(const cw_handle *h) { return h ? h->frames_seen : -1; }

int32_t cw_index_bytes(const cw_handle *h) { return h ? h->idx_bytes : -1; }

int32_t cw_is_generic(const cw_handle *h) { return h ? (h->generic ? 1 : 0) : -1; }

int32_t cw_kernel_kind(const cw_handle *h) { return h ? h->kind : -1; }

int cw_jit_prebuild(const cw_params *p, const char *dir)
{
    if (!p || !dir)
        return fail(nullptr, CW_ERR_VALUE, "null argument");
    auto sym = [](const double *g, int n) {
        if (n % 2 == 0 || g[n / 2] != 0.0)
            return false;
        for (int i = 0; i < n / 2; i++)
            if (g[i] != -g[n - 1 - i])
                return false;
        return true;
    };
    const int nl = (p->n_lag_x == p->n_lag_y && sym(p->lag_x, p->n_lag_x) && sym(p->lag_y, p->n_lag_y)) ? p->n_lag_x : 0;
    if (!jit_supported(p->kx, p->ky, p->kz, p->bx, p->by, p->n_lag_x, p->n_lag_y))
        return fail(nullptr, CW_ERR_UNSUPPORTED, "geometry beyond the fused kernel (runtime-geometry path)");
    std::string err;
    if (jit_prebuild(p->kx, p->ky, p->kz, p->bx, p->by, nl, dir, &err) != 0)
        return fail(nullptr, CW_ERR_UNSUPPORTED, err);
    return CW_OK;
}

int cw_next_frame_slot(cw_handle *h, float **slot)
{
    if (!h || !slot)
        return CW_ERR_VALUE;
    const size_t HW = (size_t)h->W * h->H;
    *slot = h->d_frames + (size_t)(h->frames_seen % h->nslots) * HW;
    return CW_OK;
}

static cudaStream_t pick_stream(cw_handle *h, void *stream)
{
    return stream ? reinterpret_cast<cudaStream_t>(stream) : h->own;
}

// The frame already sits in its ring slot: run the fused kernel.
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// Outputs go to the handle's double-buffered device set unless res_o /
// pred_o / vidx_o (device-addressable pointers, e.g. mapped host memory)
// override them.
struct FlagWants {
    unsigned int up_want, down_want;
};

static int run_frame(cw_handle *h, cudaStream_t s, int32_t *ready, int64_t *frame_index, float *res_o = nullptr,
                     float *pred_o = nullptr, uint8_t *vidx_o = nullptr, const float *frame_src = nullptr,
                     bool chain = false, const FlagWants *flags = nullptr, bool ring_fill = true)
{
    // chain: static split, and a programmatic dependent launch when the
    // previous fused launch was static too (done[] then names the same
    // units per CTA); otherwise a plain launch (full stream order), which
    // may use the dynamic tail
    chain = chain && chained(h);
    const bool pdl = chain && h->last_static;
    h->dl_flagged[h->frames_seen % cw_handle::NEV] = false;  // set again by a flagged cw_submit
    h->dl_any[h->frames_seen % cw_handle::NEV] = false;
    NvtxRange nvtx("cw_frame");
    const size_t HW = (size_t)h->W * h->H;
    const long long n = h->frames_seen;
    const int rd = (n + 1 >= h->mz) ? 1 : 0;
    FrameArgs a;
    a.frame = h->d_frames + (size_t)(n % h->nslots) * HW;
    a.delayed = rd ? h->d_frames + (size_t)((n - h->mhz) % h->nslots) * HW : nullptr;
    a.state = reinterpret_cast<float2 *>(h->d_state);
    a.that = reinterpret_cast<float2 *>(h->d_that);
    a.coefP = reinterpret_cast<const float2 *>(h->d_coef);
    const size_t set = (size_t)(n & 1);  // double-buffered outputs
    a.res = res_o ? res_o : h->d_res + set * HW;
    a.pred = pred_o ? pred_o : h->d_pred + set * HW;
    a.vidx = vidx_o ? vidx_o : h->d_vidx + set * HW * 2 * h->idx_bytes;
    a.W = h->W;
    a.H = h->H;
    a.NXB = h->NXB;
    a.y_begin = h->halo;
    a.y_off = h->row_off;
    a.ready = rd;
    a.first = (rd && !h->have_that) ? 1 : 0;
    a.forced_ix = h->forced_ix;
    a.forced_iy = h->forced_iy;
    a.mhx = h->mhx;
    a.mhy = h->mhy;
    {
        const long long units = (long long)h->NXB * (h->H - h->halo);
        const long long su = (long long)(h->dyn_static * (double)units);
        // dynamic chunks pay a run restart each: only for long per-CTA runs
        const bool dyn = !chain && h->dyn_static < 1.0 && su < units && units >= 20LL * h->grid;
        a.work = dyn ? h->d_work : nullptr;
        a.parity = (int)(n & 1);
        a.static_units = su < 0 ? 0 : su;
        a.dyn_chunk = h->dyn_chunk;
    }
    a.rank_g = reinterpret_cast<const uint16_t *>(h->d_rank);
    a.rxy_g = h->d_rank ? h->d_rank + (size_t)h->nlx * h->nly * 2 : nullptr;
    a.det = nullptr;
    a.done = h->d_done;
    a.seq = h->seq + 1;  // committed once the launch went in (a failed launch publishes no flags)
    a.ring_dst = nullptr;
    a.up_flag = a.down_flag = nullptr;
    a.up_want = a.down_want = 0;
    if (flags) {
        if (flags->up_want) {
            a.up_flag = h->d_flags;
            a.up_want = flags->up_want;
        }
        if (flags->down_want) {
            a.down_flag = h->d_flags + 1;
            a.down_want = flags->down_want;
        }
    }
    if (frame_src) {  // chained resident frame: the kernel reads the caller's frame (x stage) ...
        if (ring_fill)  // ... and fills its ring slot itself (else a copy-engine copy does, flagged)
            a.ring_dst = const_cast<float *>(a.frame);
        a.frame = frame_src;
    }
    // the delayed frame's slot, if a flagged copy filled it: wait for the flag
    a.ring_flag = nullptr;
    a.ring_want = 0;
    if (rd && h->d_flags) {
        const unsigned int tag = h->ring_tag[(size_t)((n - h->mhz) % h->nslots)];
        if (tag) {
            a.ring_flag = h->d_flags + 2;
            a.ring_want = tag;
        }
    }
    h->ring_tag[(size_t)(n % h->nslots)] = h->next_ring_tag;
    h->next_ring_tag = 0;
    a.det_tau = h->det_tau;
    a.det_cap = h->det_cap;
    if (h->det_on && rd) {
        a.det = h->d_det + set * h->det_bytes;
        CW_CUDA(h, cudaMemsetAsync(a.det, 0, det_head_bytes(h), s));
    }
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (h->timing) {
        while (h->ev_pool.size() < h->ev_used + 2) {
            cudaEvent_t e;
            CW_CUDA(h, cudaEventCreate(&e));
            h->ev_pool.push_back(e);
        }
        e0 = h->ev_pool[h->ev_used];
        e1 = h->ev_pool[h->ev_used + 1];
        h->ev_used += 2;
        CW_CUDA(h, cudaEventRecord(e0, s));
    }
    if (h->generic) {
        GenArgs g;
        g.frames = h->d_frames;
        g.nslots = h->nslots;
        g.n = n;
        g.delayed = a.delayed;
        g.xf = h->d_xf;
        g.state = reinterpret_cast<float2 *>(h->d_state);
        g.that = reinterpret_cast<float2 *>(h->d_that);
        g.res = a.res;
        g.pred = a.pred;
        g.vidx = a.vidx;
        g.idx16 = h->idx_bytes == 2;
        g.W = h->W;
        g.H = h->H;
        g.NXB = h->NXB;
        g.y_begin = h->halo;
        g.y_off = h->row_off;
        g.kx = h->kx;
        g.ky = h->ky;
        g.kz = h->kz;
        g.mx = h->mx;
        g.my = h->my;
        g.mz = h->mz;
        g.nb = h->mx * h->my * h->mz;
        g.nlx = h->nlx;
        g.nly = h->nly;
        g.nc = (2 * h->kz + 1) * (2 * h->bx + 1) * (2 * h->by + 1);
        g.mhx = h->mhx;
        g.mhy = h->mhy;
        g.ready = rd;
        g.first = a.first;
        g.naive = h->naive;
        g.forced_ix = h->forced_ix;
        g.forced_iy = h->forced_iy;
        g.alpha = (float)h->alpha;
        g.beta = (float)(1.0 - h->alpha);
        g.inv_mz = (float)(1.0 / h->mz);
        g.det = a.det;
        g.det_tau = a.det_tau;
        g.det_cap = a.det_cap;
        CW_CUDA(h, gen_launch(g, h->gt, h->sms, s));
    } else if (h->naive && rd) {
        // non-recursive spectrum of frames n-Mz+1 .. n into the state packets
        NaiveArgs na;
        na.frames = h->d_frames;
        na.nslots = h->nslots;
        na.n = n;
        na.state = reinterpret_cast<float2 *>(h->d_state);
        na.W = h->W;
        na.H = h->H;
        na.NXB = h->NXB;
        na.y_begin = h->halo;
        na.y_off = h->row_off;
        if (h->fn.launch_naive) {
            h->fn.launch_naive(na, h->tab, h->naive_grid, s);
        } else {
            void *args[] = {&na, &h->tab};
            CW_CUDA(h, cudaLaunchKernel(h->fn.naive_kernel, dim3(h->naive_grid), dim3(h->fn.threads), args,
                                        h->fn.naive_smem, s));
        }
        CW_CUDA(h, cudaGetLastError());
    }
    if (!h->generic) {
        if (pdl) {
            // programmatic dependent launch: may start while the previous
            // frame's kernel drains; the kernel orders itself per CTA (done[])
            void *args[] = {&a, &h->tab};
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(h->grid);
            cfg.blockDim = dim3(h->fn.threads);
            cfg.dynamicSmemBytes = h->fn.smem;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            CW_CUDA(h, cudaLaunchKernelExC(&cfg, h->fn.kernel, args));
        } else if (h->fn.launch) {
            h->fn.launch(a, h->tab, h->grid, s);
        } else {  // run-time compiled instance
            void *args[] = {&a, &h->tab};
            CW_CUDA(h, cudaLaunchKernel(h->fn.kernel, dim3(h->grid), dim3(h->fn.threads), args, h->fn.smem, s));
        }
        CW_CUDA(h, cudaGetLastError());
        h->last_static = a.work == nullptr;
        h->seq = a.seq;
    }
    CW_CUDA(h, cudaEventRecord(h->ev_k[n % cw_handle::NEV], s));  // ring-slot reuse order (resident copies)
    if (h->timing)
        CW_CUDA(h, cudaEventRecord(e1, s));
    if (a.det) {  // results to the pinned mirror of this frame (ordered on s)
        CW_CUDA(h, cudaMemcpyAsync(h->h_det + (size_t)(n % cw_handle::NEV) * h->det_bytes, a.det,
                                   h->det_bytes, cudaMemcpyDeviceToHost, s));
    }
    h->frames_seen = n + 1;
    if (rd)
        h->have_that = true;
    if (ready)
        *ready = rd;
    if (frame_index)
        *frame_index = rd ? n - h->mhz : -1;
    return CW_OK;
}

int cw_push_inplace(cw_handle *h, int32_t *ready, int64_t *frame_index, void *stream)
{
    DeviceGuard dg(h);
    if (!h)
        return CW_ERR_VALUE;
    return run_frame(h, pick_stream(h, stream), ready, frame_index);
}

int cw_push_device(cw_handle *h, const float *frame_dev, int32_t *ready, int64_t *frame_index, void *stream)
{
    DeviceGuard dg(h);
    if (!h || !frame_dev)
        return CW_ERR_VALUE;
    cudaStream_t s = pick_stream(h, stream);
    float *slot;
    cw_next_frame_slot(h, &slot);
    const size_t HW = (size_t)h->W * h->H;
    if (slot != frame_dev)
        CW_CUDA(h, cudaMemcpyAsync(slot, frame_dev, HW * 4, cudaMemcpyDeviceToDevice, s));
    return run_frame(h, s, ready, frame_index);
}

// Device address of page-locked host memory (UVA maps cudaHostAlloc /
// torch pin_memory buffers at their host address), else nullptr.
static void *mapped_host(const void *p)
{
    if (!p)
        return nullptr;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// cw_push's buffers must be host memory (device frames: cw_push_device)
static bool is_device_memory(const void *p)
{
    if (!p)
        return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice;
}

int cw_push(cw_handle *h, const float *frame, float *residual, float *prediction, uint8_t *vidx, int32_t *ready,
            int64_t *frame_index, void *stream)
{
    DeviceGuard dg(h);
    NvtxRange nvtx("cw_push");
    if (!h || !frame)
        return CW_ERR_VALUE;
    if (is_device_memory(frame) || is_device_memory(residual) || is_device_memory(prediction) ||
        is_device_memory(vidx))
        return fail(h, CW_ERR_VALUE, "cw_push takes host buffers (device frames: cw_push_device)");
    cudaStream_t s = pick_stream(h, stream);
    float *slot;
    cw_next_frame_slot(h, &slot);
    const size_t HW = (size_t)h->W * h->H;
    const float *src = frame;
    if (!mapped_host(frame)) {
        // pageable frame: a parallel copy into a pinned staging buffer, then
        // one DMA (the driver's own pageable path stages single-threaded)
        if (!h->h_stage) {
            CW_CUDA(h, cudaHostAlloc(reinterpret_cast<void **>(&h->h_stage), HW * 4, cudaHostAllocDefault));
            CW_CUDA(h, cudaEventCreateWithFlags(&h->ev_stage, cudaEventDisableTiming));
        } else {
            CW_CUDA(h, cudaEventSynchronize(h->ev_stage));  // previous upload done with the buffer
        }
#ifdef _OPENMP
        const int nt = std::max(1, std::min(8, omp_get_max_threads()));
#else
        const int nt = 1;
#endif
        // NPIECE pieces: the DMA of piece k overlaps the staging copy of k+1
        constexpr int NPIECE = 4;
        const size_t piece = (HW + NPIECE - 1) / NPIECE;
        for (int k = 0; k < NPIECE; k++) {
            const size_t p0 = k * piece, p1 = std::min(HW, p0 + piece);
            if (p0 >= p1)
                break;
            const long long chunk = ((long long)(p1 - p0) + nt - 1) / nt;
#pragma omp parallel for num_threads(nt) schedule(static)
            for (int t = 0; t < nt; t++) {
                const long long b = (long long)p0 + t * chunk, e = std::min((long long)p1, b + chunk);
                if (b < e)
                    std::memcpy(h->h_stage + b, frame + b, sizeof(float) * (size_t)(e - b));
            }
            CW_CUDA(h, cudaMemcpyAsync(slot + p0, h->h_stage + p0, (p1 - p0) * 4, cudaMemcpyHostToDevice, s));
        }
        src = h->h_stage;
    } else {
        CW_CUDA(h, cudaMemcpyAsync(slot, src, HW * 4, cudaMemcpyHostToDevice, s));
    }
    if (src == h->h_stage)
        CW_CUDA(h, cudaEventRecord(h->ev_stage, s));
    int32_t rd = 0;
    const size_t set = (size_t)(h->frames_seen & 1);
    const bool will_be_ready = h->frames_seen + 1 >= h->mz;
    // Direct outputs: when every requested output buffer is page-locked host
    // memory, the kernel writes residual / prediction / velocity straight
    // into it over PCIe while it runs (10 B per pixel, far below the link
    // rate), so no device-to-host copies follow the kernel.  The kernel
    // writes the valid output rectangle and every velocity pair; the
    // residual / prediction border outside valid_bounds (pipeline.py:41-50)
    // is zeroed here on the host.  Full frames only (no strip halo).
    float *res_d = nullptr, *pred_d = nullptr;
    uint8_t *vidx_d = nullptr;
    bool direct = will_be_ready && h->halo == 0 && h->row_off == 0 && (residual || prediction || vidx);
    if (direct) {
        res_d = static_cast<float *>(mapped_host(residual));
        pred_d = static_cast<float *>(mapped_host(prediction));
        vidx_d = static_cast<uint8_t *>(mapped_host(vidx));
        direct = (!residual || res_d) && (!prediction || pred_d) && (!vidx || vidx_d);
    }
    if (direct) {
        const int W = h->W, H = h->H;
        const int x0 = h->mx - 1 - h->mhx, x1 = W - 1 - h->mhx, y0 = h->my - 1 - h->mhy, y1 = H - 1 - h->mhy;
        for (float *o : {residual, prediction}) {
            if (!o)
                continue;
            if (y0 > 0)
                std::memset(o, 0, sizeof(float) * (size_t)y0 * W);
            if (y1 + 1 < H)
                std::memset(o + (size_t)(y1 + 1) * W, 0, sizeof(float) * (size_t)(H - 1 - y1) * W);
            for (int y = std::max(y0, 0); y <= std::min(y1, H - 1); y++) {
                float *row = o + (size_t)y * W;
                if (x0 > 0)
                    std::memset(row, 0, sizeof(float) * x0);
                if (x1 + 1 < W)
                    std::memset(row + x1 + 1, 0, sizeof(float) * (W - 1 - x1));
            }
        }
    }
    int rc = direct ? run_frame(h, s, &rd, frame_index, res_d, pred_d, vidx_d) : run_frame(h, s, &rd, frame_index);
    if (rc != CW_OK)
        return rc;
    if (ready)
        *ready = rd;
    // return only once the caller's buffers are no longer read or written:
    // host outputs given (as documented), or a page-locked input frame whose
    // upload is still in flight (a pageable one was staged synchronously)
    bool sync = direct || residual || prediction || vidx || src != h->h_stage;
    if (rd && !direct) {
        if (residual) {
            CW_CUDA(h, cudaMemcpyAsync(residual, h->d_res + set * HW, HW * 4, cudaMemcpyDeviceToHost, s));
            sync = true;
        }
        if (prediction) {
            CW_CUDA(h, cudaMemcpyAsync(prediction, h->d_pred + set * HW, HW * 4, cudaMemcpyDeviceToHost, s));
            sync = true;
        }
        if (vidx) {
            CW_CUDA(h, cudaMemcpyAsync(vidx, h->d_vidx + set * HW * 2 * h->idx_bytes, HW * 2 * h->idx_bytes, cudaMemcpyDeviceToHost, s));
            sync = true;
        }
    }
    if (sync)
        CW_CUDA(h, cudaStreamSynchronize(s));
    return CW_OK;
}

int cw_device_outputs(cw_handle *h, float **residual, float **prediction, uint8_t **vidx)
{
    if (!h)
        return CW_ERR_VALUE;
    const size_t HW = (size_t)h->W * h->H;
    const size_t set = (size_t)((h->frames_seen + 1) & 1);  // set of the latest pushed frame
    if (residual)
        *residual = h->d_res + set * HW;
    if (prediction)
        *prediction = h->d_pred + set * HW;
    if (vidx)
        *vidx = h->d_vidx + set * HW * 2 * h->idx_bytes;
    return CW_OK;
}

// Asynchronous pipelined push: upload (stream `up`), frame kernel (own
// stream) and download (stream `down`) of consecutive frames overlap.
//  H2D(n) into slot n % (mhat_z+2) waits for kernel(n-2), the last reader
//  of that slot (as the delayed frame of n-2 ... or current frame n-R);
//  kernel(n) waits for H2D(n) and for D2H(n-2), which read output set n % 2;
//  D2H(n) waits for kernel(n).  Host buffers should be pinned.
// PGM16 payload -> float32 frame slot: big-endian u16 q, v = f32(f64(q) *
// scale + offset) with the multiply and add rounded separately, as numpy
// evaluates q.astype(f64) * scale + offset (seqio.py:199-202).  8 samples
// per thread from one 16-byte load.
__global__ void cw_decode_pgm16_kernel(const uint16_t *__restrict__ src, float *__restrict__ dst, size_t n,
                                       double scale, double offset)
{
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const size_t n8 = n / 8;
    auto cvt = [&](uint32_t q) { return (float)__dadd_rn(__dmul_rn((double)q, scale), offset); };
    for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n8; k += stride) {
        const uint4 v = reinterpret_cast<const uint4 *>(src)[k];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        float *o = dst + 8 * k;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t s = __byte_perm(w[j], 0, 0x2301);  // swap the bytes of both halves
            o[2 * j] = cvt(s & 0xffffu);
            o[2 * j + 1] = cvt(s >> 16);
        }
    }
    for (size_t i = 8 * n8 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t q = src[i];
        dst[i] = cvt(((q & 0xffu) << 8) | (q >> 8));
    }
}

static int submit_impl(cw_handle *h, const void *samples, int format, double scale, double offset,
                       float *residual, float *prediction, uint8_t *vidx, int64_t *ticket);

int cw_submit(cw_handle *h, const float *frame, float *residual, float *prediction, uint8_t *vidx,
              int64_t *ticket)
{
    return submit_impl(h, frame, CW_FMT_F32LE, 1.0, 0.0, residual, prediction, vidx, ticket);
}

int cw_submit_raw(cw_handle *h, const void *samples, int32_t format, double scale, double offset,
                  float *residual, float *prediction, uint8_t *vidx, int64_t *ticket)
{
    if (h && format != CW_FMT_F32LE && format != CW_FMT_PGM16)
        return fail(h, CW_ERR_VALUE, "unknown sample format");
    if (h && format == CW_FMT_PGM16 && !(scale > 0.0))
        return fail(h, CW_ERR_VALUE, "scale must be > 0");
    return submit_impl(h, samples, format, scale, offset, residual, prediction, vidx, ticket);
}

static int submit_impl(cw_handle *h, const void *samples, int format, double scale, double offset,
                       float *residual, float *prediction, uint8_t *vidx, int64_t *ticket)
{
    DeviceGuard dg(h);
    NvtxRange nvtx("cw_submit");
    const void *frame = samples;
    if (!h || !frame || !ticket)
        return CW_ERR_VALUE;
    const size_t HW = (size_t)h->W * h->H;
    const long long n = h->frames_seen;
    const int e = (int)(n % cw_handle::NEV);
    if (n >= cw_handle::NEV)  // ticket n - NEV must have been collected
        CW_CUDA(h, cudaEventSynchronize(h->ev_down[e]));
    if (n >= 2)
        CW_CUDA(h, cudaStreamWaitEvent(h->up, h->ev_k[(n - 2) % cw_handle::NEV], 0));
    float *slot = h->d_frames + (size_t)(n % h->nslots) * HW;
    // chained: the kernel's stream carries no cross-stream wait (it would
    // serialise consecutive frame kernels); the upload and the download of
    // frame n - 2 (this output set) post flags the kernel waits on instead.
    // Only copy-engine work may feed a flag the kernel spins on: the PGM16
    // decode kernel needs SM slots the spinning CTAs could hold.
    const bool flagged = chained(h) && h->write_value && format != CW_FMT_PGM16;
    if (format == CW_FMT_PGM16) {
        if (!h->d_raw) {
            CW_CUDA(h, cudaMalloc(&h->d_raw, HW * 2 + 16));
        }
        // the staging buffer is reused in `up` stream order: H2D(n+1) follows decode(n)
        CW_CUDA(h, cudaMemcpyAsync(h->d_raw, frame, HW * 2, cudaMemcpyHostToDevice, h->up));
        const int blocks = (int)std::min<size_t>((HW / 8 + 255) / 256 + 1, (size_t)h->sms * 8);
        cw_decode_pgm16_kernel<<<blocks, 256, 0, h->up>>>(reinterpret_cast<const uint16_t *>(h->d_raw), slot, HW,
                                                         scale, offset);
        CW_CUDA(h, cudaGetLastError());
    } else {
        CW_CUDA(h, cudaMemcpyAsync(slot, frame, HW * 4, cudaMemcpyHostToDevice, h->up));
    }
    CW_CUDA(h, cudaEventRecord(h->ev_up[e], h->up));
    FlagWants fw{};
    if (flagged) {
        const unsigned int tag = (unsigned int)(n + 1);
        if (h->write_value(reinterpret_cast<CUstream>(h->up), reinterpret_cast<CUdeviceptr>(h->d_flags), tag, 0) !=
            CUDA_SUCCESS)
            return fail(h, CW_ERR_CUDA, "cuStreamWriteValue32 failed");
        fw.up_want = tag;
        // frame n - 2 wrote this output set: a flagged download posted n - 1,
        // any other download is waited for by its event
        if (n >= 2 && h->dl_flagged[(n - 2) % cw_handle::NEV])
            fw.down_want = (unsigned int)(n - 1);
        else if (n >= 2 && h->dl_any[(n - 2) % cw_handle::NEV])
            CW_CUDA(h, cudaStreamWaitEvent(h->own, h->ev_down[(n - 2) % cw_handle::NEV], 0));
    } else {
        CW_CUDA(h, cudaStreamWaitEvent(h->own, h->ev_up[e], 0));
        if (n >= 2)
            CW_CUDA(h, cudaStreamWaitEvent(h->own, h->ev_down[(n - 2) % cw_handle::NEV], 0));
    }
    int32_t rd = 0;
    int64_t fi = -1;
    const size_t set = (size_t)(n & 1);
    int rc = run_frame(h, h->own, &rd, &fi, nullptr, nullptr, nullptr, nullptr, true, flagged ? &fw : nullptr);
    if (rc != CW_OK)
        return rc;
    CW_CUDA(h, cudaEventRecord(h->ev_k[e], h->own));
    CW_CUDA(h, cudaStreamWaitEvent(h->down, h->ev_k[e], 0));
    if (rd) {
        if (residual)
            CW_CUDA(h, cudaMemcpyAsync(residual, h->d_res + set * HW, HW * 4, cudaMemcpyDeviceToHost, h->down));
        if (prediction)
            CW_CUDA(h, cudaMemcpyAsync(prediction, h->d_pred + set * HW, HW * 4, cudaMemcpyDeviceToHost, h->down));
        if (vidx)
            CW_CUDA(h, cudaMemcpyAsync(vidx, h->d_vidx + set * HW * 2 * h->idx_bytes, HW * 2 * h->idx_bytes, cudaMemcpyDeviceToHost, h->down));
    }
    h->dl_any[e] = rd && (residual || prediction || vidx);
    if (flagged) {
        if (h->write_value(reinterpret_cast<CUstream>(h->down), reinterpret_cast<CUdeviceptr>(h->d_flags + 1),
                           (unsigned int)(n + 1), 0) != CUDA_SUCCESS)
            return fail(h, CW_ERR_CUDA, "cuStreamWriteValue32 failed");
        h->dl_flagged[e] = true;
    }
    CW_CUDA(h, cudaEventRecord(h->ev_down[e], h->down));
    h->ready_of[e] = rd;
    h->fidx_of[e] = fi;
    *ticket = n;
    return CW_OK;
}

// Pipelined push of a frame already in device memory (e.g. a strip
// assembled from NCCL halo receives): the handle's stream waits for the
// producer stream, copies the frame into its ring slot, and the producer
// stream is then ordered after that copy (the caller may overwrite its
// buffer with work enqueued later on `producer`); kernel and result download
// overlap the next frames exactly as cw_submit's.
static int submit_device_impl(cw_handle *h, const float *frame_dev, float *residual, float *prediction,
                              uint8_t *vidx, int64_t *ticket, void *producer, bool resident_frame);

int cw_submit_device(cw_handle *h, const float *frame_dev, float *residual, float *prediction, uint8_t *vidx,
                     int64_t *ticket, void *producer)
{
    return submit_device_impl(h, frame_dev, residual, prediction, vidx, ticket, producer, false);
}

int cw_submit_resident(cw_handle *h, const float *frame_dev, float *residual, float *prediction, uint8_t *vidx,
                       int64_t *ticket)
{
    return submit_device_impl(h, frame_dev, residual, prediction, vidx, ticket, nullptr, true);
}

static int submit_device_impl(cw_handle *h, const float *frame_dev, float *residual, float *prediction,
                              uint8_t *vidx, int64_t *ticket, void *producer, bool resident_frame)
{
    NvtxRange nvtx("cw_submit_device");
    DeviceGuard dg(h);
    if (!h || !frame_dev || !ticket)
        return CW_ERR_VALUE;
    const size_t HW = (size_t)h->W * h->H;
    const long long n = h->frames_seen;
    const int e = (int)(n % cw_handle::NEV);
    if (n >= cw_handle::NEV)  // ticket n - NEV must have been collected
        CW_CUDA(h, cudaEventSynchronize(h->ev_down[e]));
    float *slot = h->d_frames + (size_t)(n % h->nslots) * HW;
    // cw_submit_resident: the frame is complete in device memory and stays
    // unchanged until this ticket is collected -- the kernel reads it and
    // fills its ring slot itself, so consecutive frame kernels overlap
    // (chained); without chaining it is copied as cw_submit_device's
    const bool resident = resident_frame && chained(h) && slot != frame_dev;
    // the ring slot (read as the delayed frame m^_z frames later) filled by a
    // copy-engine copy on the upload stream after the kernel that last read
    // the slot (n - 2 or earlier), flagged for the kernel that reads it
    const bool ce_copy = resident && h->write_value && CW_RESIDENT_CE;
    if (ce_copy) {
        if (n >= 2)
            CW_CUDA(h, cudaStreamWaitEvent(h->up, h->ev_k[(n - 2) % cw_handle::NEV], 0));
        CW_CUDA(h, cudaMemcpyAsync(slot, frame_dev, HW * 4, cudaMemcpyDeviceToDevice, h->up));
        if (h->write_value(reinterpret_cast<CUstream>(h->up), reinterpret_cast<CUdeviceptr>(h->d_flags + 2),
                           (unsigned int)(n + 1), 0) != CUDA_SUCCESS)
            return fail(h, CW_ERR_CUDA, "cuStreamWriteValue32 failed");
        h->next_ring_tag = (unsigned int)(n + 1);
    }
    if (!resident) {
        cudaStream_t ps = reinterpret_cast<cudaStream_t>(producer);
        CW_CUDA(h, cudaEventRecord(h->ev_up[e], ps));
        CW_CUDA(h, cudaStreamWaitEvent(h->own, h->ev_up[e], 0));
        if (slot != frame_dev)
            CW_CUDA(h, cudaMemcpyAsync(slot, frame_dev, HW * 4, cudaMemcpyDeviceToDevice, h->own));
        CW_CUDA(h, cudaEventRecord(h->ev_up[e], h->own));
        CW_CUDA(h, cudaStreamWaitEvent(ps, h->ev_up[e], 0));
    }
    // the output set of frame n - 2 is downloaded before kernel n rewrites
    // it.  Chained: a flagged download is waited for in the kernel, another
    // download by its event, no download not at all -- a pending
    // cross-stream wait between two frame kernels serialises them
    // (measured: it cancels the programmatic launch)
    FlagWants fw{};
    bool use_fw = false;
    if (n >= 2) {
        const int e2 = (int)((n - 2) % cw_handle::NEV);
        if (resident && h->dl_flagged[e2]) {
            fw.down_want = (unsigned int)(n - 1);
            use_fw = true;
        } else if (!resident || h->dl_any[e2]) {
            CW_CUDA(h, cudaStreamWaitEvent(h->own, h->ev_down[e2], 0));
        }
    }
    int32_t rd = 0;
    int64_t fi = -1;
    const size_t set = (size_t)(n & 1);
    int rc = run_frame(h, h->own, &rd, &fi, nullptr, nullptr, nullptr, resident ? frame_dev : nullptr, resident,
                       use_fw ? &fw : nullptr, !ce_copy);
    if (rc != CW_OK)
        return rc;
    CW_CUDA(h, cudaEventRecord(h->ev_k[e], h->own));
    CW_CUDA(h, cudaStreamWaitEvent(h->down, h->ev_k[e], 0));
    const size_t vb = HW * 2 * h->idx_bytes;
    if (rd) {
        if (residual)
            CW_CUDA(h, cudaMemcpyAsync(residual, h->d_res + set * HW, HW * 4, cudaMemcpyDeviceToHost, h->down));
        if (prediction)
            CW_CUDA(h, cudaMemcpyAsync(prediction, h->d_pred + set * HW, HW * 4, cudaMemcpyDeviceToHost, h->down));
        if (vidx)
            CW_CUDA(h, cudaMemcpyAsync(vidx, h->d_vidx + set * vb, vb, cudaMemcpyDeviceToHost, h->down));
    }
    h->dl_any[e] = rd && (residual || prediction || vidx);
    if (resident && h->dl_any[e] && h->write_value) {
        // the next-but-one resident frame waits for this download in its
        // kernel (flag), not on the kernel stream (event)
        if (h->write_value(reinterpret_cast<CUstream>(h->down), reinterpret_cast<CUdeviceptr>(h->d_flags + 1),
                           (unsigned int)(n + 1), 0) != CUDA_SUCCESS)
            return fail(h, CW_ERR_CUDA, "cuStreamWriteValue32 failed");
        h->dl_flagged[e] = true;
    }
    CW_CUDA(h, cudaEventRecord(h->ev_down[e], h->down));
    h->ready_of[e] = rd;
    h->fidx_of[e] = fi;
    *ticket = n;
    return CW_OK;
}

int cw_join(cw_handle *h, void *stream)
{
    DeviceGuard dg(h);
    if (!h)
        return CW_ERR_VALUE;
    CW_CUDA(h, cudaEventRecord(h->ev_join, h->own));
    CW_CUDA(h, cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), h->ev_join, 0));
    return CW_OK;
}

int cw_wait(cw_handle *h, int64_t ticket, int32_t *ready, int64_t *frame_index)
{
    DeviceGuard dg(h);
    if (!h || ticket < 0 || ticket >= h->frames_seen || ticket < h->frames_seen - cw_handle::NEV)
        return h ? fail(h, CW_ERR_VALUE, "unknown or expired ticket") : CW_ERR_VALUE;
    const int e = (int)(ticket % cw_handle::NEV);
    CW_CUDA(h, cudaEventSynchronize(h->ev_down[e]));
    if (ready)
        *ready = h->ready_of[e];
    if (frame_index)
        *frame_index = h->fidx_of[e];
    return CW_OK;
}

int cw_set_detection(cw_handle *h, float tau, int32_t cap)
{
    DeviceGuard dg(h);
    if (!h)
        return CW_ERR_VALUE;
    if (cap < 0) {  // off
        h->det_on = false;
        return CW_OK;
    }
    const size_t bytes = det_head_bytes(h) + (size_t)cap * 16;
    if (bytes != h->det_bytes) {
        CW_CUDA(h, cudaSetDevice(h->device));
        CW_CUDA(h, cudaDeviceSynchronize());
        cudaFree(h->d_det);
        if (h->h_det)
            cudaFreeHost(h->h_det);
        h->d_det = nullptr;
        h->h_det = nullptr;
        CW_CUDA(h, cudaMalloc(&h->d_det, 2 * bytes));
        CW_CUDA(h, cudaMallocHost(&h->h_det, cw_handle::NEV * bytes));
        std::memset(h->h_det, 0, cw_handle::NEV * bytes);
        h->det_bytes = bytes;
    }
    h->det_tau = tau;
    h->det_cap = cap;
    h->det_on = true;
    return CW_OK;
}

int cw_detections(cw_handle *h, int64_t ticket, int32_t *n_total, float *xyr, int32_t out_cap, double *stats)
{
    if (!h || !h->det_on || ticket < 0 || ticket >= h->frames_seen || ticket < h->frames_seen - cw_handle::NEV)
        return h ? fail(h, CW_ERR_VALUE, "detections unavailable for this frame") : CW_ERR_VALUE;
    const unsigned char *b = h->h_det + (size_t)(ticket % cw_handle::NEV) * h->det_bytes;
    unsigned int count;
    unsigned long long key, nval;
    std::memcpy(&count, b, 4);
    std::memcpy(&key, b + 8, 8);
    std::memcpy(&nval, b + 24, 8);
    double sumsq = 0.0;  // fixed summation order over the (row, block) partial sums
    for (size_t i = 0; i < (size_t)h->H * h->NXB; i++) {
        double v;
        std::memcpy(&v, b + 64 + 8 * i, 8);
        sumsq += v;
    }
    if (n_total)
        *n_total = (int32_t)count;
    const int k = (int)std::min<long long>(std::min<long long>(count, h->det_cap), std::max(0, out_cap));
    for (int i = 0; i < k && xyr; i++) {
        float v[4];
        std::memcpy(v, b + det_head_bytes(h) + (size_t)i * 16, 16);
        xyr[3 * i] = v[0];
        xyr[3 * i + 1] = v[1];
        xyr[3 * i + 2] = v[2];
    }
    if (stats) {
        unsigned int bits = (unsigned int)(key >> 32);
        float peak;
        std::memcpy(&peak, &bits, 4);
        const unsigned long long idx = 0xffffffffull - (key & 0xffffffffull);
        stats[0] = nval ? peak : 0.0;
        stats[1] = nval ? (double)(idx % h->W) : -1.0;
        stats[2] = nval ? (double)(idx / h->W) : -1.0;
        stats[3] = sumsq;
        stats[4] = (double)nval;
    }
    return CW_OK;
}

#ifdef CW_PHASE_TIMING
extern "C" int cw_phase_clocks(unsigned long long *dst)  // [8][16], then zeroed
{
    if (!g_phase_clocks) return CW_ERR_VALUE;
    g_phase_clocks(dst);
    return 0;
}
#endif

// Checkpoint / resume: the whole stream state -- observer
// state, T^, frame ring, counters -- as one host blob.
struct SnapHeader {
    uint64_t magic, version;
    int64_t frames_seen;
    int32_t have_that, W, H, kx, ky, kz, nslots, pad;
    uint64_t state_bytes, that_bytes, frames_bytes;
};
static const uint64_t SNAP_MAGIC = 0x43574232534e4150ull;  // "CWB2SNAP"

int cw_snapshot_size(const cw_handle *h, size_t *bytes)
{
    if (!h || !bytes)
        return CW_ERR_VALUE;
    *bytes = sizeof(SnapHeader) + (h->state_floats + h->that_floats) * 4 + (size_t)h->W * h->H * 4 * h->nslots;
    return CW_OK;
}

int cw_snapshot(cw_handle *h, void *dst, size_t bytes)
{
    DeviceGuard dg(h);
    size_t need = 0;
    cw_snapshot_size(h, &need);
    if (!h || !dst || bytes != need)
        return h ? fail(h, CW_ERR_VALUE, "snapshot buffer size mismatch") : CW_ERR_VALUE;
    CW_CUDA(h, cudaSetDevice(h->device));
    CW_CUDA(h, cudaDeviceSynchronize());
    SnapHeader hd{SNAP_MAGIC, 1, h->frames_seen, h->have_that ? 1 : 0, h->W, h->H, h->kx, h->ky, h->kz, h->nslots, 0,
                  h->state_floats * 4, h->that_floats * 4, (size_t)h->W * h->H * 4 * h->nslots};
    unsigned char *o = static_cast<unsigned char *>(dst);
    std::memcpy(o, &hd, sizeof hd);
    o += sizeof hd;
    CW_CUDA(h, cudaMemcpy(o, h->d_state, hd.state_bytes, cudaMemcpyDeviceToHost));
    o += hd.state_bytes;
    CW_CUDA(h, cudaMemcpy(o, h->d_that, hd.that_bytes, cudaMemcpyDeviceToHost));
    o += hd.that_bytes;
    CW_CUDA(h, cudaMemcpy(o, h->d_frames, hd.frames_bytes, cudaMemcpyDeviceToHost));
    return CW_OK;
}

int cw_restore(cw_handle *h, const void *src, size_t bytes)
{
    DeviceGuard dg(h);
    size_t need = 0;
    cw_snapshot_size(h, &need);
    if (!h || !src || bytes != need)
        return h ? fail(h, CW_ERR_VALUE, "snapshot size does not match this pipeline") : CW_ERR_VALUE;
    SnapHeader hd;
    std::memcpy(&hd, src, sizeof hd);
    if (hd.magic != SNAP_MAGIC || hd.version != 1 || hd.W != h->W || hd.H != h->H || hd.kx != h->kx ||
        hd.ky != h->ky || hd.kz != h->kz || hd.nslots != h->nslots)
        return fail(h, CW_ERR_VALUE, "snapshot was taken from a different pipeline geometry");
    CW_CUDA(h, cudaSetDevice(h->device));
    CW_CUDA(h, cudaDeviceSynchronize());
    const unsigned char *p = static_cast<const unsigned char *>(src) + sizeof hd;
    CW_CUDA(h, cudaMemcpy(h->d_state, p, hd.state_bytes, cudaMemcpyHostToDevice));
    p += hd.state_bytes;
    CW_CUDA(h, cudaMemcpy(h->d_that, p, hd.that_bytes, cudaMemcpyHostToDevice));
    p += hd.that_bytes;
    CW_CUDA(h, cudaMemcpy(h->d_frames, p, hd.frames_bytes, cudaMemcpyHostToDevice));
    h->frames_seen = hd.frames_seen;
    h->have_that = hd.have_that != 0;
    // the submit flags are tagged with frame numbers: restart them
    if (h->d_flags)
        CW_CUDA(h, cudaMemset(h->d_flags, 0, 3 * sizeof(unsigned int)));
    std::fill(h->ring_tag.begin(), h->ring_tag.end(), 0u);
    h->next_ring_tag = 0;
    for (bool &f : h->dl_flagged)
        f = false;
    for (bool &f : h->dl_any)
        f = false;
    return CW_OK;
}

int cw_copy_to_host(cw_handle *h, void *dst, const void *src_dev, size_t bytes)
{
    DeviceGuard dg(h);
    if (!h || !dst || !src_dev)
        return CW_ERR_VALUE;
    CW_CUDA(h, cudaMemcpy(dst, src_dev, bytes, cudaMemcpyDeviceToHost));
    return CW_OK;
}

int cw_launch_info(const cw_handle *h, int32_t *kernels_per_push, int32_t *grid, int32_t *block,
                   int32_t *smem_bytes)
{
    if (!h)
        return CW_ERR_VALUE;
    if (kernels_per_push)
        *kernels_per_push = h->generic ? 3 : 1;
    if (grid)
        *grid = h->generic ? 0 : h->grid;
    if (block)
        *block = h->generic ? 128 : h->fn.threads;
    if (smem_bytes)
        *smem_bytes = h->generic ? 0 : (int32_t)h->fn.smem;
    return CW_OK;
}

int cw_set_backend(cw_handle *h, int32_t naive)
{
    DeviceGuard dg(h);
    if (!h)
        return CW_ERR_VALUE;
    if (h->generic) {
        if (naive && ensure_xf(h, h->mz) != CW_OK)
            return CW_ERR_NOMEM;
        h->naive = naive != 0;
        return CW_OK;
    }
    if (naive && !h->naive_grid) {
        CW_CUDA(h, cudaSetDevice(h->device));
        CW_CUDA(h, cudaFuncSetAttribute(h->fn.naive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)h->fn.naive_smem));
        int occ = 0, sms = 0;
        CW_CUDA(h, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, h->fn.naive_kernel, h->fn.threads,
                                                                 h->fn.naive_smem));
        CW_CUDA(h, cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
        h->naive_grid = std::max(1, occ * sms);
    }
    // the naive kernel reads Mz ring frames without waiting on flags: any
    // flagged (copy-engine) ring copy must be complete
    if (naive && h->up) {
        CW_CUDA(h, cudaStreamSynchronize(h->up));
        std::fill(h->ring_tag.begin(), h->ring_tag.end(), 0u);
    }
    h->naive = naive != 0;
    return CW_OK;
}

int cw_set_timing(cw_handle *h, int32_t on)
{
    if (!h)
        return CW_ERR_VALUE;
    h->timing = on != 0;
    h->ev_used = 0;
    return CW_OK;
}

int cw_kernel_time(cw_handle *h, double *total_ms, int64_t *launches)
{
    DeviceGuard dg(h);
    if (!h || !total_ms || !launches)
        return CW_ERR_VALUE;
    double tot = 0.0;
    for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
        CW_CUDA(h, cudaEventSynchronize(h->ev_pool[i + 1]));
        float ms = 0.f;
        CW_CUDA(h, cudaEventElapsedTime(&ms, h->ev_pool[i], h->ev_pool[i + 1]));
        tot += ms;
    }
    *total_ms = tot;
    *launches = (int64_t)(h->ev_used / 2);
    h->ev_used = 0;
    return CW_OK;
}

// Parity views: unpack the packet layout into the reference layouts.
int cw_read_view(cw_handle *h, int32_t what, void *dst, size_t bytes)
{
    DeviceGuard dg(h);
    if (!h || !dst)
        return CW_ERR_VALUE;
    CW_CUDA(h, cudaSetDevice(h->device));
    CW_CUDA(h, cudaDeviceSynchronize());
    const int W = h->W, H = h->H, NXB = h->NXB;
    const int Mx = h->mx, My = h->my, Mz = h->mz, KX = h->kx, KY = h->ky, KZ = h->kz;
    if (what == 2) {
        if (bytes != h->state_floats * 4)
            return fail(h, CW_ERR_VALUE, "view size mismatch");
        CW_CUDA(h, cudaMemcpy(dst, h->d_state, bytes, cudaMemcpyDeviceToHost));
        return CW_OK;
    }
    if (h->generic && (what == 0 || what == 1)) {
        // planes [plane][pixel] of the full spectrum: state = z+, S = norm z+;
        // T^ planes (My, Mx) -- transposed into the reference layouts
        const size_t HW = (size_t)W * H, np = what == 0 ? (size_t)Mx * My * Mz : (size_t)Mx * My;
        if (bytes != HW * np * 16)
            return fail(h, CW_ERR_VALUE, "view size mismatch");
        std::vector<float2> pl(HW * np);
        CW_CUDA(h, cudaMemcpy(pl.data(), what == 0 ? h->d_state : h->d_that, pl.size() * 8, cudaMemcpyDeviceToHost));
        const double sc = what == 0 ? 1.0 / std::sqrt((double)Mx * My * Mz) : 1.0;
        double *o = static_cast<double *>(dst);
        for (size_t q = 0; q < np; q++)
            for (size_t px = 0; px < HW; px++) {
                const float2 v = pl[q * HW + px];
                o[2 * (px * np + q)] = sc * v.x;
                o[2 * (px * np + q) + 1] = sc * v.y;
            }
        return CW_OK;
    }
    // pair j of pixel (y, x) in a packet buffer of `np` pairs per pixel
    auto pairs_of = [&](const std::vector<float> &pk, int np, int y, int x, int j, double *re, double *im) {
        const float *f = pk.data() + ((((size_t)y * NXB + x / 32) * np + j) * 32 + (x % 32)) * 2;
        *re = f[0];
        *im = f[1];
    };
    if (what == 0) {
        const size_t nb = (size_t)Mx * My * Mz;
        if (bytes != (size_t)H * W * nb * 16)
            return fail(h, CW_ERR_VALUE, "view size mismatch");
        // the stored state is z = w(kz) z+ of the last frame: S = norm conj(w) z
        std::vector<float> pk(h->state_floats);
        CW_CUDA(h, cudaMemcpy(pk.data(), h->d_state, h->state_floats * 4, cudaMemcpyDeviceToHost));
        const double PI = 3.14159265358979323846, norm = 1.0 / std::sqrt((double)Mx * My * Mz);
        double *o = static_cast<double *>(dst);
        const int NSP = h->fn.nsp;
        const int row0 = (KZ + 1) + KX * Mz, rown = Mx * Mz;
        for (int y = 0; y < H; y++)
            for (int x = 0; x < W; x++) {
                const size_t pb = ((size_t)y * W + x) * nb;
                auto put = [&](int kz, int ky, int kx, double zr, double zi) {
                    const double c = std::cos(2 * PI * kz / Mz), sn = -std::sin(2 * PI * kz / Mz);
                    const double re = norm * (c * zr - sn * zi), im = norm * (c * zi + sn * zr);
                    size_t i = pb + (((size_t)(kz + KZ) * My + (ky + KY)) * Mx + (kx + KX));
                    o[2 * i] = re;
                    o[2 * i + 1] = im;
                    size_t k = pb + (((size_t)(-kz + KZ) * My + (-ky + KY)) * Mx + (-kx + KX));
                    o[2 * k] = re;
                    o[2 * k + 1] = -im;
                };
                double re, im;
                for (int kz = 0; kz <= KZ; kz++) {
                    pairs_of(pk, NSP, y, x, kz, &re, &im);
                    put(kz, 0, 0, re, kz == 0 ? 0.0 : im);
                }
                for (int kx = 1; kx <= KX; kx++)
                    for (int kz = -KZ; kz <= KZ; kz++) {
                        pairs_of(pk, NSP, y, x, KZ + 1 + (kx - 1) * Mz + (kz + KZ), &re, &im);
                        put(kz, 0, kx, re, im);
                    }
                for (int ky = 1; ky <= KY; ky++)
                    for (int kx = -KX; kx <= KX; kx++)
                        for (int kz = -KZ; kz <= KZ; kz++) {
                            pairs_of(pk, NSP, y, x, row0 + (ky - 1) * rown + (kx + KX) * Mz + (kz + KZ), &re, &im);
                            put(kz, ky, kx, re, im);
                        }
            }
        return CW_OK;
    }
    if (what == 1) {
        const size_t nt = (size_t)Mx * My;
        if (bytes != (size_t)H * W * nt * 16)
            return fail(h, CW_ERR_VALUE, "view size mismatch");
        std::vector<float> pk(h->that_floats);
        CW_CUDA(h, cudaMemcpy(pk.data(), h->d_that, h->that_floats * 4, cudaMemcpyDeviceToHost));
        double *o = static_cast<double *>(dst);
        const int NTP = h->fn.ntp;
        for (int y = 0; y < H; y++)
            for (int x = 0; x < W; x++) {
                const size_t pb = ((size_t)y * W + x) * nt;
                auto put = [&](int ky, int kx, double re, double im) {
                    size_t i = pb + (size_t)(ky + KY) * Mx + (kx + KX);
                    o[2 * i] = re;
                    o[2 * i + 1] = im;
                    size_t k = pb + (size_t)(-ky + KY) * Mx + (-kx + KX);
                    o[2 * k] = re;
                    o[2 * k + 1] = -im;
                };
                double re, im;
                pairs_of(pk, NTP, y, x, 0, &re, &im);
                put(0, 0, re, 0.0);
                for (int kx = 1; kx <= KX; kx++) {
                    pairs_of(pk, NTP, y, x, kx, &re, &im);
                    put(0, kx, re, im);
                }
                for (int ky = 1; ky <= KY; ky++)
                    for (int kx = -KX; kx <= KX; kx++) {
                        pairs_of(pk, NTP, y, x, (KX + 1) + (ky - 1) * Mx + (kx + KX), &re, &im);
                        put(ky, kx, re, im);
                    }
            }
        return CW_OK;
    }
    return fail(h, CW_ERR_VALUE, "unknown view");
}

}  // extern "C"
