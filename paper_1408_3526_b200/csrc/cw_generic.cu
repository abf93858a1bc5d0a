// cw_generic.cu -- runtime-geometry kernels (see cw_generic.cuh).
#include "cw_frame.cuh"  // FrameArgs + detect_epilogue (shared detection epilogue)
#include "cw_generic.cuh"

#include <algorithm>

namespace cwb {
namespace {

__device__ __forceinline__ float2 cmul(float2 a, float2 b)
{
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

// X(f, ikx; y, x) for the frames the spectrum needs: f = 0 (recursive
// backend: frame n) or f = 0..Mz-1 (naive: frame n - f).
__global__ void __launch_bounds__(256) gen_xstage(const GenArgs a, const GenTables t, int nf)
{
    const long long HW = (long long)a.W * a.H;
    const long long total = HW * nf;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(i / HW);
        const long long p = i - (long long)f * HW;
        const int y = (int)(p / a.W), x = (int)(p - (long long)y * a.W);
        if (x < a.mx - 1 || y < a.y_begin - (a.my - 1))
            continue;
        const float *img = a.frames + (size_t)((a.n - f) % a.nslots) * HW + (size_t)y * a.W;
        float2 *out = a.xf + (size_t)f * a.mx * HW + p;
        for (int k = 0; k < a.mx; k++) {
            float2 acc = make_float2(0.f, 0.f);
            for (int m = 0; m < a.mx; m++) {
                const float v = img[x - m];
                const float2 e = t.ex[k * a.mx + m];
                acc.x += e.x * v;
                acc.y += e.y * v;
            }
            out[(size_t)k * HW] = acc;
        }
    }
}

// y window sums + the deadbeat observer (or the naive window DFT).
__global__ void __launch_bounds__(256) gen_observer(const GenArgs a, const GenTables t)
{
    const long long HW = (long long)a.W * a.H;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < HW; p += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(p / a.W), x = (int)(p - (long long)y * a.W);
        if (x < a.mx - 1 || y < a.y_begin || y < a.my - 1 || y + a.y_off < a.my - 1)
            continue;  // no full window: the spectrum stays 0 (_kernels.py:48-90 skip the border)
        for (int ky = 0; ky < a.my; ky++)
            for (int kx = 0; kx < a.mx; kx++) {
                if (!a.naive) {
                    float2 u = make_float2(0.f, 0.f);
                    for (int m = 0; m < a.my; m++)
                        u = cadd(u, cmul(t.ey[ky * a.my + m], a.xf[(size_t)kx * HW + p - (long long)m * a.W]));
                    // z = w z+ (last frame); e = u - sum z / Mz; z+ = z + e
                    float2 z[64];
                    float2 s = make_float2(0.f, 0.f);
                    for (int kz = 0; kz < a.mz; kz++) {
                        const float2 zp = a.state[((size_t)(kz * a.my + ky) * a.mx + kx) * HW + p];
                        const float2 r = cmul(t.w[kz], zp);
                        if (kz < 64) z[kz] = r;
                        s = cadd(s, r);
                    }
                    const float2 e = make_float2(u.x - s.x * a.inv_mz, u.y - s.y * a.inv_mz);
                    for (int kz = 0; kz < a.mz; kz++) {
                        float2 *sp = a.state + ((size_t)(kz * a.my + ky) * a.mx + kx) * HW + p;
                        const float2 r = kz < 64 ? z[kz] : cmul(t.w[kz], *sp);
                        *sp = cadd(r, e);
                    }
                } else {
                    // D(kz) = sum_f e^{+j2pi kz f / Mz} U_{n-f}: the ring DFT of the
                    // spatial spectra (temporal_dft, _kernels.py:71-90), from raw frames
                    for (int kz = 0; kz < a.mz; kz++) {
                        float2 d = make_float2(0.f, 0.f);
                        for (int f = 0; f < a.mz; f++) {
                            float2 u = make_float2(0.f, 0.f);
                            const float2 *xf = a.xf + ((size_t)f * a.mx + kx) * HW + p;
                            for (int m = 0; m < a.my; m++)
                                u = cadd(u, cmul(t.ey[ky * a.my + m], xf[-(long long)m * a.W]));
                            d = cadd(d, cmul(t.ez[kz * a.mz + f], u));
                        }
                        a.state[((size_t)(kz * a.my + ky) * a.mx + kx) * HW + p] = d;
                    }
                }
            }
    }
}

__device__ __forceinline__ int wrap(int i, int m) { return i < 0 ? i + m : (i >= m ? i - m : i); }

// conditioning + T^ + contraction/argmax + PEF for one anchor per thread;
// a warp is 32 adjacent columns of one row (the detection epilogue's unit)
__global__ void __launch_bounds__(128) gen_flow(const GenArgs a, const GenTables t)
{
    const int lane = threadIdx.x;
    const int x = blockIdx.x * 32 + lane;
    const int y = a.y_begin + blockIdx.y * blockDim.y + threadIdx.y;
    if (y >= a.H)
        return;  // warp-uniform
    const long long HW = (long long)a.W * a.H;
    const long long p = (long long)y * a.W + x;
    const bool colv = x < a.W;
    const bool anchor = colv && x >= a.mx - 1 && y + a.y_off >= a.my - 1;
    int vix = t.rix[0], viy = t.riy[0];  // flat surface: the lowest-rank lag (zero velocity first)
    float rv = 0.f;
    if (anchor) {
        const int KX = a.kx, KY = a.ky;
        auto cond = [&](int kz, int ky, int kx) -> float2 {
            if (ky == KY && kx == KX)
                return make_float2(0.f, 0.f);  // zero_spatial_dc (_kernels.py:167-174)
            return a.state[((size_t)(kz * a.my + ky) * a.mx + kx) * HW + p];
        };
        const float hw[3] = {-0.25f, 0.5f, -0.25f};
        // hann3 (_kernels.py:177-217) is separable: G(kz') = (Hy Hx C)(kz', ky, kx)
        // from 9 taps, then Hz over a rolling window G(kz-1), G(kz), G(kz+1)
        auto gxy = [&](int kz, int ky, int kx) -> float2 {
            float2 sy = make_float2(0.f, 0.f);
            for (int dy = 0; dy < 3; dy++) {
                const int iy = wrap(ky + dy - 1, a.my);
                float2 sx = make_float2(0.f, 0.f);
                for (int dx = 0; dx < 3; dx++) {
                    const float2 c = cond(kz, iy, wrap(kx + dx - 1, a.mx));
                    sx.x += hw[dx] * c.x;
                    sx.y += hw[dx] * c.y;
                }
                sy.x += hw[dy] * sx.x;
                sy.y += hw[dy] * sx.y;
            }
            return sy;
        };
        for (int ky = 0; ky < a.my; ky++)
            for (int kx = 0; kx < a.mx; kx++) {
                float2 tz = make_float2(0.f, 0.f);
                const float2 glast = gxy(a.mz - 1, ky, kx), gfirst = gxy(0, ky, kx);
                float2 gm = glast, g0 = gfirst;
                for (int kz = 0; kz < a.mz; kz++) {
                    const float2 gp = kz + 1 < a.mz ? (kz + 1 == a.mz - 1 ? glast : gxy(kz + 1, ky, kx)) : gfirst;
                    const float2 h = make_float2(hw[0] * gm.x + hw[1] * g0.x + hw[2] * gp.x,
                                                 hw[0] * gm.y + hw[1] * g0.y + hw[2] * gp.y);
                    const float pw = h.x * h.x + h.y * h.y;  // power (_kernels.py:220-227)
                    tz.x += t.az[kz].x * pw;
                    tz.y += t.az[kz].y * pw;
                    gm = g0;
                    g0 = gp;
                }
                float2 *th = a.that + (size_t)(ky * a.mx + kx) * HW + p;
                if (a.first) {
                    *th = tz;  // first ready frame: R^ := R (pipeline.py:245-247)
                } else {
                    const float2 o = *th;  // smooth (_kernels.py:261-271), on T^ by linearity
                    *th = make_float2(a.beta * tz.x + a.alpha * o.x, a.beta * tz.y + a.alpha * o.y);
                }
            }
        // R(ly, lx) = Re sum_ky ayl(ly) B(ky, lx), B = sum_kx axl(lx) T^ (gains
        // folded; the separable order of _kernels.py:230-258); total-order argmax
        float best = 0.f;
        uint32_t brank = 0xffffffffu;
        constexpr int MAXB = 64;
        float2 bk[MAXB];
        for (int lx = 0; lx < a.nlx; lx++) {
            const bool cache = a.my <= MAXB;
            if (cache)
                for (int ky = 0; ky < a.my; ky++) {
                    float2 b = make_float2(0.f, 0.f);
                    for (int kx = 0; kx < a.mx; kx++)
                        b = cadd(b, cmul(t.axl[lx * a.mx + kx], a.that[(size_t)(ky * a.mx + kx) * HW + p]));
                    bk[ky] = b;
                }
            for (int ly = 0; ly < a.nly; ly++) {
                float r = 0.f;
                for (int ky = 0; ky < a.my; ky++) {
                    float2 b;
                    if (cache) {
                        b = bk[ky];
                    } else {
                        b = make_float2(0.f, 0.f);
                        for (int kx = 0; kx < a.mx; kx++)
                            b = cadd(b, cmul(t.axl[lx * a.mx + kx], a.that[(size_t)(ky * a.mx + kx) * HW + p]));
                    }
                    const float2 e = t.ayl[ly * a.my + ky];
                    r += e.x * b.x - e.y * b.y;
                }
                const uint32_t rk = t.rank[ly * a.nlx + lx];
                if (brank == 0xffffffffu || r > best || (r == best && rk < brank)) {
                    best = r;
                    brank = rk;
                }
            }
        }
        vix = t.rix[brank];
        viy = t.riy[brank];
    }
    if (a.forced_ix >= 0) {
        vix = a.forced_ix;
        viy = a.forced_iy;
    }
    if (colv) {
        if (a.idx16)
            reinterpret_cast<ushort2 *>(a.vidx)[p] = make_ushort2((unsigned short)vix, (unsigned short)viy);
        else
            reinterpret_cast<uchar2 *>(a.vidx)[p] = make_uchar2((unsigned char)vix, (unsigned char)viy);
    }
    if (anchor) {
        // PEF (_kernels.py:330-342): pred = Re sum_j bank[v][j] S[retained_j]
        const float2 *c = t.coef + (size_t)(viy * a.nlx + vix) * a.nc;
        float pr = 0.f;
        for (int j = 0; j < a.nc; j++) {
            const float2 z = a.state[(size_t)t.ret[j] * HW + p];
            pr += c[j].x * z.x - c[j].y * z.y;
        }
        const long long o = (long long)(y - a.mhy) * a.W + (x - a.mhx);
        rv = a.delayed[o] - pr;
        a.res[o] = rv;
        if (a.pred)
            a.pred[o] = pr;
    }
    if (a.det) {
        FrameArgs fa;
        fa.det = a.det;
        fa.det_tau = a.det_tau;
        fa.det_cap = a.det_cap;
        fa.W = a.W;
        fa.H = a.H;
        fa.NXB = a.NXB;
        fa.mhx = a.mhx;
        fa.mhy = a.mhy;
        detect_epilogue(fa, anchor, x - a.mhx, y - a.mhy, rv);
    }
}

}  // namespace

cudaError_t gen_launch(const GenArgs &a, const GenTables &t, int sms, cudaStream_t s)
{
    const long long HW = (long long)a.W * a.H;
    const int nf = a.naive ? a.mz : 1;
    if (a.naive && !a.ready)
        return cudaSuccess;  // the naive spectrum is needed only for ready frames
    auto grid = [&](long long n) { return (int)std::min<long long>((n + 255) / 256, (long long)sms * 16); };
    gen_xstage<<<grid(HW * nf), 256, 0, s>>>(a, t, nf);
    gen_observer<<<grid(HW), 256, 0, s>>>(a, t);
    if (a.ready) {
        const int rows = a.H - a.y_begin;
        gen_flow<<<dim3(a.NXB, (rows + 3) / 4), dim3(32, 4), 0, s>>>(a, t);
    }
    return cudaGetLastError();
}

}  // namespace cwb
