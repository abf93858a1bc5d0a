// cw_naive.cuh -- the non-recursive ("naive") spectrum backend (sm_100a).
//
// Reference: NaiveSpectrumStream (spectrum.py:257-327) and
// _kernels.naive_spectrum (_kernels.py:93-127): every pixel's local 3-D
// spectrum is evaluated directly from its own Mx x My x Mz raw window, with
// no recursion in x, y or t.  Here the result D (the unnormalised spectrum,
// S = D / sqrt(Mx My Mz)) is written into the observer-state packets; the
// fused frame kernel then runs unchanged: its observer update gives
//   z+ = D + u - (1/Mz) sum_kz D = D      (since (1/Mz) sum_kz D = u_n),
// so flow, PEF and residual see the naive spectrum.
#pragma once
#include "cw_frame.cuh"

namespace cwb {

struct NaiveArgs {
    const float *frames;   // frame ring base, slot s at frames + s * H * W
    int nslots;
    long long n;           // current frame number (frames n-Mz+1 .. n are in the ring)
    float2 *state;         // observer-state packets (overwritten with D)
    int W, H, NXB;
    int y_begin, y_off;
};

// scalar complex multiply-accumulate acc + a * b (this kernel is a
// reference-style direct evaluation; the packed helpers of the frame kernel
// only raise its register pressure)
__device__ __forceinline__ cf cmac_s(cf acc, cf a, cf b)
{
    return cf{acc.r + (a.r * b.r - a.i * b.i), acc.i + (a.r * b.i + a.i * b.r)};
}

template <class G>
__global__ void __launch_bounds__(G::NTHREADS, 1)
cw_naive_kernel(const NaiveArgs a, const Tables t)
{
    constexpr int KX = G::KX, KZ = G::KZ;
    constexpr int MX = G::MX, MY = G::MY, MZ = G::MZ, NR = G::NR;
    constexpr int SW = 32 + MX - 1;  // staged columns per row
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float *samp = reinterpret_cast<float *>(smem_raw);  // [MZ][MY][SW]
    float *xf = samp + MZ * MY * SW;                     // [MZ][MY][XF][32]

    const int lane = threadIdx.x & 31, r = threadIdx.x >> 5;
    const int W = a.W, H = a.H, NXB = a.NXB;
    const int rows = H - a.y_begin;
    const long long units = (long long)NXB * rows;
    const size_t HW = (size_t)W * H;
    for (long long u = blockIdx.x; u < units; u += gridDim.x) {
        const int xb = (int)(u / rows);
        const int y = a.y_begin + (int)(u % rows);
        const int x0 = xb * 32, x = x0 + lane;
        __syncthreads();
        // stage the raw window rows: frame n-mz, rows y-my, columns x0-(MX-1) ..
        for (int i = threadIdx.x; i < MZ * MY * SW; i += G::NTHREADS) {
            const int c = i % SW, my = (i / SW) % MY, mz = i / (SW * MY);
            const int yy = y - my, gx = x0 - (MX - 1) + c;
            const float *f = a.frames + (size_t)(((a.n - mz) % a.nslots + a.nslots) % a.nslots) * HW;
            samp[i] = (yy >= 0 && gx >= 0 && gx < W) ? __ldg(f + (size_t)yy * W + gx) : 0.f;
        }
        __syncthreads();
        // x DFT of every staged (frame, row) at this lane's column (_kernels.py:108-115)
        for (int fr = r; fr < MZ * MY; fr += NR) {
            float acc[G::XF];
#pragma unroll
            for (int f = 0; f < G::XF; f++) acc[f] = 0.f;
#pragma unroll
            for (int m = 0; m < MX; m++) {
                const float v = samp[fr * SW + lane + MX - 1 - m];
                acc[0] += v;
#pragma unroll
                for (int k = 1; k <= KX; k++) {
                    acc[2 * k - 1] = fmaf(t.exc[k][m], v, acc[2 * k - 1]);
                    acc[2 * k] = fmaf(t.exs[k][m], v, acc[2 * k]);
                }
            }
#pragma unroll
            for (int f = 0; f < G::XF; f++) xf[(fr * G::XF + f) * 32 + lane] = acc[f];
        }
        __syncthreads();
        const bool anchor = x < W && x >= MX - 1 && (y + a.y_off) >= MY - 1;
        auto xfv = [&](int mz, int my, int kx) -> cf {
            const float *p = xf + ((mz * MY + my) * G::XF) * 32 + lane;
            if (kx == 0) return cmk(p[0], 0.f);
            if (kx > 0) return cmk(p[(2 * kx - 1) * 32], p[(2 * kx) * 32]);
            return cmk(p[(-2 * kx - 1) * 32], -p[(-2 * kx) * 32]);
        };
        // y DFT per frame, then the temporal DFT (_kernels.py:116-127)
        float2 *st = a.state + (((size_t)y * NXB + xb) * G::NSP + G::spair(r)) * 32 + lane;
        // temporal phases e^{+j 2 pi kz mz / Mz}: w(kz)^mz with w(kz) = t.wc/ws[kz + KZ]
        auto tphase = [&](int kz, int mz) -> cf {
            const int e = ((kz * mz) % MZ + MZ) % MZ;  // w(kz)^mz = w(1)^(kz mz) = w(e)
            const int idx = e <= KZ ? e + KZ : e - MZ + KZ;
            return cmk(t.wc[idx], t.ws[idx]);
        };
        auto spectrum = [&](int kx, cf *out) {
            cf yv[MZ];
#pragma unroll
            for (int mz = 0; mz < MZ; mz++) {
                cf acc = cmk(0.f, 0.f);
#pragma unroll
                for (int my = 0; my < MY; my++)
                    acc = cmac_s(acc, cmk(t.eyc[r][my], t.eys[r][my]), xfv(mz, my, kx));
                yv[mz] = acc;
            }
#pragma unroll
            for (int kzi = 0; kzi < MZ; kzi++) {
                cf acc = cmk(0.f, 0.f);
#pragma unroll
                for (int mz = 0; mz < MZ; mz++) acc = cmac_s(acc, tphase(kzi - KZ, mz), yv[mz]);
                out[kzi] = anchor ? acc : cmk(0.f, 0.f);
            }
        };
        if (r == 0) {
            cf d[MZ];
            spectrum(0, d);  // DC bin: kz = 0 real, kz = 1..KZ
            st[0] = make_float2(d[KZ].r, 0.f);
#pragma unroll
            for (int kz = 1; kz <= KZ; kz++) st[kz * 32] = f2(d[KZ + kz]);
#pragma unroll
            for (int kx = 1; kx <= KX; kx++) {
                spectrum(kx, d);
#pragma unroll
                for (int kzi = 0; kzi < MZ; kzi++) st[(KZ + 1 + (kx - 1) * MZ + kzi) * 32] = f2(d[kzi]);
            }
        } else {
#pragma unroll
            for (int kxi = 0; kxi < MX; kxi++) {
                cf d[MZ];
                spectrum(kxi - KX, d);
#pragma unroll
                for (int kzi = 0; kzi < MZ; kzi++) st[(kxi * MZ + kzi) * 32] = f2(d[kzi]);
            }
        }
    }
}

}  // namespace cwb
