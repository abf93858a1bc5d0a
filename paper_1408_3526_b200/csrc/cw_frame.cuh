// cw_frame.cuh -- the fused per-frame kernel (sm_100a).
//
// One launch per frame runs the whole per-pixel chain of the reference
// Pipeline.process_frame (/root/reference/pkg/src/clutterwhiten/
// pipeline.py:201-294):
//
//   spatial SDFT (x: 9-tap window sums, y: comb + resonator recursion,
//                 _kernels.py:31-68)
//   temporal deadbeat observer (replaces the ring DFT, _kernels.py:71-90)
//   DC suppression + 3-D Hann + power (_kernels.py:156-227)
//   kz collapse + smoothing of T^ (81 reals, == smoothing R^ by linearity,
//                 _kernels.py:230-271)
//   lag contraction with pick gains folded + total-order argmax
//                 (_kernels.py:274-302)
//   velocity-tuned PEF on the retained band + residual (_kernels.py:305-342)
//
// Work mapping: a CTA owns 32 adjacent columns (lane = pixel
// column) and one warp per spatial-frequency row ky = 0..KY (real input =>
// conjugate symmetry, only the half space is kept).  It walks a contiguous
// run of the linearised (column-block, row) space, carrying the y-SDFT
// resonator state in registers from row to row.  Per-pixel state lives in
// HBM in "packet" layout [row*NXB + xb][float j][lane]: every warp access
// is one full 128-byte line.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cwb {

constexpr int MAXK = 5;    // largest half window supported by the tables
constexpr int MAXM = 2 * MAXK + 1;
constexpr int MAXL = 33;   // largest lag grid per axis
constexpr int RESTART = 32;  // rows between direct y-SDFT restarts (bounds f32 drift)

struct Tables {
    // x stage: cos/sin(2 pi kx m / Mx), kx = 0..KX, m = 0..Mx-1
    float exc[MAXK + 1][MAXM], exs[MAXK + 1][MAXM];
    // y stage direct restart: cos/sin(2 pi ky m / My), ky = 0..KY
    float eyc[MAXK + 1][MAXM], eys[MAXK + 1][MAXM];
    // y resonators: exp(+j 2 pi ky / My)
    float twc[MAXK + 1], tws[MAXK + 1];
    // observer rotation w(kz) = exp(+j 2 pi kz / Mz), index kz + KZ
    float wc[MAXM], ws[MAXM];
    // kz collapse a_z(kz) = exp(-j 2 pi kz / Mz), index kz + KZ
    float azc[MAXM], azs[MAXM];
    // stage 1 (gx folded): B(ky,lx) = g*T(0) + sum_kx c*A - j s*D
    float s1g[MAXL], s1c[MAXL][MAXK], s1s[MAXL][MAXK];
    // stage 2 (gy and the factor 2 folded)
    float s2g[MAXL], s2c[MAXL][MAXK], s2s[MAXL][MAXK];
    // argmax total order: rank[ly * nlx + lx]; rank -> (ix, iy)
    uint16_t rank[MAXL * MAXL];
    uint8_t rix[MAXL * MAXL], riy[MAXL * MAXL];
    float cS;      // Mz / sqrt(Mx My Mz): S = cS * xhat+
    float inv_mz;  // observer gain 1/Mz
    float alpha, beta;
    int nlx, nly;
};

struct FrameArgs {
    const float *frame;    // (H, W) current frame (local strip)
    const float *delayed;  // (H, W) frame n - mhat_z (nullptr until ready)
    float *state;          // observer state, packets [H*NXB][NS][32]
    float *that;           // smoothing state T^, packets [H*NXB][NT][32]
    const float *coefP;    // PEF coefficients [Ly*Lx][NRET]
    float *res;            // (H, W) residual out
    float *pred;           // (H, W) prediction out (nullable)
    uint8_t *vidx;         // (H, W, 2) velocity index out
    float *dbgS;           // spectrum dump, packets [H*NXB][NS][32] (nullable)
    int W, H, NXB;
    int y_begin;           // first local anchor row (strip halo)
    int y_off;             // global row of local row 0
    int ready, first;      // flow/PEF enabled; first ready frame (T^ := T)
    int forced_ix, forced_iy;  // < 0: no override
    int mhx, mhy;
};

template <int KX_, int KY_, int KZ_, int BX_, int BY_>
struct Geo {
    static constexpr int KX = KX_, KY = KY_, KZ = KZ_, BX = BX_, BY = BY_;
    static constexpr int MX = 2 * KX + 1, MY = 2 * KY + 1, MZ = 2 * KZ + 1;
    static constexpr int WX = 2 * BX + 1, WY = 2 * BY + 1;
    static constexpr int NR = KY + 1;            // warps = spatial-frequency rows
    static constexpr int NTHREADS = 32 * NR;
    static constexpr int NS = MX * MY * MZ;       // observer floats per pixel
    static constexpr int ROW0 = MZ * MX;          // ... in row ky = 0
    static constexpr int ROWN = 2 * MX * MZ;      // ... in rows ky >= 1
    static constexpr int NT = MX * MY;            // T^ floats per pixel
    static constexpr int TROW0 = MX, TROWN = 2 * MX;
    static constexpr int NRET = MZ * WX * WY;     // retained floats (== coefficient count)
    static constexpr int PROW0 = MZ * WX, PROWN = 2 * MZ * WX;
    static constexpr int RING = MY + 2;           // x-stage ring rows
    static constexpr int XF = MX;                 // x-stage floats per (row, col)
    __host__ __device__ static constexpr int srow(int r) { return r == 0 ? 0 : ROW0 + (r - 1) * ROWN; }
    __host__ __device__ static constexpr int trow(int r) { return r == 0 ? 0 : TROW0 + (r - 1) * TROWN; }
    __host__ __device__ static constexpr int prow(int r) { return r == 0 ? 0 : PROW0 + (r - 1) * PROWN; }
    // shared memory plan (floats)
    static constexpr int SM_XF = RING * XF * 32;
    static constexpr int SM_CX = NR * MZ * MX * 2 * 32;
    static constexpr int SM_BB = NR * MAXL * 2 * 32;
    static constexpr int SM_CXBB = SM_CX > SM_BB ? SM_CX : SM_BB;
    static constexpr int SM_RET = NRET * 32;
    static constexpr int SM_BEST = NR * 32 * 2;
    static constexpr int SM_PEF = (BY + 1) * 32;
    static constexpr int SMEM_FLOATS = SM_XF + SM_CXBB + SM_RET + SM_BEST + SM_PEF;
    static constexpr size_t SMEM_BYTES = sizeof(float) * SMEM_FLOATS;
};

struct cf {
    float r, i;
};
__device__ __forceinline__ cf cmk(float r, float i) { return cf{r, i}; }
__device__ __forceinline__ cf cadd(cf a, cf b) { return cf{a.r + b.r, a.i + b.i}; }
__device__ __forceinline__ cf csub(cf a, cf b) { return cf{a.r - b.r, a.i - b.i}; }
__device__ __forceinline__ cf cmul(cf a, cf b) { return cf{a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ cf cconj(cf a) { return cf{a.r, -a.i}; }
// 1/2 c - 1/4 (a + b): one tap of the circular (-1/4, 1/2, -1/4) Hann
__device__ __forceinline__ cf hann(cf a, cf c, cf b)
{
    return cf{fmaf(0.5f, c.r, -0.25f * (a.r + b.r)), fmaf(0.5f, c.i, -0.25f * (a.i + b.i))};
}

// Total order of the reference pick (_kernels.py:286-298): larger score,
// then smaller rank (rank sorts by |v|^2, then ix, then iy).
__device__ __forceinline__ bool better(float v, int rk, float best, int brk)
{
    return v > best || (v == best && rk < brk);
}

template <class G>
__global__ void __launch_bounds__(G::NTHREADS, 2)
cw_frame_kernel(const FrameArgs a, const Tables t)
{
    constexpr int KX = G::KX, KY = G::KY, KZ = G::KZ, BX = G::BX, BY = G::BY;
    constexpr int MX = G::MX, MY = G::MY, MZ = G::MZ;
    constexpr int NR = G::NR, RING = G::RING;

    extern __shared__ float smem[];
    float *xfr = smem;                      // [RING][XF][32]
    float *cxb = xfr + G::SM_XF;            // [NR][MZ][MX][2][32]   (Hy exchange)
    float *bb = cxb;                        // [NR][nlx][2][32]      (stage-1 exchange, aliased)
    float *sret = cxb + G::SM_CXBB;         // [NRET][32]            (retained xhat+)
    float *pbest = sret + G::SM_RET;        // [NR][32] score
    int *prank = reinterpret_cast<int *>(pbest + NR * 32);  // [NR][32]
    float *ppef = pbest + G::SM_BEST;       // [BY+1][32]

    const int lane = threadIdx.x & 31;
    const int r = threadIdx.x >> 5;  // spatial-frequency row ky of this warp
    const int W = a.W, H = a.H, NXB = a.NXB;
    const int rows = H - a.y_begin;
    const long long units = (long long)NXB * rows;
    const long long u0 = units * blockIdx.x / gridDim.x;
    const long long u1 = units * (blockIdx.x + 1) / gridDim.x;

#define XFR(slot, f) xfr[((slot) * G::XF + (f)) * 32 + lane]
#define CXB(rr, kzi, kxi, c) cxb[((((rr) * MZ + (kzi)) * MX + (kxi)) * 2 + (c)) * 32 + lane]

    // x stage for local row yy at column x: 9-tap windowed sums (the row
    // sweep), zero padding outside the frame.  kx = 0 real, kx > 0 complex.
    auto xstage = [&](int yy, int x, int slot) {
        float acc[G::XF];
#pragma unroll
        for (int f = 0; f < G::XF; f++) acc[f] = 0.f;
        if (yy >= 0 && yy < H) {
            const float *row = a.frame + (size_t)yy * W;
#pragma unroll
            for (int m = 0; m < MX; m++) {
                const int xx = x - m;
                const float v = (xx >= 0 && xx < W) ? __ldg(row + xx) : 0.f;
                acc[0] += v;
#pragma unroll
                for (int k = 1; k <= KX; k++) {
                    acc[2 * k - 1] = fmaf(t.exc[k][m], v, acc[2 * k - 1]);
                    acc[2 * k] = fmaf(t.exs[k][m], v, acc[2 * k]);
                }
            }
        }
#pragma unroll
        for (int f = 0; f < G::XF; f++) XFR(slot, f) = acc[f];
    };
    auto ring_slot = [&](int yy) { return ((yy % RING) + RING) % RING; };
    // x-stage value for bin kx (negative kx by conjugate symmetry)
    auto xfv = [&](int slot, int kx) -> cf {
        if (kx == 0) return cmk(XFR(slot, 0), 0.f);
        if (kx > 0) return cmk(XFR(slot, 2 * kx - 1), XFR(slot, 2 * kx));
        return cmk(XFR(slot, -2 * kx - 1), -XFR(slot, -2 * kx));
    };

    long long u = u0;
    while (u < u1) {
        const int xb = (int)(u / rows);
        const int ys = a.y_begin + (int)(u % rows);
        const long long left = u1 - u;
        const int ye = (int)((ys + left) < H ? (ys + left) : H);
        const int x = xb * 32 + lane;
        const bool colv = x < W;

        // prologue: x stage of rows ys-MY+1 .. ys (split over warps)
        __syncthreads();
        for (int k = r; k < MY; k += NR) {
            const int yy = ys - MY + 1 + k;
            xstage(yy, x, ring_slot(yy));
        }
        __syncthreads();

        // y-SDFT resonator state of this warp's row, kx = -KX..KX
        cf sp[MX];
#pragma unroll
        for (int i = 0; i < MX; i++) sp[i] = cmk(0.f, 0.f);

        for (int yy = ys; yy < ye; yy++) {
            // ---------------- phase B: spatial, observer, Hz, Hx ----------------
            if (r == 0 && yy + 1 < ye) xstage(yy + 1, x, ring_slot(yy + 1));
            if (((yy - ys) % RESTART) == 0) {
                // direct restart: sp = sum_my e^{+j 2 pi ky my / My} xf(yy - my)
#pragma unroll
                for (int i = 0; i < MX; i++) sp[i] = cmk(0.f, 0.f);
                for (int m = 0; m < MY; m++) {
                    const int sl = ring_slot(yy - m);
                    const cf e = cmk(t.eyc[r][m], t.eys[r][m]);
#pragma unroll
                    for (int i = 0; i < MX; i++) sp[i] = cadd(sp[i], cmul(e, xfv(sl, i - KX)));
                }
            } else {
                const int s1 = ring_slot(yy), s0 = ring_slot(yy - MY);
                const cf tw = cmk(t.twc[r], t.tws[r]);
#pragma unroll
                for (int i = 0; i < MX; i++) sp[i] = cadd(cmul(tw, sp[i]), csub(xfv(s1, i - KX), xfv(s0, i - KX)));
            }
            const bool anchor = colv && x >= MX - 1 && (yy + a.y_off) >= MY - 1;
            const size_t pix = (size_t)yy * NXB + xb;
            float *st = a.state + pix * G::NS * 32 + lane;
            float *dbg = a.dbgS ? a.dbgS + pix * G::NS * 32 + lane : nullptr;

            // observer + Hz: cz[kxi][kzi] (kxi = kx + KX); row 0 uses kx >= 0 only
            cf cz[MX][MZ];
            if (r == 0) {
                // DC spatial bin: real input, states kz = 0 (real) and kz = 1..KZ
                {
                    const float u0v = anchor ? sp[KX].r : 0.f;
                    float s0 = st[0];
                    cf s[KZ + 1];
#pragma unroll
                    for (int kz = 1; kz <= KZ; kz++) s[kz] = cmk(st[(1 + 2 * (kz - 1)) * 32], st[(2 + 2 * (kz - 1)) * 32]);
                    float sum = s0;
#pragma unroll
                    for (int kz = 1; kz <= KZ; kz++) sum += 2.f * s[kz].r;
                    const float e = (u0v - sum) * t.inv_mz;
                    const float xp0 = s0 + e;
                    st[0] = xp0;
                    if (BY >= 0) sret[0 * 32 + lane] = xp0;
                    if (dbg) dbg[0] = t.cS * xp0;
#pragma unroll
                    for (int kz = 1; kz <= KZ; kz++) {
                        const cf xp = cmk(s[kz].r + e, s[kz].i);
                        const cf xn = cmul(cmk(t.wc[kz + KZ], t.ws[kz + KZ]), xp);
                        st[(1 + 2 * (kz - 1)) * 32] = xn.r;
                        st[(2 + 2 * (kz - 1)) * 32] = xn.i;
                        sret[(1 + 2 * (kz - 1)) * 32 + lane] = xp.r;
                        sret[(2 + 2 * (kz - 1)) * 32 + lane] = xp.i;
                        if (dbg) {
                            dbg[(1 + 2 * (kz - 1)) * 32] = t.cS * xp.r;
                            dbg[(2 + 2 * (kz - 1)) * 32] = t.cS * xp.i;
                        }
                    }
                }
                // DC suppression (_kernels.py:167-174): C(kz, 0, 0) = 0
#pragma unroll
                for (int kzi = 0; kzi < MZ; kzi++) cz[KX][kzi] = cmk(0.f, 0.f);
#pragma unroll
                for (int kx = 1; kx <= KX; kx++) {
                    const int base = MZ + (kx - 1) * 2 * MZ;
                    const cf uv = anchor ? sp[KX + kx] : cmk(0.f, 0.f);
                    cf s[MZ];
                    cf sum = cmk(0.f, 0.f);
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        s[kzi] = cmk(st[(base + 2 * kzi) * 32], st[(base + 2 * kzi + 1) * 32]);
                        sum = cadd(sum, s[kzi]);
                    }
                    const cf e = cmk((uv.r - sum.r) * t.inv_mz, (uv.i - sum.i) * t.inv_mz);
                    cf xp[MZ];
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        xp[kzi] = cadd(s[kzi], e);
                        const cf xn = cmul(cmk(t.wc[kzi], t.ws[kzi]), xp[kzi]);
                        st[(base + 2 * kzi) * 32] = xn.r;
                        st[(base + 2 * kzi + 1) * 32] = xn.i;
                        if (kx <= BX) {
                            sret[(base + 2 * kzi) * 32 + lane] = xp[kzi].r;
                            sret[(base + 2 * kzi + 1) * 32 + lane] = xp[kzi].i;
                        }
                        if (dbg) {
                            dbg[(base + 2 * kzi) * 32] = t.cS * xp[kzi].r;
                            dbg[(base + 2 * kzi + 1) * 32] = t.cS * xp[kzi].i;
                        }
                    }
                    // Hz (temporal Hann, circular) scaled to the unitary spectrum
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        const cf h = hann(xp[(kzi + MZ - 1) % MZ], xp[kzi], xp[(kzi + 1) % MZ]);
                        cz[KX + kx][kzi] = cmk(t.cS * h.r, t.cS * h.i);
                    }
                }
                // kx < 0 by symmetry: C(kz, 0, -kx) = conj C(-kz, 0, kx)
#pragma unroll
                for (int kx = 1; kx <= KX; kx++)
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) cz[KX - kx][kzi] = cconj(cz[KX + kx][MZ - 1 - kzi]);
            } else {
                float *sr = st + G::srow(r) * 32;
                float *dr = dbg ? dbg + G::srow(r) * 32 : nullptr;
                float *rr = sret + (G::prow(r < BY + 1 ? r : 0) * 32) + lane;
#pragma unroll
                for (int kxi = 0; kxi < MX; kxi++) {
                    const int base = kxi * MZ * 2;
                    const cf uv = anchor ? sp[kxi] : cmk(0.f, 0.f);
                    cf s[MZ];
                    cf sum = cmk(0.f, 0.f);
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        s[kzi] = cmk(sr[(base + 2 * kzi) * 32], sr[(base + 2 * kzi + 1) * 32]);
                        sum = cadd(sum, s[kzi]);
                    }
                    const cf e = cmk((uv.r - sum.r) * t.inv_mz, (uv.i - sum.i) * t.inv_mz);
                    cf xp[MZ];
                    const int kxb = kxi - KX + BX;  // retained-band column
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        xp[kzi] = cadd(s[kzi], e);
                        const cf xn = cmul(cmk(t.wc[kzi], t.ws[kzi]), xp[kzi]);
                        sr[(base + 2 * kzi) * 32] = xn.r;
                        sr[(base + 2 * kzi + 1) * 32] = xn.i;
                        if (r <= BY && kxb >= 0 && kxb < G::WX) {
                            rr[((kxb * MZ + kzi) * 2) * 32] = xp[kzi].r;
                            rr[((kxb * MZ + kzi) * 2 + 1) * 32] = xp[kzi].i;
                        }
                        if (dr) {
                            dr[(base + 2 * kzi) * 32] = t.cS * xp[kzi].r;
                            dr[(base + 2 * kzi + 1) * 32] = t.cS * xp[kzi].i;
                        }
                    }
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        const cf h = hann(xp[(kzi + MZ - 1) % MZ], xp[kzi], xp[(kzi + 1) % MZ]);
                        cz[kxi][kzi] = cmk(t.cS * h.r, t.cS * h.i);
                    }
                }
            }
            if (a.ready) {
                // Hx (circular along kx), full row to shared memory
#pragma unroll
                for (int kzi = 0; kzi < MZ; kzi++)
#pragma unroll
                    for (int kxi = 0; kxi < MX; kxi++) {
                        const cf h = hann(cz[(kxi + MX - 1) % MX][kzi], cz[kxi][kzi], cz[(kxi + 1) % MX][kzi]);
                        CXB(r, kzi, kxi, 0) = h.r;
                        CXB(r, kzi, kxi, 1) = h.i;
                    }
            }
            __syncthreads();  // (1) Cx rows visible; x stage of yy+1 done
            if (!a.ready) continue;

            // ---------------- phase C1: Hy, power, kz collapse, smoothing ----------------
            cf T[MX];
            {
                const int klo = (r == 0) ? KX : 0;  // row 0: kx >= 0 only
#pragma unroll
                for (int kxi = 0; kxi < MX; kxi++) {
                    T[kxi] = cmk(0.f, 0.f);
                    if (kxi < klo) continue;
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        const cf own = cmk(CXB(r, kzi, kxi, 0), CXB(r, kzi, kxi, 1));
                        cf up, dn;
                        if (r == 0) {
                            up = cmk(CXB(1, MZ - 1 - kzi, MX - 1 - kxi, 0), -CXB(1, MZ - 1 - kzi, MX - 1 - kxi, 1));
                            dn = cmk(CXB(1, kzi, kxi, 0), CXB(1, kzi, kxi, 1));
                        } else {
                            up = cmk(CXB(r - 1, kzi, kxi, 0), CXB(r - 1, kzi, kxi, 1));
                            if (r < KY)
                                dn = cmk(CXB(r + 1, kzi, kxi, 0), CXB(r + 1, kzi, kxi, 1));
                            else
                                dn = cmk(CXB(KY, MZ - 1 - kzi, MX - 1 - kxi, 0), -CXB(KY, MZ - 1 - kzi, MX - 1 - kxi, 1));
                        }
                        const cf c = hann(up, own, dn);
                        const float p = fmaf(c.r, c.r, c.i * c.i);
                        T[kxi].r = fmaf(t.azc[kzi], p, T[kxi].r);
                        T[kxi].i = fmaf(t.azs[kzi], p, T[kxi].i);
                    }
                }
                // smoothing (_kernels.py:261-271; first ready frame copies)
                const size_t pix = (size_t)yy * NXB + xb;
                float *th = a.that + pix * G::NT * 32 + G::trow(r) * 32 + lane;
                if (r == 0) {
                    // T(0,0) real, then kx = 1..KX complex
                    float v = T[KX].r;
                    if (!a.first) v = fmaf(t.beta, v, t.alpha * th[0]);
                    th[0] = v;
                    T[KX] = cmk(v, 0.f);
#pragma unroll
                    for (int kx = 1; kx <= KX; kx++) {
                        cf v2 = T[KX + kx];
                        if (!a.first)
                            v2 = cmk(fmaf(t.beta, v2.r, t.alpha * th[(2 * kx - 1) * 32]),
                                     fmaf(t.beta, v2.i, t.alpha * th[(2 * kx) * 32]));
                        th[(2 * kx - 1) * 32] = v2.r;
                        th[(2 * kx) * 32] = v2.i;
                        T[KX + kx] = v2;
                    }
                } else {
#pragma unroll
                    for (int kxi = 0; kxi < MX; kxi++) {
                        cf v2 = T[kxi];
                        if (!a.first)
                            v2 = cmk(fmaf(t.beta, v2.r, t.alpha * th[(2 * kxi) * 32]),
                                     fmaf(t.beta, v2.i, t.alpha * th[(2 * kxi + 1) * 32]));
                        th[(2 * kxi) * 32] = v2.r;
                        th[(2 * kxi + 1) * 32] = v2.i;
                        T[kxi] = v2;
                    }
                }
            }
            __syncthreads();  // (2) all Hy reads of cxb done before bb overwrites it

            // ---------------- phase C2: stage-1 lag contraction along kx ----------------
            {
                const int nlx = t.nlx;
                if (r == 0) {
                    for (int lx = 0; lx < nlx; lx++) {
                        float b = t.s1g[lx] * T[KX].r;
#pragma unroll
                        for (int kx = 1; kx <= KX; kx++) {
                            b = fmaf(2.f * t.s1c[lx][kx - 1], T[KX + kx].r, b);
                            b = fmaf(2.f * t.s1s[lx][kx - 1], T[KX + kx].i, b);
                        }
                        bb[((0 * MAXL + lx) * 2) * 32 + lane] = b;
                    }
                } else {
                    cf A[KX + 1], D[KX + 1];
#pragma unroll
                    for (int kx = 1; kx <= KX; kx++) {
                        A[kx] = cadd(T[KX + kx], T[KX - kx]);
                        D[kx] = csub(T[KX + kx], T[KX - kx]);
                    }
                    for (int lx = 0; lx < nlx; lx++) {
                        const float g = t.s1g[lx];
                        float br = g * T[KX].r, bi = g * T[KX].i;
#pragma unroll
                        for (int kx = 1; kx <= KX; kx++) {
                            const float c = t.s1c[lx][kx - 1], s = t.s1s[lx][kx - 1];
                            br = fmaf(c, A[kx].r, fmaf(s, D[kx].i, br));
                            bi = fmaf(c, A[kx].i, fmaf(-s, D[kx].r, bi));
                        }
                        bb[((r * MAXL + lx) * 2) * 32 + lane] = br;
                        bb[((r * MAXL + lx) * 2 + 1) * 32 + lane] = bi;
                    }
                }
            }
            __syncthreads();  // (3) B(ky, lx) visible

            // ---------------- phase D: stage-2 contraction along ky + partial argmax ----------------
            {
                const int nlx = t.nlx, nly = t.nly;
                float best = -INFINITY;
                int brk = 0x7fffffff;
                for (int lx = r; lx < nlx; lx += NR) {
                    const float b0 = bb[((0 * MAXL + lx) * 2) * 32 + lane];
                    float br[KY + 1], bi[KY + 1];
#pragma unroll
                    for (int k = 1; k <= KY; k++) {
                        br[k] = bb[((k * MAXL + lx) * 2) * 32 + lane];
                        bi[k] = bb[((k * MAXL + lx) * 2 + 1) * 32 + lane];
                    }
                    for (int ly = 0; ly < nly; ly++) {
                        float v = t.s2g[ly] * b0;
#pragma unroll
                        for (int k = 1; k <= KY; k++) {
                            v = fmaf(t.s2c[ly][k - 1], br[k], v);
                            v = fmaf(t.s2s[ly][k - 1], bi[k], v);
                        }
                        const int rk = t.rank[ly * nlx + lx];
                        if (better(v, rk, best, brk)) {
                            best = v;
                            brk = rk;
                        }
                    }
                }
                pbest[r * 32 + lane] = best;
                prank[r * 32 + lane] = brk;
            }
            __syncthreads();  // (4) partial maxima visible

            // ---------------- phase E: final pick, PEF partial per row ----------------
            int vix, viy;
            {
                float best = pbest[lane];
                int brk = prank[lane];
#pragma unroll
                for (int w = 1; w < NR; w++) {
                    const float v = pbest[w * 32 + lane];
                    const int rk = prank[w * 32 + lane];
                    if (better(v, rk, best, brk)) {
                        best = v;
                        brk = rk;
                    }
                }
                if (a.forced_ix >= 0) {
                    vix = a.forced_ix;
                    viy = a.forced_iy;
                } else {
                    vix = t.rix[brk];
                    viy = t.riy[brk];
                }
            }
            if (r <= BY) {
                const float *cp = a.coefP + (size_t)(viy * t.nlx + vix) * G::NRET + G::prow(r);
                const float *sr = sret + G::prow(r) * 32 + lane;
                const int n = (r == 0) ? G::PROW0 : G::PROWN;
                float acc = 0.f;
#pragma unroll 5
                for (int j = 0; j < n; j++) acc = fmaf(__ldg(cp + j), sr[j * 32], acc);
                ppef[r * 32 + lane] = acc;
            }
            if (r == 0 && colv) {
                uint8_t *vp = a.vidx + ((size_t)yy * W + x) * 2;
                *reinterpret_cast<uchar2 *>(vp) = make_uchar2((uint8_t)vix, (uint8_t)viy);
            }
            __syncthreads();  // (5) PEF partials visible

            // ---------------- phase F: residual ----------------
            if (r == 0 && anchor) {
                float p = 0.f;
#pragma unroll
                for (int k = 0; k <= BY; k++) p += ppef[k * 32 + lane];
                const size_t o = (size_t)(yy - a.mhy) * W + (x - a.mhx);
                a.res[o] = __ldg(a.delayed + o) - p;
                if (a.pred) a.pred[o] = p;
            }
        }
        u += ye - ys;
    }
#undef XFR
#undef CXB
}

}  // namespace cwb
