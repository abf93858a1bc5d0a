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
constexpr int RESTART = 32;
#ifndef CW_MINB
#define CW_MINB 2  // resident CTAs per SM the register budget is sized for
#endif  // rows between direct y-SDFT restarts (bounds f32 drift)

struct Tables {
    // x stage: cos/sin(2 pi kx m / Mx), kx = 0..KX, m = 0..Mx-1
    float exc[MAXK + 1][MAXM], exs[MAXK + 1][MAXM];
    // y stage direct restart: cos/sin(2 pi ky m / My), ky = 0..KY
    float eyc[MAXK + 1][MAXM], eys[MAXK + 1][MAXM];
    // y resonators: exp(+j 2 pi ky / My)
    float twc[MAXK + 1], tws[MAXK + 1];
    // observer rotation w(kz) = exp(+j 2 pi kz / Mz), index kz + KZ
    float wc[MAXM], ws[MAXM];
    // kz collapse a_z(kz) = exp(-j 2 pi kz / Mz), index kz + KZ, times
    // norm^2 / 4096 (the three unscaled Hann passes each carry a factor 4)
    float azc[MAXM], azs[MAXM];
    // stage 1 (gx folded): B(ky,lx) = g*T(0) + sum_kx c*A - j s*D
    float s1g[MAXL], s1c[MAXL][MAXK], s1s[MAXL][MAXK];
    // stage 2 (gy and the factor 2 folded)
    float s2g[MAXL], s2c[MAXL][MAXK], s2s[MAXL][MAXK];
    // argmax total order: rank[ly * nlx + lx]; rank -> (ix, iy)
    uint16_t rank[MAXL * MAXL];
    uint8_t rix[MAXL * MAXL], riy[MAXL * MAXL];
    float norm;    // 1/sqrt(Mx My Mz): S = norm * z+ (z = Mz * xhat, unnormalised DFT)
    float inv_mz;  // observer gain 1/Mz
    float alpha, beta;
    int nlx, nly;
    int sym_x, sym_y;  // lag grid symmetric about an exact 0 (odd length): +-l pairing
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
    static constexpr int SM_RANK = (MAXL * MAXL + 1) / 2;  // uint16 rank table
    static constexpr int SMEM_FLOATS = SM_XF + SM_CXBB + SM_RET + SM_BEST + SM_PEF + SM_RANK;
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
// 2c - (a + b) = 4 x one tap of the circular (-1/4, 1/2, -1/4) Hann
// (_kernels.py:177-217); the 4^3 is folded into the kz-collapse table.
__device__ __forceinline__ cf hann4(cf a, cf c, cf b)
{
    return cf{fmaf(2.f, c.r, -(a.r + b.r)), fmaf(2.f, c.i, -(a.i + b.i))};
}

// Total order of the reference pick (_kernels.py:286-298): larger score,
// then smaller rank (rank sorts by |v|^2, then ix, then iy).
__device__ __forceinline__ bool better(float v, int rk, float best, int brk)
{
    return v > best || (v == best && rk < brk);
}

template <class G>
__global__ void __launch_bounds__(G::NTHREADS, CW_MINB)
cw_frame_kernel(const FrameArgs a, const Tables t)
{
    constexpr int KX = G::KX, KY = G::KY, KZ = G::KZ, BX = G::BX, BY = G::BY;
    constexpr int MX = G::MX, MY = G::MY, MZ = G::MZ;
    constexpr int NR = G::NR, RING = G::RING;

    extern __shared__ float smem[];
    float *xfr = smem;                      // [RING][XF][32]       x-stage ring
    float *cxb = xfr + G::SM_XF;            // [NR][MZ][MX][2][32]  Hy exchange
    float *bb = cxb;                        // [NR][MAXL][2][32]    stage-1 exchange (aliased)
    float *sret = cxb + G::SM_CXBB;         // [NRET][32]           retained z+
    float *pbest = sret + G::SM_RET;        // [NR][32] score
    int *prank = reinterpret_cast<int *>(pbest + NR * 32);  // [NR][32]
    float *ppef = pbest + G::SM_BEST;       // [BY+1][32]
    uint16_t *srank = reinterpret_cast<uint16_t *>(ppef + G::SM_PEF);  // [nly][nlx]

    const int lane = threadIdx.x & 31;
    const int r = threadIdx.x >> 5;  // spatial-frequency row ky of this warp
    const int W = a.W, H = a.H, NXB = a.NXB;
    const int nlx = t.nlx, nly = t.nly;
    const int rows = H - a.y_begin;
    const long long units = (long long)NXB * rows;
    const long long u0 = units * blockIdx.x / gridDim.x;
    const long long u1 = units * (blockIdx.x + 1) / gridDim.x;

    for (int i = threadIdx.x; i < nlx * nly; i += G::NTHREADS) srank[i] = t.rank[i];

#define XFR(slot, f) xfr[((slot) * G::XF + (f)) * 32 + lane]
#define CXB(rr, kzi, kxi, c) cxb[((((rr) * MZ + (kzi)) * MX + (kxi)) * 2 + (c)) * 32 + lane]
#define BB(rr, lx, c) bb[(((rr) * MAXL + (lx)) * 2 + (c)) * 32 + lane]

    // x stage for local row yy at column x: Mx-tap window sums (the row
    // sweep, _kernels.py:31-45), zero outside the frame; kx = 0 real.
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
    auto xfv = [&](int slot, int kx) -> cf {
        if (kx == 0) return cmk(XFR(slot, 0), 0.f);
        if (kx > 0) return cmk(XFR(slot, 2 * kx - 1), XFR(slot, 2 * kx));
        return cmk(XFR(slot, -2 * kx - 1), -XFR(slot, -2 * kx));
    };
    // this warp's observer floats and T^ floats of pixel row yy (registers)
    const int nst = (r == 0) ? G::ROW0 : G::ROWN;
    const int nth = (r == 0) ? G::TROW0 : G::TROWN;
    float st[G::ROWN];
    float thv[G::TROWN];
    auto load_rows = [&](int yy, int xb, bool with_that) {
        const size_t pix = (size_t)yy * NXB + xb;
        const float *sp_ = a.state + (pix * G::NS + G::srow(r)) * 32 + lane;
#pragma unroll
        for (int j = 0; j < G::ROWN; j++)
            if (j < nst) st[j] = sp_[j * 32];
        if (with_that) {
            const float *tp = a.that + (pix * G::NT + G::trow(r)) * 32 + lane;
#pragma unroll
            for (int j = 0; j < G::TROWN; j++)
                if (j < nth) thv[j] = tp[j * 32];
        }
    };

    long long u = u0;
    while (u < u1) {
        const int xb = (int)(u / rows);
        const int ys = a.y_begin + (int)(u % rows);
        const long long left = u1 - u;
        const int ye = (int)((ys + left) < H ? (ys + left) : H);
        const int x = xb * 32 + lane;
        const bool colv = x < W;

        __syncthreads();  // ring reuse across chunks
        for (int k = r; k < MY; k += NR) {
            const int yy = ys - MY + 1 + k;
            xstage(yy, x, ring_slot(yy));
        }
        load_rows(ys, xb, a.ready && !a.first);
        __syncthreads();

        cf sp[MX];  // y-SDFT resonators of row ky = r, kx = -KX..KX
#pragma unroll
        for (int i = 0; i < MX; i++) sp[i] = cmk(0.f, 0.f);

        for (int yy = ys; yy < ye; yy++) {
            // ---------------- phase B: spatial SDFT, observer, Hz, Hx ----------------
            if (r == 0 && yy + 1 < ye) xstage(yy + 1, x, ring_slot(yy + 1));
            if (((yy - ys) % RESTART) == 0) {
                // direct restart sum_my e^{+j 2 pi ky my / My} xf(yy - my) (_kernels.py:58-61)
#pragma unroll
                for (int i = 0; i < MX; i++) sp[i] = cmk(0.f, 0.f);
                for (int m = 0; m < MY; m++) {
                    const int sl = ring_slot(yy - m);
                    const cf e = cmk(t.eyc[r][m], t.eys[r][m]);
#pragma unroll
                    for (int i = 0; i < MX; i++) sp[i] = cadd(sp[i], cmul(e, xfv(sl, i - KX)));
                }
            } else {
                // comb + resonator (_kernels.py:62-68)
                const int s1 = ring_slot(yy), s0 = ring_slot(yy - MY);
                const cf tw = cmk(t.twc[r], t.tws[r]);
#pragma unroll
                for (int i = 0; i < MX; i++) sp[i] = cadd(cmul(tw, sp[i]), csub(xfv(s1, i - KX), xfv(s0, i - KX)));
            }
            const bool anchor = colv && x >= MX - 1 && (yy + a.y_off) >= MY - 1;
            const size_t pix = (size_t)yy * NXB + xb;
            float *stg = a.state + (pix * G::NS + G::srow(r)) * 32 + lane;
            float *dbg = a.dbgS ? a.dbgS + (pix * G::NS + G::srow(r)) * 32 + lane : nullptr;

            // Deadbeat observer on z = Mz * xhat (state in HBM, in place):
            //   e = u - (1/Mz) sum_kz z ;  z+ = z + e ;  z <- w(kz) z+
            // z+ is exactly the reference's unnormalised temporal DFT of the
            // last Mz spatial spectra (_kernels.py:71-90, S = norm * z+).
            cf cz[MX][MZ];  // 4 x Hz(z+) per kx column
            if (r == 0) {
                {   // DC spatial bin: real input; z(0) real, z(1..KZ) complex
                    const float uv = anchor ? sp[KX].r : 0.f;
                    float sum = st[0];
#pragma unroll
                    for (int kz = 1; kz <= KZ; kz++) sum = fmaf(2.f, st[2 * kz - 1], sum);
                    const float e = fmaf(-t.inv_mz, sum, uv);
                    const float z0 = st[0] + e;
                    stg[0] = z0;
                    sret[lane] = z0;
                    if (dbg) dbg[0] = t.norm * z0;
#pragma unroll
                    for (int kz = 1; kz <= KZ; kz++) {
                        const cf zp = cmk(st[2 * kz - 1] + e, st[2 * kz]);
                        const cf zn = cmul(cmk(t.wc[kz + KZ], t.ws[kz + KZ]), zp);
                        stg[(2 * kz - 1) * 32] = zn.r;
                        stg[(2 * kz) * 32] = zn.i;
                        sret[(2 * kz - 1) * 32 + lane] = zp.r;
                        sret[(2 * kz) * 32 + lane] = zp.i;
                        if (dbg) {
                            dbg[(2 * kz - 1) * 32] = t.norm * zp.r;
                            dbg[(2 * kz) * 32] = t.norm * zp.i;
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
                    cf sum = cmk(0.f, 0.f);
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) sum = cadd(sum, cmk(st[base + 2 * kzi], st[base + 2 * kzi + 1]));
                    const cf e = cmk(fmaf(-t.inv_mz, sum.r, uv.r), fmaf(-t.inv_mz, sum.i, uv.i));
                    cf zp[MZ];
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        zp[kzi] = cmk(st[base + 2 * kzi] + e.r, st[base + 2 * kzi + 1] + e.i);
                        const cf zn = (kzi == KZ) ? zp[kzi] : cmul(cmk(t.wc[kzi], t.ws[kzi]), zp[kzi]);
                        stg[(base + 2 * kzi) * 32] = zn.r;
                        stg[(base + 2 * kzi + 1) * 32] = zn.i;
                        if (kx <= BX) {
                            sret[(base + 2 * kzi) * 32 + lane] = zp[kzi].r;
                            sret[(base + 2 * kzi + 1) * 32 + lane] = zp[kzi].i;
                        }
                        if (dbg) {
                            dbg[(base + 2 * kzi) * 32] = t.norm * zp[kzi].r;
                            dbg[(base + 2 * kzi + 1) * 32] = t.norm * zp[kzi].i;
                        }
                    }
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++)
                        cz[KX + kx][kzi] = hann4(zp[(kzi + MZ - 1) % MZ], zp[kzi], zp[(kzi + 1) % MZ]);
                }
                // kx < 0 by symmetry: C(kz, 0, -kx) = conj C(-kz, 0, kx)
#pragma unroll
                for (int kx = 1; kx <= KX; kx++)
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) cz[KX - kx][kzi] = cconj(cz[KX + kx][MZ - 1 - kzi]);
            } else {
                float *rr = sret + G::prow(r <= BY ? r : 0) * 32 + lane;
#pragma unroll
                for (int kxi = 0; kxi < MX; kxi++) {
                    const int base = kxi * MZ * 2;
                    const cf uv = anchor ? sp[kxi] : cmk(0.f, 0.f);
                    cf sum = cmk(0.f, 0.f);
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) sum = cadd(sum, cmk(st[base + 2 * kzi], st[base + 2 * kzi + 1]));
                    const cf e = cmk(fmaf(-t.inv_mz, sum.r, uv.r), fmaf(-t.inv_mz, sum.i, uv.i));
                    cf zp[MZ];
                    const int kxb = kxi - KX + BX;  // retained-band column
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        zp[kzi] = cmk(st[base + 2 * kzi] + e.r, st[base + 2 * kzi + 1] + e.i);
                        const cf zn = (kzi == KZ) ? zp[kzi] : cmul(cmk(t.wc[kzi], t.ws[kzi]), zp[kzi]);
                        stg[(base + 2 * kzi) * 32] = zn.r;
                        stg[(base + 2 * kzi + 1) * 32] = zn.i;
                        if (r <= BY && kxb >= 0 && kxb < G::WX) {
                            rr[((kxb * MZ + kzi) * 2) * 32] = zp[kzi].r;
                            rr[((kxb * MZ + kzi) * 2 + 1) * 32] = zp[kzi].i;
                        }
                        if (dbg) {
                            dbg[(base + 2 * kzi) * 32] = t.norm * zp[kzi].r;
                            dbg[(base + 2 * kzi + 1) * 32] = t.norm * zp[kzi].i;
                        }
                    }
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++)
                        cz[kxi][kzi] = hann4(zp[(kzi + MZ - 1) % MZ], zp[kzi], zp[(kzi + 1) % MZ]);
                }
            }
            if (a.ready) {
                // Hx (circular along kx), full row to shared memory
#pragma unroll
                for (int kzi = 0; kzi < MZ; kzi++)
#pragma unroll
                    for (int kxi = 0; kxi < MX; kxi++) {
                        const cf h = hann4(cz[(kxi + MX - 1) % MX][kzi], cz[kxi][kzi], cz[(kxi + 1) % MX][kzi]);
                        CXB(r, kzi, kxi, 0) = h.r;
                        CXB(r, kzi, kxi, 1) = h.i;
                    }
            }
            __syncthreads();  // (1) Cx rows visible; x stage of yy+1 done

            // ---------------- phase C1: Hy, power, kz collapse, smoothing ----------------
            cf T[MX];
            if (a.ready) {
                const int klo = (r == 0) ? KX : 0;  // row 0: kx >= 0 only
#pragma unroll
                for (int kxi = 0; kxi < MX; kxi++) {
                    T[kxi] = cmk(0.f, 0.f);
                    if (kxi < klo) continue;
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        const cf own = cmk(CXB(r, kzi, kxi, 0), CXB(r, kzi, kxi, 1));
                        cf up, dn;
                        if (r == 0) {  // row -1 = conj-flip of row 1
                            up = cmk(CXB(1, MZ - 1 - kzi, MX - 1 - kxi, 0), -CXB(1, MZ - 1 - kzi, MX - 1 - kxi, 1));
                            dn = cmk(CXB(1, kzi, kxi, 0), CXB(1, kzi, kxi, 1));
                        } else {
                            up = cmk(CXB(r - 1, kzi, kxi, 0), CXB(r - 1, kzi, kxi, 1));
                            if (r < KY)
                                dn = cmk(CXB(r + 1, kzi, kxi, 0), CXB(r + 1, kzi, kxi, 1));
                            else  // row KY+1 == -KY = conj-flip of row KY
                                dn = cmk(CXB(KY, MZ - 1 - kzi, MX - 1 - kxi, 0), -CXB(KY, MZ - 1 - kzi, MX - 1 - kxi, 1));
                        }
                        const cf c = hann4(up, own, dn);
                        const float p = fmaf(c.r, c.r, c.i * c.i);
                        T[kxi].r = fmaf(t.azc[kzi], p, T[kxi].r);
                        T[kxi].i = fmaf(t.azs[kzi], p, T[kxi].i);
                    }
                }
                // smoothing of T^ (_kernels.py:261-271; first ready frame copies)
                float *th = a.that + (pix * G::NT + G::trow(r)) * 32 + lane;
                if (r == 0) {
                    float v = T[KX].r;
                    if (!a.first) v = fmaf(t.beta, v, t.alpha * thv[0]);
                    th[0] = v;
                    T[KX] = cmk(v, 0.f);
#pragma unroll
                    for (int kx = 1; kx <= KX; kx++) {
                        cf v2 = T[KX + kx];
                        if (!a.first)
                            v2 = cmk(fmaf(t.beta, v2.r, t.alpha * thv[2 * kx - 1]), fmaf(t.beta, v2.i, t.alpha * thv[2 * kx]));
                        th[(2 * kx - 1) * 32] = v2.r;
                        th[(2 * kx) * 32] = v2.i;
                        T[KX + kx] = v2;
                    }
                } else {
#pragma unroll
                    for (int kxi = 0; kxi < MX; kxi++) {
                        cf v2 = T[kxi];
                        if (!a.first)
                            v2 = cmk(fmaf(t.beta, v2.r, t.alpha * thv[2 * kxi]), fmaf(t.beta, v2.i, t.alpha * thv[2 * kxi + 1]));
                        th[(2 * kxi) * 32] = v2.r;
                        th[(2 * kxi + 1) * 32] = v2.i;
                        T[kxi] = v2;
                    }
                }
            }
            // prefetch the next row's observer and T^ rows (consumed after the
            // remaining phases: hides the HBM latency behind them)
            if (yy + 1 < ye) load_rows(yy + 1, xb, a.ready && !a.first);
            if (!a.ready) continue;
            __syncthreads();  // (2) Hy reads of cxb done before bb overwrites it

            // ---------------- phase C2: stage-1 lag contraction along kx ----------------
            // B(ky, lx) = gx(lx) sum_kx e^{-j 2 pi kx lx / Mx} T^(ky, kx)
            if (t.sym_x) {
                const int c0 = nlx >> 1;  // lag 0; lags +-p at c0 +- p
                if (r == 0) {
                    for (int q = 0; q <= c0; q++) {
                        const int lx = c0 + q;
                        float cp = t.s1g[lx] * T[KX].r, sp2 = 0.f;
#pragma unroll
                        for (int kx = 1; kx <= KX; kx++) {
                            cp = fmaf(2.f * t.s1c[lx][kx - 1], T[KX + kx].r, cp);
                            sp2 = fmaf(2.f * t.s1s[lx][kx - 1], T[KX + kx].i, sp2);
                        }
                        BB(0, c0 + q, 0) = cp + sp2;
                        BB(0, c0 - q, 0) = cp - sp2;
                    }
                } else {
                    cf A[KX + 1], D[KX + 1];
#pragma unroll
                    for (int kx = 1; kx <= KX; kx++) {
                        A[kx] = cadd(T[KX + kx], T[KX - kx]);
                        D[kx] = csub(T[KX + kx], T[KX - kx]);
                    }
                    for (int q = 0; q <= c0; q++) {
                        const int lx = c0 + q;
                        const float g = t.s1g[lx];
                        float cr = g * T[KX].r, ci = g * T[KX].i, sr = 0.f, si = 0.f;
#pragma unroll
                        for (int kx = 1; kx <= KX; kx++) {
                            const float c = t.s1c[lx][kx - 1], s = t.s1s[lx][kx - 1];
                            cr = fmaf(c, A[kx].r, cr);
                            ci = fmaf(c, A[kx].i, ci);
                            sr = fmaf(s, D[kx].i, sr);
                            si = fmaf(-s, D[kx].r, si);
                        }
                        BB(r, c0 + q, 0) = cr + sr;
                        BB(r, c0 + q, 1) = ci + si;
                        BB(r, c0 - q, 0) = cr - sr;
                        BB(r, c0 - q, 1) = ci - si;
                    }
                }
            } else {
                if (r == 0) {
                    for (int lx = 0; lx < nlx; lx++) {
                        float b = t.s1g[lx] * T[KX].r;
#pragma unroll
                        for (int kx = 1; kx <= KX; kx++) {
                            b = fmaf(2.f * t.s1c[lx][kx - 1], T[KX + kx].r, b);
                            b = fmaf(2.f * t.s1s[lx][kx - 1], T[KX + kx].i, b);
                        }
                        BB(0, lx, 0) = b;
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
                        BB(r, lx, 0) = br;
                        BB(r, lx, 1) = bi;
                    }
                }
            }
            __syncthreads();  // (3) B(ky, lx) visible

            // ---------------- phase D: stage-2 contraction along ky + partial argmax ----------------
            // score(ly, lx) = gy gx R^(ly, lx) = s2g B0 + sum_ky s2c Re B + s2s Im B
            {
                float best = -INFINITY;
                int brk = 0x7fffffff;
                for (int lx = r; lx < nlx; lx += NR) {
                    const float b0 = BB(0, lx, 0);
                    float br[KY + 1], bi[KY + 1];
#pragma unroll
                    for (int k = 1; k <= KY; k++) {
                        br[k] = BB(k, lx, 0);
                        bi[k] = BB(k, lx, 1);
                    }
                    if (t.sym_y) {
                        // visit ly = 0, -1, +1, -2, +2, ...: ascending rank order within
                        // a column (|v|^2 grows with |ly|, then iy ascending), so a
                        // strict '>' keeps the reference's tie winner (_kernels.py:286-298)
                        const int c0 = nly >> 1;
                        float cb = t.s2g[c0] * b0;
#pragma unroll
                        for (int k = 1; k <= KY; k++) cb = fmaf(t.s2c[c0][k - 1], br[k], cb);
                        int ci = c0;
                        for (int q = 1; q <= c0; q++) {
                            const int ly = c0 + q;
                            float e = t.s2g[ly] * b0, o = 0.f;
#pragma unroll
                            for (int k = 1; k <= KY; k++) {
                                e = fmaf(t.s2c[ly][k - 1], br[k], e);
                                o = fmaf(t.s2s[ly][k - 1], bi[k], o);
                            }
                            const float vm = e - o, vp = e + o;
                            if (vm > cb) { cb = vm; ci = c0 - q; }
                            if (vp > cb) { cb = vp; ci = ly; }
                        }
                        const int rk = srank[ci * nlx + lx];
                        if (better(cb, rk, best, brk)) { best = cb; brk = rk; }
                    } else {
                        for (int ly = 0; ly < nly; ly++) {
                            float v = t.s2g[ly] * b0;
#pragma unroll
                            for (int k = 1; k <= KY; k++) {
                                v = fmaf(t.s2c[ly][k - 1], br[k], v);
                                v = fmaf(t.s2s[ly][k - 1], bi[k], v);
                            }
                            const int rk = srank[ly * nlx + lx];
                            if (better(v, rk, best, brk)) { best = v; brk = rk; }
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
                    if (better(v, rk, best, brk)) { best = v; brk = rk; }
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
                // PEF on the retained band (_kernels.py:330-342), folded to the
                // stored half space: pred = sum_j coef[v][j] * z+[j]
                const float *cp = a.coefP + (size_t)(viy * nlx + vix) * G::NRET + G::prow(r);
                const float *sr = sret + G::prow(r) * 32 + lane;
                const int n = (r == 0) ? G::PROW0 : G::PROWN;
                float acc0 = 0.f, acc1 = 0.f;
#pragma unroll 10
                for (int j = 0; j < n; j += 2) {
                    acc0 = fmaf(__ldg(cp + j), sr[j * 32], acc0);
                    if (j + 1 < n) acc1 = fmaf(__ldg(cp + j + 1), sr[(j + 1) * 32], acc1);
                }
                ppef[r * 32 + lane] = acc0 + acc1;
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
#undef BB
}

}  // namespace cwb
