// cw_inst.cuh -- compiled kernel instances (geometry x lag count) and the
// launch table the host side (cw_api.cu) dispatches through.
#pragma once
#include "cw_frame.cuh"
#include "cw_naive.cuh"

namespace cwb {

struct LaunchFn {
    // compiled instances: launch / launch_naive; run-time compiled ones
    // (cw_jit.cu): launch == nullptr, kernel / naive_kernel are cudaKernel_t
    void (*launch)(const FrameArgs &, const Tables &, int grid, cudaStream_t);
    void (*launch_naive)(const NaiveArgs &, const Tables &, int grid, cudaStream_t);
    const void *naive_kernel;
    size_t naive_smem;
    const void *kernel;
    int threads;
    size_t smem;
    int nsp, ntp, retp;  // float2 pairs per pixel: observer state, T^, retained (PEF rows padded)
    int nl;              // compiled lag count (0: runtime loops)
    int pef_l2;          // PEF reads the stored state: coefficients carry conj(w(kz))
    int compact;         // rank tables read from global memory (FrameArgs.rank_g / rxy_g)
    void (*phase_clocks)(unsigned long long *dst);  // CW_PHASE_TIMING builds: this unit's clocks
};

#ifdef CW_PHASE_TIMING
static void phase_clocks_read(unsigned long long *dst)  // [8][16] + CTA spans [2][1024][6], clocks zeroed
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(dst, cw_phase_clk, sizeof(unsigned long long) * 128);
    cudaMemcpyFromSymbol(dst + 128, cw_cta_span, sizeof(unsigned long long) * 12288);
    static unsigned long long zero[128] = {};
    cudaMemcpyToSymbol(cw_phase_clk, zero, sizeof zero);
}
#endif

// (KX, KY, KZ, BX, BY, NL): the default geometry and the SURVEY §8d C5 sweep;
// NL = 9 / 17 / 33 are the fully unrolled symmetric-grid contractions.
#ifdef CW_DEV_DEFAULT_ONLY  // dev builds (tools/dev_build.sh; CW_DEV_GEO picks the geometry)
#ifndef CW_DEV_KX  // -DCW_DEV_KX=.. -DCW_DEV_KY=.. (nvcc splits a comma list)
#define CW_DEV_KX 4
#define CW_DEV_KY 4
#define CW_DEV_KZ 2
#define CW_DEV_BX 3
#define CW_DEV_BY 3
#endif
#define CW_DEV_X(X, a, b, c, d, e) X(a, b, c, d, e, 0) X(a, b, c, d, e, 17) X(a, b, c, d, e, 33)
#define CW_DEV_X2(X, a, b, c, d, e) CW_DEV_X(X, a, b, c, d, e)
#define CW_INSTANCES(X) CW_DEV_X2(X, CW_DEV_KX, CW_DEV_KY, CW_DEV_KZ, CW_DEV_BX, CW_DEV_BY)
#else
#define CW_INSTANCES_GEO(X, a, b, c, d, e) X(a, b, c, d, e, 0) X(a, b, c, d, e, 9) X(a, b, c, d, e, 17) X(a, b, c, d, e, 33)
#define CW_INSTANCES(X)                   \
    CW_INSTANCES_GEO(X, 4, 4, 2, 3, 3)    \
    CW_INSTANCES_GEO(X, 3, 3, 2, 2, 2)    \
    CW_INSTANCES_GEO(X, 5, 5, 2, 4, 4)    \
    CW_INSTANCES_GEO(X, 4, 4, 1, 3, 3)
#endif
#define CW_INST_FN(a, b, c, d, e, n) cw_inst_##a##_##b##_##c##_##d##_##e##_##n

template <int KX, int KY, int KZ, int BX, int BY, int NL>
void launch_inst(const FrameArgs &a, const Tables &t, int grid, cudaStream_t s)
{
    using G = Geo<KX, KY, KZ, BX, BY>;
    cw_frame_kernel<G, NL><<<grid, G::NTHREADS, G::SMEM_BYTES, s>>>(a, t);
}

template <class G>
constexpr size_t naive_smem_bytes()
{
    return sizeof(float) * (G::MZ * G::MY * (32 + G::MX - 1) + G::MZ * G::MY * G::XF * 32);
}

template <int KX, int KY, int KZ, int BX, int BY>
void launch_naive_inst(const NaiveArgs &a, const Tables &t, int grid, cudaStream_t s)
{
    using G = Geo<KX, KY, KZ, BX, BY>;
    cw_naive_kernel<G><<<grid, G::NTHREADS, naive_smem_bytes<G>(), s>>>(a, t);
}

template <int KX, int KY, int KZ, int BX, int BY, int NL>
LaunchFn make_inst()
{
    using G = Geo<KX, KY, KZ, BX, BY>;
    constexpr GeoSizes gs = geo_sizes(KX, KY, KZ, BX, BY);
    static_assert(gs.threads == G::NTHREADS && gs.nsp == G::NSP && gs.ntp == G::NTP && gs.retpp == G::RETPP &&
                      gs.smem == G::SMEM_BYTES && gs.naive_smem == naive_smem_bytes<G>() &&
                      gs.compact == (G::COMPACT ? 1 : 0) && gs.pef_l2 == (G::PEF_L2 ? 1 : 0),
                  "geo_sizes() must mirror Geo");
    LaunchFn f{};
    f.launch = &launch_inst<KX, KY, KZ, BX, BY, NL>;
    if constexpr (NL == 0) {  // one naive kernel per geometry (in the NL = 0 unit)
        f.launch_naive = &launch_naive_inst<KX, KY, KZ, BX, BY>;
        f.naive_kernel = reinterpret_cast<const void *>(&cw_naive_kernel<G>);
        f.naive_smem = naive_smem_bytes<G>();
    }
    f.kernel = reinterpret_cast<const void *>(&cw_frame_kernel<G, NL>);
    f.threads = G::NTHREADS;
    f.smem = G::SMEM_BYTES;
    f.nsp = G::NSP;
    f.ntp = G::NTP;
    f.retp = G::RETPP;
    f.nl = NL;
    f.pef_l2 = G::PEF_L2 ? 1 : 0;
    f.compact = G::COMPACT ? 1 : 0;
#ifdef CW_PHASE_TIMING
    f.phase_clocks = &phase_clocks_read;
#endif
    return f;
}

}  // namespace cwb
