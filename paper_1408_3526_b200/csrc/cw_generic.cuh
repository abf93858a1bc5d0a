// cw_generic.cuh -- the runtime-geometry path: every validate-legal
// FilterParams (params.py:114-158) on the device.
//
// The fused kernel (cw_frame.cuh) is compiled per (KX, KY, KZ, BX, BY) with
// its state layout, shared-memory stages and lag contraction unrolled for
// that geometry (K <= 5, <= 33 lags).  Geometries outside the compiled set
// -- any window or bandwidth, any lag grid (up to 65535 entries per axis) --
// run here instead: three kernels per frame with runtime loops over the
// geometry and every per-pixel quantity in HBM as planes [plane][pixel]
// (pixel = y * W + x, so a warp's 32 columns are one coalesced access):
//
//  gen_xstage   x window sums X(kx; y, x) = sum_mx e^{+j2pi kx mx/Mx} I(y, x-mx)
//               (sdft_rows, _kernels.py:31-45, evaluated directly)
//  gen_observer y window sums u(ky, kx) = sum_my e^{+j2pi ky my/My} X(kx; y-my, x)
//               (sdft_cols, _kernels.py:48-68) and the deadbeat observer
//               over kz (replaces temporal_dft, _kernels.py:71-90): the state
//               planes hold z+ of the last frame, S = z+ / sqrt(Mx My Mz);
//               the naive backend (spectrum.py:257-327) writes the direct
//               window DFT of the last Mz frames instead
//  gen_flow     DC suppression + 3-D Hann (27-point stencil) + power + kz
//               collapse + smoothing of T^ (_kernels.py:156-271), the lag
//               contraction with the pick gains folded and the reference's
//               total-order argmax (_kernels.py:230-302), then the PEF and
//               residual of the anchor's output pixel (_kernels.py:305-342)
//               and the detection epilogue
//
// The arithmetic is float32 like the fused kernel's; the state is the full
// (not half) spectrum.  This path is for correctness over the whole
// parameter domain; the compiled geometries are the throughput path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cwb {

struct GenTables {
    const float2 *ex;    // [Mx][Mx]  e^{+j2pi kx mx / Mx}, ikx = kx + KX
    const float2 *ey;    // [My][My]
    const float2 *ez;    // [Mz][Mz]  e^{+j2pi kz mz / Mz} (naive backend)
    const float2 *w;     // [Mz]      observer rotation e^{+j2pi kz / Mz}
    const float2 *az;    // [Mz]      e^{-j2pi kz / Mz} / (Mx My Mz)  (kz collapse of |S|^2)
    const float2 *axl;   // [nlx][Mx] gx(l) e^{-j2pi kx lx / Mx}
    const float2 *ayl;   // [nly][My] gy(l) e^{-j2pi ky ly / My}
    const uint32_t *rank;  // [nly * nlx] reference total order (_kernels.py:286-298)
    const uint32_t *rix, *riy;  // rank -> (ix, iy)
    const float2 *coef;  // [nly * nlx][nc] bank / sqrt(Mx My Mz): pred = Re sum coef z+
    const int32_t *ret;  // [nc] state plane of retained bin j (design.py:195-205)
};

struct GenArgs {
    const float *frames;  // frame ring base (nslots slots of H * W)
    int nslots;
    long long n;          // index of the current frame
    const float *delayed; // frame n - mhat_z (nullptr until ready)
    float2 *xf;           // x-stage planes [nf][Mx][H*W] (nf = 1, or Mz for the naive backend)
    float2 *state;        // z+ planes [Mx*My*Mz][H*W], bin order (kz, ky, kx) as the reference's flat index
    float2 *that;         // T^ planes [My*Mx][H*W]
    float *res, *pred;    // (H, W) outputs (pred nullable)
    void *vidx;           // (H, W, 2) uint8 (idx16: uint16) velocity indices
    int idx16;
    int W, H, NXB, y_begin, y_off;
    int kx, ky, kz, mx, my, mz, nb, nlx, nly, nc, mhx, mhy;
    int ready, first, naive, forced_ix, forced_iy;
    float alpha, beta, inv_mz;
    unsigned char *det;
    float det_tau;
    int det_cap;
};

// host launchers (cw_generic.cu); all three on `s`
cudaError_t gen_launch(const GenArgs &a, const GenTables &t, int sms, cudaStream_t s);

}  // namespace cwb
