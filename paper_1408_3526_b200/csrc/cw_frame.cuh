// cw_frame.cuh -- the fused per-frame kernel (sm_100a).
//
// One launch per frame runs the whole per-pixel chain of the reference
// Pipeline.process_frame (/root/reference/pkg/src/clutterwhiten/
// pipeline.py:201-294):
//
//   spatial SDFT (x: Mx-tap window sums, y: comb + resonator recursion,
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
// column) and KY+1 warps (real input => conjugate symmetry, only the half
// space is kept).  It walks a contiguous run of the linearised (column-block,
// row) space, carrying the y-SDFT resonator state in registers from row to
// row.  The owner of the work changes between phases: in the SDFT/observer
// phase warp r owns spatial-frequency row ky = r (Hz, Hx in registers); in
// the Hy/power/T^ phase it owns the columns kx = +-r over all rows (each Cx
// value read once from shared memory); in the contraction it owns two lag
// column pairs, processed jointly.
//
// Per-pixel state lives in HBM as "packets": for a (row, 32-column block),
// the observer state is float2 P[pair][lane] (re/im pairs, lane-minor), so
// one (row, block) is a single contiguous 52 KB span.  Each row's packet is
// brought into shared memory by TMA bulk copies (cp.async.bulk + mbarrier)
// issued as soon as the previous row has released the buffer; the observer
// writes the updated state straight back to HBM with 256-byte coalesced
// stores and overwrites the staged copy in place with the Hann-conditioned
// spectrum that the neighbouring rows need.  Per row: 4 CTA barriers.
#pragma once
#ifdef __CUDACC_RTC__
// run-time compiled (NVRTC, cw_jit.cu): no host headers, libcu++ instead
#include <cuda/std/cstdint>
#include <cuda/std/type_traits>
typedef cuda::std::uint8_t uint8_t;
typedef cuda::std::uint16_t uint16_t;
typedef cuda::std::uint32_t uint32_t;
typedef cuda::std::uint64_t uint64_t;
typedef cuda::std::int64_t int64_t;
namespace std {
using cuda::std::integral_constant;
}
#ifndef INFINITY
#define INFINITY __int_as_float(0x7f800000)
#endif
#else
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#endif

namespace cwb {

constexpr int MAXK = 5;    // largest half window supported by the tables
constexpr int MAXM = 2 * MAXK + 1;
constexpr int MAXL = 33;   // largest lag grid per axis
constexpr int LREC = (1 + 2 * MAXK + 3) / 4 * 4;  // floats per lag coefficient record
#ifndef CW_RESTART
#define CW_RESTART 64
#endif
constexpr int RESTART = CW_RESTART;  // rows between direct y-SDFT restarts (bounds f32 drift)
#ifndef CW_MEMONLY
#define CW_MEMONLY 0  // diagnostic build: state / T^ / frame / output traffic only (tools: memory floor)
#endif
#ifndef CW_L2ONLY
#define CW_L2ONLY 0  // diagnostic build: each CTA reuses one private packet (L2-resident state: the compute floor)
#endif
#ifndef CW_ST_NA
#define CW_ST_NA 1  // state / T^ stores with L1::no_allocate
#endif
#ifndef CW_TMA_CHUNKS
#define CW_TMA_CHUNKS 1  // bulk copies per state packet (1: one copy per row, measured fastest)
#endif
#ifndef CW_PEF_L2
// PEF reads the retained z+ back from the state row just written to HBM
// (an L2 hit; z+ = conj(w) z, conj(w) folded into the coefficients on the
// host) instead of a 32 KB retained-z+ stage in shared memory
#define CW_PEF_L2 0
#endif
#ifndef CW_SBULK
// updated observer state written into the staged packet in place and sent
// to HBM by TMA bulk stores (one per kx column of a row) instead of STG
#define CW_SBULK 0
#endif
#ifndef CW_TBULK
// T^ write-back as one TMA bulk store of the smoothed T^ stage (issued after
// barrier 2 by the issuing thread) instead of per-warp STG
#define CW_TBULK 0
#endif
#ifndef CW_FENCE_ALL
#define CW_FENCE_ALL 1  // every thread orders its generic stage reads before the next TMA write
#endif
#ifndef CW_JQ_WIDE
#define CW_JQ_WIDE 1  // lag column pairs per contraction group for grids of more than 17 lags (2: 1.73 vs 1.27 ms, C5 lag 1/8)
#endif
#ifndef CW_PQ_UNROLL_WIDE
#define CW_PQ_UNROLL_WIDE 16  // unroll of the stage-2 lag loop for grids of more than 17 lags
#endif
#ifndef CW_ARGMAX_ONLY
#define CW_ARGMAX_ONLY 0  // diagnostic build: stage-2 lag scores without their FMAs (what a tensor-core contraction would leave)
#endif
#ifndef CW_EARLY_PREROLL
#define CW_EARLY_PREROLL 1  // chained launches: first run's x-stage pre-roll before the wait for the previous frame
#endif
#ifndef CW_SMSP_17
#define CW_SMSP_17 1  // the 17-lag grid too: one pair per group, dealt by smsp_sched (C3 -1.7%, C2 -4.5%, C5 -1.4..-2.6%)
#endif
#ifndef CW_SMSP_FIX
#define CW_SMSP_FIX 1  // smsp_sched: pair counts that also balance the SM-mate CTA (5 warps; C3 -0.8%)
#endif
#ifndef CW_SMSP_9
#define CW_SMSP_9 0  // the 9-lag grid too
#endif
#ifndef CW_SMSP_SCHED
#define CW_SMSP_SCHED 1  // grids of more than 17 lags: lag column pairs dealt by scheduler load (smsp_sched)
#endif
#ifndef CW_ROLL_WIDE
#define CW_ROLL_WIDE 1  // the group loop of grids of more than 17 lags is not unrolled (instruction cache)
#endif

// Lag column pairs of a symmetric grid (q = 0..C0; q = 0 is the centre
// column) dealt to the NR warps of a CTA by scheduler load: warp w issues
// on sub-partition w % 4, so with NR = 5 warps 0 and NR-1 share one
// scheduler in every phase, and the SM-mate CTA's warp w issues on
// (w + 1) % 4.  Greedy: each pair goes to the warp whose scheduler has the
// least work (the last warp carries the next row's x stage as half a
// pair), ties to the warp with fewer pairs, within per-warp caps that also
// balance the SM-mate's copy (CW_SMSP_FIX).  33 lags, 5 warps: pairs
// 2/4/5/4/2 instead of round robin's 4/4/3/3/3.  Per warp a list of q, 5 bits each,
// terminated by 31, one 32-bit word per warp (at most 6 pairs).
struct SmspSched {
    unsigned int code[8];
    bool ok;
};
__host__ __device__ constexpr SmspSched smsp_sched(int c0, int nr)
{
    SmspSched s{};
    int n[8] = {}, load2[4] = {};  // pairs per warp; scheduler load in half pairs
    for (int w = 0; w < 8; w++) s.code[w] = ~0u;
    s.ok = nr >= 2 && nr <= 8 && c0 < 31;
    if (!s.ok) return s;
    int cap[8] = {7, 7, 7, 7, 7, 7, 7, 7};  // pairs per warp at most
    if (CW_SMSP_FIX && nr == 5 && (c0 == 16 || c0 == 8)) {
        // counts that also balance the SM-mate CTA's schedulers (its warp w
        // issues on (w + 1) % 4): 33 lags 2/4/5/4/2, 17 lags 1/2/3/2/1
        const int c16[5] = {2, 4, 5, 4, 2}, c8[5] = {1, 2, 3, 2, 1};
        for (int w = 0; w < 5; w++) cap[w] = c0 == 16 ? c16[w] : c8[w];
    }
    load2[(nr - 1) % 4] += 1;
    for (int q = 0; q <= c0; q++) {
        int b = -1;
        for (int w = 0; w < nr; w++) {
            if (n[w] >= cap[w]) continue;
            if (b < 0) {
                b = w;
                continue;
            }
            const int lw = load2[w % 4], lb = load2[b % 4];
            if (lw < lb || (lw == lb && n[w] < n[b])) b = w;
        }
        if (b < 0 || n[b] >= 6) {
            s.ok = false;
            return s;
        }
        s.code[b] &= ~(31u << (5 * n[b]));
        s.code[b] |= (unsigned int)q << (5 * n[b]);
        n[b]++;
        load2[b % 4] += 2;
    }
    return s;
}

struct alignas(16) LagRec {
    float gain, pad;
    float2 cs[MAXK];  // cs[k - 1] = (cos, sin) coefficient of frequency k
};
static_assert(sizeof(LagRec) == 4 * LREC, "lag record layout");

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
    // the same constants as (re, im) pairs for the packed f32x2 paths:
    // ex2 = (exc, exs); w2 = (wc, ws), wn2 = (-ws, wc); az2 = (azc, azs);
    // tw2 / twn2 likewise for the y resonators
    float2 ex2[MAXK + 1][MAXM];
    float2 w2[MAXM], wn2[MAXM], az2[MAXM];
    float2 tw2[MAXK + 1], twn2[MAXK + 1];
    // lag-contraction coefficients, one 16-byte aligned record per lag
    // (LagRec: gain, then the (cos, sin) pair of each frequency k = 1..MAXK).
    // stage 1 (gx folded): B(ky,lx) = g*T(0) + sum_kx c*A - j s*D
    // stage 2 (gy and the factor 2 folded): R = g B0 + sum_ky c Re B + s Im B
    LagRec s1v[MAXL];
    LagRec s2v[MAXL];
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
    float2 *state;         // observer state packets [H*NXB][NSP][32]
    float2 *that;          // smoothing state T^ packets [H*NXB][NTP][32]
    const float2 *coefP;   // PEF coefficients [Ly*Lx][RETPP] (rows padded to even pair counts)
    float *res;            // (H, W) residual out
    float *pred;           // (H, W) prediction out (nullable)
    uint8_t *vidx;         // (H, W, 2) velocity index out
    int W, H, NXB;
    int y_begin;           // first local anchor row (strip halo)
    int y_off;             // global row of local row 0
    int ready, first;      // flow/PEF enabled; first ready frame (T^ := T)
    int forced_ix, forced_iy;  // < 0: no override
    // work split: the first static_units (column-block, row) units are dealt
    // out in equal contiguous runs, the rest in dyn_chunk-row chunks that
    // CTAs claim from work[parity] (atomic counter; the kernel zeroes
    // work[parity ^ 1] for the next launch): CTAs that run slower (die,
    // L2-slice distance, SM-mate) take fewer chunks, so they all end together
    unsigned int *work;
    int parity;
    const uint16_t *rank_g;  // compact-mode instances: rank table [nly * nlx] ...
    const uint8_t *rxy_g;    // ... and rank -> (ix, iy) pairs, in global memory
    long long static_units;
    int dyn_chunk;
    int mhx, mhy;
    // detection epilogue (nullable): 64-byte header {u32 count; u64 peak
    // key; -; u64 n valid}, f64 sum res^2 per (local row, column block)
    // [H * NXB], then float4 (x, y, res, 0) x det_cap
    unsigned char *det;
    float det_tau;  // |res| >= det_tau is a detection (<= 0: list off)
    int det_cap;
    // frame chaining: CTA i of a launch works on exactly the (column block,
    // row) units CTA i of the previous launch worked on (static split, same
    // grid), so it needs only that CTA's packets: it waits for
    // done[i] >= seq - 1 before its first state / T^ / output access and
    // publishes done[i] = seq when it is through.  With programmatic
    // dependent launch (cw_api.cu) the next frame's CTAs start in the SM
    // slots this frame's early finishers free, instead of after its last CTA.
    unsigned int *done;  // [grid] (nullable: no chaining)
    unsigned int seq;
    // chained pushes of device frames: `frame` is the caller's buffer and the
    // kernel copies it into this ring slot itself (a share per CTA, once
    // every CTA of launch seq - 2 is through: the slot's previous frame and
    // the delayed frame are then no longer / already written), so no copy
    // sits between consecutive frame kernels (nullable)
    float *ring_dst;
    // chained cw_submit: the frame upload and the previous download of this
    // output set signal completion by stream memory writes (cw_api.cu)
    // instead of events the kernel's stream would wait on; the kernel waits
    // for up_flag >= up_want and down_flag >= down_want (nullable)
    const unsigned int *up_flag, *down_flag;
    unsigned int up_want, down_want;
    // the delayed frame's ring slot filled by a flagged copy (resident
    // frames, copy engine): wait for ring_flag >= ring_want (nullable)
    const unsigned int *ring_flag;
    unsigned int ring_want;
};

// Fused "final threshold" and the ground-truth-free metrics of
// cli.compute_metrics_row (cli.py:157-208): detections |res| >= tau, the peak
// |res| (ties -> first pixel in row-major order, as np.argmax) and sum res^2
// over the valid outputs.  One warp (the residual lanes of a CTA row).
__device__ __forceinline__ void detect_epilogue(const FrameArgs &a, bool valid, int ox, int oy, float res)
{
    unsigned int *count = reinterpret_cast<unsigned int *>(a.det);
    unsigned long long *peak = reinterpret_cast<unsigned long long *>(a.det + 8);
    unsigned long long *nval = reinterpret_cast<unsigned long long *>(a.det + 24);
    // sum res^2 per (row, 32-column block) slot, summed on the host in a
    // fixed order: the metric is bit-reproducible run to run
    double *sumsq = reinterpret_cast<double *>(a.det + 64);
    float4 *list = reinterpret_cast<float4 *>(a.det + 64 + 8 * (size_t)a.H * a.NXB);
    const float v = fabsf(res);
    if (valid && a.det_tau > 0.f && v >= a.det_tau) {
        const unsigned int slot = atomicAdd(count, 1u);
        if (slot < (unsigned int)a.det_cap) list[slot] = make_float4((float)ox, (float)oy, res, 0.f);
    }
    unsigned long long key =
        valid ? ((unsigned long long)__float_as_uint(v) << 32) | (0xffffffffull - (unsigned long long)((size_t)oy * a.W + ox))
              : 0ull;
    double sq = valid ? (double)res * (double)res : 0.0;  // exact square, as f64(res)**2
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(0xffffffffu, key, o);
        key = k2 > key ? k2 : key;
        sq += __shfl_xor_sync(0xffffffffu, sq, o);
    }
    const unsigned int nv = __popc(__ballot_sync(0xffffffffu, valid));
    if ((threadIdx.x & 31) == 0 && nv) {
        atomicMax(peak, key);
        sumsq[(size_t)(oy + a.mhy) * a.NXB + (ox + a.mhx) / 32] = sq;
        atomicAdd(nval, (unsigned long long)nv);
    }
}

template <int KX_, int KY_, int KZ_, int BX_, int BY_>
struct Geo {
    static constexpr int KX = KX_, KY = KY_, KZ = KZ_, BX = BX_, BY = BY_;
    static constexpr int MX = 2 * KX + 1, MY = 2 * KY + 1, MZ = 2 * KZ + 1;
    static constexpr int WX = 2 * BX + 1, WY = 2 * BY + 1;
    static constexpr int NR = KY + 1;            // warps = spatial-frequency rows
    static constexpr int NTHREADS = 32 * NR;
    // observer state pairs per pixel: row 0 = DC bin (kz = 0 real + pad,
    // kz = 1..KZ) + kx = 1..KX (all kz); rows >= 1 = MX * MZ
    static constexpr int ROW0P = (KZ + 1) + KX * MZ;
    static constexpr int ROWNP = MX * MZ;
    static constexpr int NSP = ROW0P + KY * ROWNP;
    // T^ pairs: row 0 = T(0,0) real + pad, kx = 1..KX; rows >= 1 = MX
    static constexpr int TROW0P = KX + 1, TROWNP = MX;
    static constexpr int NTP = TROW0P + KY * TROWNP;
    // retained z+ pairs (== PEF coefficient pairs)
    static constexpr int PROW0P = (KZ + 1) + BX * MZ, PROWNP = WX * MZ;
    static constexpr int RETP = PROW0P + BY * PROWNP;
    // the same rows padded to even pair counts: 16-byte (2-pair) coefficient
    // loads and (re, im, re, im) retained-z+ quads in shared memory
    static constexpr int PROW0Q = (PROW0P + 1) / 2, PROWNQ = (PROWNP + 1) / 2;  // quads per row
    static constexpr int RETPP = 2 * (PROW0Q + BY * PROWNQ);                    // padded pairs
    // x-stage ring rows: yy - MY (comb) .. yy; the next row's x stage reuses
    // the slot of yy - MY once phase B of yy is past (barrier-ordered)
    static constexpr int RING = MY + 1;
    static constexpr int XF = MX;                 // x-stage floats per (row, col)
    __host__ __device__ static constexpr int spair(int r) { return r == 0 ? 0 : ROW0P + (r - 1) * ROWNP; }
    __host__ __device__ static constexpr int tpair(int r) { return r == 0 ? 0 : TROW0P + (r - 1) * TROWNP; }
    __host__ __device__ static constexpr int ppair(int r) { return r == 0 ? 0 : PROW0P + (r - 1) * PROWNP; }
    __host__ __device__ static constexpr int pquad(int r) { return r == 0 ? 0 : PROW0Q + (r - 1) * PROWNQ; }
    // shared memory plan (bytes)
    static constexpr int SM_STAGE = NSP * 32 * 8;     // state packet -> Cx in place
    static constexpr int SM_TSTAGE = NTP * 32 * 8;    // T^ packet
    static constexpr int SM_RET_FULL = RETPP * 32 * 8;  // retained z+ quads
    static constexpr int SM_XF = RING * XF * 32 * 4;  // x-stage ring
    static constexpr int SM_BEST = NR * 32 * 8;       // partial argmax (score, rank)
    static constexpr int SM_PEF = (BY + 1) * 32 * 4;
    static constexpr int SM_RANK_FULL = ((MAXL * MAXL * 4) + 15) / 16 * 16;  // rank u16 + (ix, iy) u8 pairs
    static constexpr int SM_ROW = ((32 + MX - 1) * 4 + 15) / 16 * 16;  // next frame row segment
    static constexpr int SM_DEL = 32 * 4;                               // delayed-frame values
    static constexpr int SM_BAR = 16;
    static constexpr size_t SMEM_BASE = SM_STAGE + SM_TSTAGE + SM_XF + SM_BEST + SM_PEF + SM_ROW + SM_DEL + SM_BAR;
    // Compact mode: when the full plan keeps the SM at one CTA but dropping
    // the retained-z+ stage (PEF reads z+ back from the state row in L2,
    // conj(w) folded into the coefficients) and the smem rank table (read
    // from global) fits two, the second CTA is worth more than both
    // (e.g. (4,4,3,3,3): 1.61 -> 1.49 ms per 1280x1024 frame); C3's geometry
    // already fits two.  Not for KY >= 5: at two CTAs the 168-register cap
    // spills its contraction ((5,5,2,4,4): 1.55 -> 1.74 ms, measured).
    static constexpr bool fits2(size_t b) { return 2 * (b + 1024 + 64) <= 228 * 1024; }
    static constexpr bool COMPACT =
        KY <= 4 && !fits2(SMEM_BASE + SM_RET_FULL + SM_RANK_FULL) && fits2(SMEM_BASE);
    static constexpr bool PEF_L2 = CW_PEF_L2 || COMPACT;
    static constexpr int SM_RET = PEF_L2 ? 0 : SM_RET_FULL;
    static constexpr int SM_RANK = COMPACT ? 0 : SM_RANK_FULL;
    static constexpr size_t SMEM_BYTES = SMEM_BASE + SM_RET + SM_RANK;
    // resident CTAs per SM the register budget is sized for: as many as the
    // 228 KB of shared memory hold (1 KB reserved per CTA), at most 3
    static constexpr int MINB_SMEM = (int)((228 * 1024) / (SMEM_BYTES + 1024));
#ifdef CW_FORCE_MINB  // experiments: the register budget of CW_FORCE_MINB CTAs per SM
    static constexpr int MINB = CW_FORCE_MINB;
#else
    static constexpr int MINB = MINB_SMEM < 1 ? 1 : (MINB_SMEM > 3 ? 3 : MINB_SMEM);
#endif
};

// The sizes of Geo<kx, ky, kz, bx, by> as runtime values (for geometries
// compiled at run time, cw_jit.cu); make_inst checks them against Geo for
// every compiled instance.
struct GeoSizes {
    int threads, nsp, ntp, retpp;
    unsigned long long smem, naive_smem;
    int compact, pef_l2;
};
__host__ __device__ constexpr GeoSizes geo_sizes(int kx, int ky, int kz, int bx, int by)
{
    const int mx = 2 * kx + 1, my = 2 * ky + 1, mz = 2 * kz + 1, wx = 2 * bx + 1;
    const int nr = ky + 1;
    const int row0p = (kz + 1) + kx * mz, rownp = mx * mz;
    const int nsp = row0p + ky * rownp;
    const int ntp = (kx + 1) + ky * mx;
    const int prow0p = (kz + 1) + bx * mz, prownp = wx * mz;
    const int retpp = 2 * ((prow0p + 1) / 2 + by * ((prownp + 1) / 2));
    const unsigned long long base = (unsigned long long)nsp * 256 + (unsigned long long)ntp * 256 +
                                    (unsigned long long)(my + 1) * mx * 128 + nr * 256 + (by + 1) * 128 +
                                    ((32 + mx - 1) * 4 + 15) / 16 * 16 + 128 + 16;
    const unsigned long long ret = (unsigned long long)retpp * 256, rank = ((MAXL * MAXL * 4) + 15) / 16 * 16;
    const bool compact =
        ky <= 4 && !(2 * (base + ret + rank + 1024 + 64) <= 228 * 1024) && 2 * (base + 1024 + 64) <= 228 * 1024;
    const bool pef_l2 = CW_PEF_L2 || compact;
    const unsigned long long smem = base + (pef_l2 ? 0 : ret) + (compact ? 0 : rank);
    const unsigned long long naive = 4ull * (mz * my * (32 + mx - 1) + mz * my * mx * 32);
    return GeoSizes{32 * nr, nsp, ntp, retpp, smem, naive, compact ? 1 : 0, pef_l2 ? 1 : 0};
}

struct cf {
    float r, i;
};
__device__ __forceinline__ cf cmk(float r, float i) { return cf{r, i}; }
__device__ __forceinline__ cf c2(float2 v) { return cf{v.x, v.y}; }
__device__ __forceinline__ float2 f2(cf v) { return make_float2(v.r, v.i); }
// Complex arithmetic on packed f32x2 (sm_100 FADD2 / FMUL2 / FFMA2: one
// instruction for the re and im lanes; scalar operands broadcast for free).
__device__ __forceinline__ unsigned long long pk(cf a)
{
    unsigned long long v;
    asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(a.r), "f"(a.i));
    return v;
}
__device__ __forceinline__ cf upk(unsigned long long v)
{
    cf a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.r), "=f"(a.i) : "l"(v));
    return a;
}
__device__ __forceinline__ cf cadd(cf a, cf b)
{
    unsigned long long r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
__device__ __forceinline__ cf csub(cf a, cf b)
{
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)));
    return upk(r);
}
// lane-wise a * b + c
__device__ __forceinline__ cf cfma2(cf a, cf b, cf c)
{
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(a)), "l"(pk(b)), "l"(pk(c)));
    return upk(r);
}
__device__ __forceinline__ cf cmul(cf a, cf b)
{
    // (a.r b.r - a.i b.i, a.r b.i + a.i b.r) = a.r (b.r, b.i) + a.i (-b.i, b.r)
    unsigned long long t;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(cf{a.r, a.r})), "l"(pk(b)));
    return cfma2(cf{a.i, a.i}, cf{-b.i, b.r}, upk(t));
}
// z * w for a constant w supplied as the pairs w = (wr, wi), wn = (-wi, wr):
// z.r (wr, wi) + z.i (-wi, wr), two packed instructions
__device__ __forceinline__ cf cmulw(cf z, float2 w, float2 wn)
{
    unsigned long long t;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(cf{z.r, z.r})), "l"(pk(cf{w.x, w.y})));
    return cfma2(cf{z.i, z.i}, cf{wn.x, wn.y}, upk(t));
}
// lane-wise a * b
__device__ __forceinline__ cf cmul2(cf a, cf b)
{
    unsigned long long t;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(pk(a)), "l"(pk(b)));
    return upk(t);
}
__device__ __forceinline__ cf cconj(cf a) { return cf{a.r, -a.i}; }
// (a + b) - 2c = -4 x one tap of the circular (-1/4, 1/2, -1/4) Hann
// (_kernels.py:177-217), exactly the negation of 2c - (a + b): the three
// passes give -H C, whose power is bit-identical; the 4^3 is folded into
// the kz-collapse table.  Two packed instructions per complex bin.
__device__ __forceinline__ cf hann4(cf a, cf c, cf b)
{
    return cfma2(cf{-2.f, -2.f}, c, cadd(a, b));
}

// Total order of the reference pick (_kernels.py:286-298): larger score,
// then smaller rank (rank sorts by |v|^2, then ix, then iy).
__device__ __forceinline__ bool better(float v, int rk, float best, int brk)
{
    return v > best || (v == best && rk < brk);
}

// ---- TMA bulk copy + mbarrier (PTX) ----------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
// frame chaining (FrameArgs::done): acquire-wait on this CTA's flag, bounded
// (a lost flag traps instead of hanging the GPU)
__device__ __forceinline__ void chain_wait(const unsigned int *flag, unsigned int want)
{
    unsigned int v, ns = 32;
    for (long long it = 0;; it++) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flag) : "memory");
        if ((int)(v - want) >= 0) break;
        if (it > (1ll << 24)) asm volatile("trap;");
        __nanosleep(ns);
        ns = ns < 256 ? 2 * ns : 256;
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");  // later TMA reads see the acquired writes
}
__device__ __forceinline__ void chain_publish(unsigned int *flag, unsigned int v)
{
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(smem_addr(bar)), "r"(phase)
            : "memory");
    } while (!ok);
}

#ifdef CW_PHASE_TIMING
// per-warp clock64 accumulators (phase-timing builds only): [warp][event]
__device__ unsigned long long cw_phase_clk[8][16];
// per-CTA %globaltimer (ns) at kernel entry and exit, last launch: [cta][2]
// [seq & 1][CTA]: start, setup done, ring copy done, pre-roll done, chain wait done, end
__device__ unsigned long long cw_cta_span[2][1024][6];
__device__ __forceinline__ unsigned long long cw_gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    return t;
}
// the "memory" clobber pins each stamp between the surrounding barriers and
// shared-memory accesses (a plain clock64() may be moved across them)
__device__ __forceinline__ unsigned long long cw_clock_pinned()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}
#define CW_STAMP(k)                                   \
    do {                                              \
        const unsigned long long now = cw_clock_pinned(); \
        clk_acc[k] += now - clk_prev;                 \
        clk_prev = now;                               \
    } while (0)
#else
#define CW_STAMP(k) \
    do {            \
    } while (0)
#endif

// state / T^ write-back: streaming stores that do not allocate in L1 (keep
// the ~28 KB of L1 next to the shared memory for the PEF coefficients)
__device__ __forceinline__ void st_state(float2 *p, float2 v)
{
#if CW_ST_NA
    asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y));
#else
    *p = v;
#endif
}

__device__ __forceinline__ float4 ldg_coef4(const float4 *p) { return __ldg(p); }

// TMA bulk store shared -> global (bulk_group), its commit and the wait for
// the shared-memory source to be read (the buffer may be overwritten then)
__device__ __forceinline__ void tma_store(void *dst, const void *src, uint32_t bytes)
{
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// 4-byte cp.async (LDGSTS) with zero fill when !valid (src-size 0)
__device__ __forceinline__ void cp_async4(void *dst, const float *src, bool valid)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <class G, int NL>
__global__ void __launch_bounds__(G::NTHREADS, G::MINB)
cw_frame_kernel(const FrameArgs a, const Tables t)
{
#ifdef CW_PHASE_TIMING
    unsigned long long clk_prev = cw_clock_pinned();
    unsigned long long clk_acc[11] = {};
    if (threadIdx.x == 0 && blockIdx.x < 1024) cw_cta_span[a.seq & 1][blockIdx.x][0] = cw_gtimer();
#endif
    constexpr int KX = G::KX, KY = G::KY, KZ = G::KZ, BX = G::BX, BY = G::BY;
    constexpr int MX = G::MX, MY = G::MY, MZ = G::MZ;
    constexpr int NR = G::NR, RING = G::RING;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2 *stage = reinterpret_cast<float2 *>(smem_raw);                       // [NSP][32]
    float2 *tstage = reinterpret_cast<float2 *>(smem_raw + G::SM_STAGE);        // [NTP][32]
    float2 *sret = reinterpret_cast<float2 *>(smem_raw + G::SM_STAGE + G::SM_TSTAGE);  // [RETPP][32]
    float *xfr = reinterpret_cast<float *>(smem_raw + G::SM_STAGE + G::SM_TSTAGE + G::SM_RET);
    float2 *pbest = reinterpret_cast<float2 *>(smem_raw + G::SM_STAGE + G::SM_TSTAGE + G::SM_RET + G::SM_XF);
    float *ppef = reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(pbest) + G::SM_BEST);
    uint16_t *srank_s = reinterpret_cast<uint16_t *>(reinterpret_cast<unsigned char *>(ppef) + G::SM_PEF);
    float *rowbuf = reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(srank_s) + G::SM_RANK);
    float *delbuf = reinterpret_cast<float *>(reinterpret_cast<unsigned char *>(rowbuf) + G::SM_ROW);
    uint64_t *bar = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(delbuf) + G::SM_DEL);

    const int lane = threadIdx.x & 31;
    const int r = threadIdx.x >> 5;  // spatial-frequency row ky of this warp
    const int W = a.W, H = a.H, NXB = a.NXB;
    const int nlx = NL ? NL : t.nlx, nly = NL ? NL : t.nly;
    const int rows = H - a.y_begin;
    const long long units = (long long)NXB * rows;
    const long long su = a.work ? a.static_units : units;
    long long u = su * blockIdx.x / gridDim.x;
    long long u1 = su * (blockIdx.x + 1) / gridDim.x;
    __shared__ long long s_claim;
    const bool use_that = a.ready && !a.first;

    // rank table and rank -> (ix, iy): shared memory, or (compact mode) the
    // copy the host keeps in global memory (L1-cached)
    const uint16_t *srank = G::COMPACT ? a.rank_g : srank_s;
    const uint8_t *srxy = G::COMPACT ? a.rxy_g : reinterpret_cast<const uint8_t *>(srank_s + MAXL * MAXL);
    if (!G::COMPACT) {
        uint8_t *sxy = reinterpret_cast<uint8_t *>(srank_s + MAXL * MAXL);
        for (int i = threadIdx.x; i < nlx * nly; i += G::NTHREADS) {
            srank_s[i] = t.rank[i];
            sxy[2 * i] = t.rix[i];
            sxy[2 * i + 1] = t.riy[i];
        }
    }
    const float2 tw_r = t.tw2[threadIdx.x >> 5], twn_r = t.twn2[threadIdx.x >> 5];  // this warp's y resonator
    uint64_t *bar_t = bar + 1;  // bar: observer-state packet, bar_t: T^ packet
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        mbar_init(bar_t, 1);
        fence_mbar_init();
    }
    if (a.work && blockIdx.x == 0 && threadIdx.x == 0) a.work[a.parity ^ 1] = 0u;
    // the next frame's launch may start now (it waits on done[] per CTA)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef CW_PHASE_TIMING
    if (threadIdx.x == 0 && blockIdx.x < 1024) cw_cta_span[a.seq & 1][blockIdx.x][1] = cw_gtimer();
#endif
    if ((a.up_flag || a.down_flag || a.ring_flag) && threadIdx.x == G::NTHREADS - 32) {
        if (a.up_flag) chain_wait(a.up_flag, a.up_want);
        if (a.down_flag) chain_wait(a.down_flag, a.down_want);
        if (a.ring_flag) chain_wait(a.ring_flag, a.ring_want);
    }
    if (a.ring_dst) {
        // every CTA of launch seq - 2 through: all flags read at once (relaxed,
        // then a fence before the barrier: acquire for the whole CTA), retried
        // while one is behind -- one L2 round trip, not one per flag
        for (long long it = 0;; it++) {
            bool ok = true;
            for (int j = threadIdx.x; j < (int)gridDim.x; j += G::NTHREADS) {
                unsigned int v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.done + j) : "memory");
                ok = ok && (int)(v - (a.seq - 2u)) >= 0;
            }
            __threadfence();
            if (__syncthreads_and(ok)) break;
            if (it > (1ll << 22)) asm volatile("trap;");
            __nanosleep(256);
        }
        // this CTA's share of the frame, 16-byte vectors when aligned; all
        // loads of a thread issued before its stores (a handful per thread).
        // (Writing each CTA's own units' pixels per row from the x-stage row
        // segments instead measured slower: the store lands on warp KY's
        // critical path.)
        const size_t n = (size_t)W * H;
        if ((n & 3) == 0 && ((reinterpret_cast<uintptr_t>(a.frame) | reinterpret_cast<uintptr_t>(a.ring_dst)) & 15) == 0) {
            const size_t n4 = n / 4, b0 = n4 * blockIdx.x / gridDim.x, b1 = n4 * (blockIdx.x + 1) / gridDim.x;
            const float4 *src = reinterpret_cast<const float4 *>(a.frame);
            float4 *dst = reinterpret_cast<float4 *>(a.ring_dst);
            constexpr int U = 4;
            for (size_t i = b0 + threadIdx.x; i < b1; i += U * G::NTHREADS) {
                float4 v[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const size_t k = i + (size_t)u * G::NTHREADS;
                    if (k < b1) v[u] = __ldg(src + k);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const size_t k = i + (size_t)u * G::NTHREADS;
                    if (k < b1) dst[k] = v[u];
                }
            }
        } else {
            const size_t b0 = n * blockIdx.x / gridDim.x, b1 = n * (blockIdx.x + 1) / gridDim.x;
            for (size_t i = b0 + threadIdx.x; i < b1; i += G::NTHREADS) a.ring_dst[i] = __ldg(a.frame + i);
        }
    }
#ifdef CW_PHASE_TIMING
    if (threadIdx.x == 0 && blockIdx.x < 1024) cw_cta_span[a.seq & 1][blockIdx.x][2] = cw_gtimer();
#endif
    // the TMA issuer waits for this CTA's units of the previous frame -- here,
    // or (CW_EARLY_PREROLL) after the first run's x-stage pre-roll, which
    // reads only the current frame (wide lag grids: the plain order, which
    // their register allocation prefers)
    constexpr bool EARLY = CW_EARLY_PREROLL && NL <= 17;
    bool chain_pending = EARLY && a.done != nullptr;
    if (!EARLY && a.done && threadIdx.x == G::NTHREADS - 32) chain_wait(a.done + blockIdx.x, a.seq - 1u);
    __syncthreads();
    uint32_t phase = 0, phase_t = 0;

    // one elected thread stages the (row, block) packets of the next row;
    // the state and T^ packets are freed at different barriers
    constexpr int ISSUER = G::NTHREADS - 32;  // lane 0 of warp KY: no PEF work, fewest lag columns
    auto issue = [&](int yy, int xb) {
        if (threadIdx.x == ISSUER) {
            const size_t pix = CW_L2ONLY ? (size_t)blockIdx.x : (size_t)yy * NXB + xb;
            fence_proxy_async();  // prior generic smem accesses before the async-proxy writes
            constexpr uint32_t bs = G::NSP * 32 * 8;
            mbar_expect_tx(bar, bs);
            const unsigned char *src = reinterpret_cast<const unsigned char *>(a.state + pix * G::NSP * 32);
            constexpr uint32_t CH = (bs / CW_TMA_CHUNKS + 15) / 16 * 16;
            for (uint32_t off = 0; off < bs; off += CH)
                tma_load(reinterpret_cast<unsigned char *>(stage) + off, src + off, (bs - off) < CH ? (bs - off) : CH,
                         bar);
        }
    };
    auto issue_t = [&](int yy, int xb) {
        if (use_that && threadIdx.x == ISSUER) {
            const size_t pix = CW_L2ONLY ? (size_t)blockIdx.x : (size_t)yy * NXB + xb;
            if (CW_TBULK) tma_store_wait_read();  // the T^ store has read the stage
            fence_proxy_async();
            mbar_expect_tx(bar_t, G::SM_TSTAGE);
            tma_load(tstage, a.that + pix * G::NTP * 32, G::SM_TSTAGE, bar_t);
        }
    };

#define XFR(slot, f) xfr[((slot) * G::XF + (f)) * 32 + lane]

    // x stage: Mx-tap window sums of a frame row at this lane's column (the
    // row sweep, _kernels.py:31-45), zero outside the frame; kx = 0 real,
    // kx >= 1 accumulated as packed (cos, sin) pairs
    auto xsum_store = [&](int slot, auto &&sample) {
        float dc = 0.f;
        cf acc[KX + 1];
#pragma unroll
        for (int k = 1; k <= KX; k++) acc[k] = cmk(0.f, 0.f);
#pragma unroll
        for (int m = 0; m < MX; m++) {
            const float v = sample(m);
            dc += v;
#pragma unroll
            for (int k = 1; k <= KX; k++) acc[k] = cfma2(c2(t.ex2[k][m]), cf{v, v}, acc[k]);
        }
        XFR(slot, 0) = dc;
#pragma unroll
        for (int k = 1; k <= KX; k++) {
            XFR(slot, 2 * k - 1) = acc[k].r;
            XFR(slot, 2 * k) = acc[k].i;
        }
    };
    // for local row yy from global memory (prologue / warm-up frames)
    auto xstage = [&](int yy, int x, int slot) {
        const bool rv = yy >= 0 && yy < H;
        const float *row = a.frame + (size_t)(rv ? yy : 0) * W;
        xsum_store(slot, [&](int m) {
            const int xx = x - m;
            return (rv && xx >= 0 && xx < W) ? __ldg(row + xx) : 0.f;
        });
    };
    // from the row segment prefetched into rowbuf (cp.async):
    // rowbuf[i] = frame[row][x0 - (MX-1) + i], zero outside the frame
    auto xstage_s = [&](int slot) { xsum_store(slot, [&](int m) { return rowbuf[lane + MX - 1 - m]; }); };
    auto prefetch_row = [&](int yy, int x0) {  // async: the next row's 32 + MX - 1 samples
        const bool rv = yy >= 0 && yy < H;
        const float *row = a.frame + (size_t)(rv ? yy : 0) * W;
        for (int i = lane; i < 32 + MX - 1; i += 32) {
            const int gx = x0 - (MX - 1) + i;
            const bool v = rv && gx >= 0 && gx < W;
            cp_async4(rowbuf + i, v ? row + gx : a.frame, v);
        }
    };
    auto ring_slot = [&](int yy) { return ((yy % RING) + RING) % RING; };
    auto xfv = [&](int slot, int kx) -> cf {
        if (kx == 0) return cmk(XFR(slot, 0), 0.f);
        if (kx > 0) return cmk(XFR(slot, 2 * kx - 1), XFR(slot, 2 * kx));
        return cmk(XFR(slot, -2 * kx - 1), -XFR(slot, -2 * kx));
    };
    // Cx of row rr at (kz, kx), any kx: row 0 is stored compact (kx >= 0)
    auto cx_at = [&](int rr, int kz, int kx) -> cf {
        if (rr == 0) {
            if (kx == 0) {
                const cf v = c2(stage[(kz >= 0 ? kz : -kz) * 32 + lane]);
                return kz >= 0 ? v : cconj(v);
            }
            if (kx > 0) return c2(stage[(KZ + 1 + (kx - 1) * MZ + (kz + KZ)) * 32 + lane]);
            return cconj(c2(stage[(KZ + 1 + (-kx - 1) * MZ + (-kz + KZ)) * 32 + lane]));
        }
        return c2(stage[(G::spair(rr) + (kx + KX) * MZ + (kz + KZ)) * 32 + lane]);
    };

    for (;;) {
        if (u >= u1) {  // static run done: claim the next dynamic chunk
            if (!a.work) break;
            if (threadIdx.x == 0) {
                const unsigned int k = atomicAdd(a.work + a.parity, 1u);
                s_claim = su + (long long)k * a.dyn_chunk;
            }
            __syncthreads();
            u = s_claim;
            if (u >= units) break;
            u1 = u + a.dyn_chunk < units ? u + a.dyn_chunk : units;
        }
        const int xb = (int)(u / rows);
        const int ys = a.y_begin + (int)(u % rows);
        const long long left = u1 - u;
        const int ye = (int)((ys + left) < H ? (ys + left) : H);
        const int x = xb * 32 + lane;
        const bool colv = x < W;

        if (CW_FENCE_ALL) fence_proxy_async();
        __syncthreads();  // previous chunk done with the stage and the ring
        if (!chain_pending) {
            issue(ys, xb);
            issue_t(ys, xb);
        }
        for (int k = r; k < MY; k += NR) {
            const int yy = ys - MY + 1 + k;
            xstage(yy, x, ring_slot(yy));
        }
        if (chain_pending) {  // first run: the packets after the previous frame's
            if (threadIdx.x == G::NTHREADS - 32) {
#ifdef CW_PHASE_TIMING
                if (blockIdx.x < 1024) cw_cta_span[a.seq & 1][blockIdx.x][3] = cw_gtimer();
#endif
                chain_wait(a.done + blockIdx.x, a.seq - 1u);
#ifdef CW_PHASE_TIMING
                if (blockIdx.x < 1024) cw_cta_span[a.seq & 1][blockIdx.x][4] = cw_gtimer();
#endif
            }
            issue(ys, xb);
            issue_t(ys, xb);
            chain_pending = false;
        }
        __syncthreads();

        cf sp[MX];  // y-SDFT resonators of row ky = r, kx = -KX..KX
#pragma unroll
        for (int i = 0; i < MX; i++) sp[i] = cmk(0.f, 0.f);

        for (int yy = ys; yy < ye; yy++) {
            // ---------------- phase B: spatial SDFT, observer, Hz, Hx ----------------
            CW_STAMP(0);  // previous row's tail (phase F / loop) -> here
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
#pragma unroll
                for (int i = 0; i < MX; i++) sp[i] = cadd(cmulw(sp[i], tw_r, twn_r), csub(xfv(s1, i - KX), xfv(s0, i - KX)));
            }
            const bool anchor = colv && x >= MX - 1 && (yy + a.y_off) >= MY - 1;
            const size_t pix = CW_L2ONLY ? (size_t)blockIdx.x : (size_t)yy * NXB + xb;
            float2 *stg = a.state + (pix * G::NSP + G::spair(r)) * 32 + lane;
            float2 *sst = stage + G::spair(r) * 32 + lane;
            CW_STAMP(1);  // x stage + y SDFT
            mbar_wait(bar, phase);
            CW_STAMP(2);  // state TMA wait
            phase ^= 1;

            // Deadbeat observer on z = Mz * xhat (state in HBM, in place):
            //   e = u - (1/Mz) sum_kz z ;  z+ = z + e ;  z <- w(kz) z+
            // z+ is exactly the reference's unnormalised temporal DFT of the
            // last Mz spatial spectra (_kernels.py:71-90, S = norm * z+).
            // retained z+ (the PEF input), pair q of the padded layout
            auto rput = [&](int q, cf v) {
                if (!G::PEF_L2) sret[q * 32 + lane] = f2(v);
            };
            cf cz[MX][MZ];  // 4 x Hz(z+) per kx column
            // state write-back: STG, or (SBULK) in place + bulk stores of pairs
            // [j0, j1) of this warp's row once the warp has written them
            constexpr bool SBULK = CW_SBULK && !G::PEF_L2;
            auto put_state = [&](int j, float2 v) {
                if (SBULK) sst[j * 32] = v;
                else st_state(&stg[j * 32], v);
            };
            auto flush_state = [&](int j0, int j1) {
                if (SBULK) {
                    fence_proxy_async();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store(stg - lane + j0 * 32, sst - lane + j0 * 32, (uint32_t)(j1 - j0) * 256);
                        tma_store_commit();
                    }
                }
            };
            auto flush_wait = [&]() {  // the bulk stores have read the row: it may be overwritten
                if (SBULK) {
                    if (lane == 0) tma_store_wait_read();
                    __syncwarp();
                }
            };
            if (CW_MEMONLY == 2) {  // diagnostic: the same traffic, state written back by one bulk store
                if (threadIdx.x == ISSUER) {
                    tma_store(a.state + pix * G::NSP * 32, stage, G::SM_STAGE);
                    tma_store_commit();
                    tma_store_wait_read();
                }
            } else if (CW_MEMONLY) {  // diagnostic: the same HBM traffic, no arithmetic
                const int np = r == 0 ? G::ROW0P : G::ROWNP;
                for (int j = 0; j < np; j++) st_state(&stg[j * 32], sst[j * 32]);
            } else if (r == 0) {
                {   // DC spatial bin: real input; z(0) real, z(1..KZ) complex
                    const float uv = anchor ? sp[KX].r : 0.f;
                    cf zd[KZ + 1];
#pragma unroll
                    for (int kz = 0; kz <= KZ; kz++) zd[kz] = c2(sst[kz * 32]);
                    float sum = zd[0].r;
#pragma unroll
                    for (int kz = 1; kz <= KZ; kz++) sum = fmaf(2.f, zd[kz].r, sum);
                    const float e = fmaf(-t.inv_mz, sum, uv);
                    const float z0 = zd[0].r + e;
                    put_state(0, make_float2(z0, 0.f));
                    rput(0, cmk(z0, 0.f));
#pragma unroll
                    for (int kz = 1; kz <= KZ; kz++) {
                        const cf zp = cmk(zd[kz].r + e, zd[kz].i);
                        put_state(kz, f2(cmulw(zp, t.w2[kz + KZ], t.wn2[kz + KZ])));
                        rput(kz, zp);
                    }
                }
                // DC suppression (_kernels.py:167-174): C(kz, 0, 0) = 0
#pragma unroll
                for (int kzi = 0; kzi < MZ; kzi++) cz[KX][kzi] = cmk(0.f, 0.f);
#pragma unroll
                for (int kx = 1; kx <= KX; kx++) {
                    const int base = KZ + 1 + (kx - 1) * MZ;
                    const cf uv = anchor ? sp[KX + kx] : cmk(0.f, 0.f);
                    cf z[MZ];
                    cf sum = cmk(0.f, 0.f);
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        z[kzi] = c2(sst[(base + kzi) * 32]);
                        sum = cadd(sum, z[kzi]);
                    }
                    const cf e = cfma2(cf{-t.inv_mz, -t.inv_mz}, sum, uv);
                    cf zp[MZ];
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        zp[kzi] = cadd(z[kzi], e);
                        const cf zn = (kzi == KZ) ? zp[kzi] : cmulw(zp[kzi], t.w2[kzi], t.wn2[kzi]);
                        put_state(base + kzi, f2(zn));
                        if (kx <= BX) rput(base + kzi, zp[kzi]);
                    }
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++)
                        cz[KX + kx][kzi] = hann4(zp[(kzi + MZ - 1) % MZ], zp[kzi], zp[(kzi + 1) % MZ]);
                }
                if (G::PROW0P & 1) rput(G::PROW0P, cmk(0.f, 0.f));  // pad pair (zero coefficient)
                flush_state(0, G::ROW0P);
                // kx < 0 by symmetry: C(kz, 0, -kx) = conj C(-kz, 0, kx)
#pragma unroll
                for (int kx = 1; kx <= KX; kx++)
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) cz[KX - kx][kzi] = cconj(cz[KX + kx][MZ - 1 - kzi]);
                flush_wait();
                if (a.ready) {
                    // Hx, compact row 0 in place: kx = 0 (kz = 0..KZ), kx = 1..KX (all kz)
#pragma unroll
                    for (int kz = 0; kz <= KZ; kz++) {
                        const cf h = hann4(cz[KX - 1][kz + KZ], cz[KX][kz + KZ], cz[KX + 1][kz + KZ]);
                        sst[kz * 32] = kz == 0 ? make_float2(h.r, 0.f) : f2(h);
                    }
#pragma unroll
                    for (int kx = 1; kx <= KX; kx++)
#pragma unroll
                        for (int kzi = 0; kzi < MZ; kzi++) {
                            const int kxi = KX + kx;
                            const cf h = hann4(cz[kxi - 1][kzi], cz[kxi][kzi], cz[(kxi + 1) % MX][kzi]);
                            sst[(KZ + 1 + (kx - 1) * MZ + kzi) * 32] = f2(h);
                        }
                }
            } else {
                const int rq = G::pquad(r <= BY ? r : 0);  // this row's first retained quad
#pragma unroll
                for (int kxi = 0; kxi < MX; kxi++) {
                    const cf uv = anchor ? sp[kxi] : cmk(0.f, 0.f);
                    cf z[MZ];
                    cf sum = cmk(0.f, 0.f);
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        z[kzi] = c2(sst[(kxi * MZ + kzi) * 32]);
                        sum = cadd(sum, z[kzi]);
                    }
                    const cf e = cfma2(cf{-t.inv_mz, -t.inv_mz}, sum, uv);
                    cf zp[MZ];
                    const int kxb = kxi - KX + BX;  // retained-band column
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        zp[kzi] = cadd(z[kzi], e);
                        const cf zn = (kzi == KZ) ? zp[kzi] : cmulw(zp[kzi], t.w2[kzi], t.wn2[kzi]);
                        put_state(kxi * MZ + kzi, f2(zn));
                        if (r <= BY && kxb >= 0 && kxb < G::WX) rput(2 * rq + kxb * MZ + kzi, zp[kzi]);
                    }
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++)
                        cz[kxi][kzi] = hann4(zp[(kzi + MZ - 1) % MZ], zp[kzi], zp[(kzi + 1) % MZ]);
                    flush_state(kxi * MZ, (kxi + 1) * MZ);
                }
                if (r <= BY && (G::PROWNP & 1)) rput(2 * rq + G::PROWNP, cmk(0.f, 0.f));  // pad pair
                flush_wait();
                if (a.ready) {
                    // Hx (circular along kx), in place over this row's staged state
#pragma unroll
                    for (int kxi = 0; kxi < MX; kxi++)
#pragma unroll
                        for (int kzi = 0; kzi < MZ; kzi++) {
                            const cf h = hann4(cz[(kxi + MX - 1) % MX][kzi], cz[kxi][kzi], cz[(kxi + 1) % MX][kzi]);
                            sst[(kxi * MZ + kzi) * 32] = f2(h);
                        }
                }
            }
            if (CW_FENCE_ALL && !a.ready) fence_proxy_async();  // stage reads before the next TMA write
            CW_STAMP(3);  // observer + Hz + Hx
            // the previous row's T^ bulk store has read the stage before C1
            // overwrites it (first ready frame: no T^ load orders it)
            if (CW_TBULK && threadIdx.x == ISSUER) tma_store_wait_read();
            __syncthreads();  // (1) Cx rows visible; x stage of yy+1 done
            CW_STAMP(4);  // barrier 1 wait
            if (!a.ready) {  // warm-up frame: spectrum state only
                if (yy + 1 < ye) {
                    issue(yy + 1, xb);  // stage free: next row's state
                    if (r == KY) xstage(yy + 1, x, ring_slot(yy + 1));  // over slot yy - MY, read in B
                }
                __syncthreads();  // the x stage of yy + 1 visible to the next row's phase B
                continue;
            }

            // async prefetches consumed at the end of CD (x stage of yy+1) and in F (residual)
            if (r == KY && yy + 1 < ye) prefetch_row(yy + 1, xb * 32);
            if (r == 0) {
                const size_t o = (size_t)(yy - a.mhy) * W + (x - a.mhx);
                cp_async4(delbuf + lane, anchor ? a.delayed + o : a.frame, anchor);
            }
            // ---------------- phase C1: Hy, power, kz collapse, smoothing ----------------
            // Column ownership (a transpose through shared memory): warp r owns
            // the spatial-frequency columns kx = +-c, c = r, r + NR, ..., over
            // all rows ky, so Hy reads every Cx value once (rows were owned in
            // phase B, where Hx ran in registers).  Its T^ values go to HBM
            // and, in place, to the T^ stage every warp reads in phase CD.
            {
                if (use_that) {  // T^ packet staged (TMA issued after barrier 3 of the last row)
                    mbar_wait(bar_t, phase_t);
                    phase_t ^= 1;
                }
                float2 *thg = a.that + pix * G::NTP * 32 + lane;
                // smoothing of T^ (_kernels.py:261-271; first ready frame copies)
                auto smooth = [&](int j, cf v2) {
                    if (!a.first) {
                        const float2 o = tstage[j * 32 + lane];
                        v2 = cfma2(cf{t.beta, t.beta}, v2, cmul2(cf{t.alpha, t.alpha}, c2(o)));
                    }
                    if (!CW_TBULK) st_state(&thg[j * 32], f2(v2));
                    tstage[j * 32 + lane] = f2(v2);
                };
                // 4^3 x the Hann-conditioned power, collapsed over kz with a_z
                // (up, centre, down rows of one column; kz index kzi)
                auto tcol = [&](const cf *up, const cf *ce, const cf *dn) -> cf {
                    cf acc = cmk(0.f, 0.f);
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) {
                        const cf c = hann4(up[kzi], ce[kzi], dn[kzi]);
                        const float p = fmaf(c.r, c.r, c.i * c.i);
                        acc = cfma2(c2(t.az2[kzi]), cf{p, p}, acc);
                    }
                    return acc;
                };
                auto flip = [&](cf *dst, const cf *src) {  // conj(C(-kz)): the mirrored row/column
#pragma unroll
                    for (int kzi = 0; kzi < MZ; kzi++) dst[kzi] = cconj(src[MZ - 1 - kzi]);
                };
                if (CW_MEMONLY == 2) {
                    if (threadIdx.x == ISSUER) {
                        tma_store(thg - lane, tstage, G::SM_TSTAGE);
                        tma_store_commit();
                        tma_store_wait_read();
                    }
                } else if (CW_MEMONLY) {
                    const int np = r == 0 ? G::TROW0P : G::TROWNP;
                    for (int j = 0; j < np; j++) {
                        const float2 v = tstage[(G::tpair(r) + j) * 32 + lane];
                        st_state(&thg[(G::tpair(r) + j) * 32], v);
                    }
                }
                if (!CW_MEMONLY) for (int c = r; c <= KX; c += NR) {
                    if (c == 0) {
                        // column kx = 0: rows 0..KY; C(0, 0, -kz) = conj C(0, 0, kz)
                        cf v[KY + 1][MZ];
#pragma unroll
                        for (int kzi = 0; kzi < MZ; kzi++) {
                            const cf w = c2(stage[(kzi >= KZ ? kzi - KZ : KZ - kzi) * 32 + lane]);
                            v[0][kzi] = kzi >= KZ ? w : cconj(w);
                        }
#pragma unroll
                        for (int ky = 1; ky <= KY; ky++)
#pragma unroll
                            for (int kzi = 0; kzi < MZ; kzi++)
                                v[ky][kzi] = c2(stage[(G::spair(ky) + KX * MZ + kzi) * 32 + lane]);
                        cf m[MZ];
                        flip(m, v[1]);  // row -1
                        cf t00 = tcol(m, v[0], v[1]);
                        t00.i = 0.f;  // T(0,0) is real
                        smooth(0, t00);
#pragma unroll
                        for (int ky = 1; ky <= KY; ky++) {
                            if (ky == KY) flip(m, v[KY]);  // row KY + 1 == -KY
                            smooth(G::tpair(ky) + KX, tcol(v[ky - 1], v[ky], ky < KY ? v[ky + 1] : m));
                        }
                    } else {
                        // columns kx = +c (vp) and -c (vm); row 0 stores +c only:
                        // C(0, -c, kz) = conj C(0, c, -kz)
                        const float2 *pp = stage + (KX + c) * MZ * 32 + lane;
                        const float2 *pm = stage + (KX - c) * MZ * 32 + lane;
                        const float2 *p0 = stage + (KZ + 1 + (c - 1) * MZ) * 32 + lane;
                        cf vp[KY + 1][MZ], vm[KY + 1][MZ];
#pragma unroll
                        for (int kzi = 0; kzi < MZ; kzi++) vp[0][kzi] = c2(p0[kzi * 32]);
                        flip(vm[0], vp[0]);
#pragma unroll
                        for (int ky = 1; ky <= KY; ky++)
#pragma unroll
                            for (int kzi = 0; kzi < MZ; kzi++) {
                                vp[ky][kzi] = c2(pp[(G::spair(ky) + kzi) * 32]);
                                vm[ky][kzi] = c2(pm[(G::spair(ky) + kzi) * 32]);
                            }
                        cf m[MZ];
                        flip(m, vm[1]);  // row -1 at +c
                        smooth(c, tcol(m, vp[0], vp[1]));
#pragma unroll
                        for (int ky = 1; ky <= KY; ky++) {
                            if (ky == KY) flip(m, vm[KY]);  // row KY + 1 at +c
                            smooth(G::tpair(ky) + KX + c, tcol(vp[ky - 1], vp[ky], ky < KY ? vp[ky + 1] : m));
                            if (ky == KY) flip(m, vp[KY]);  // row KY + 1 at -c
                            smooth(G::tpair(ky) + KX - c, tcol(vm[ky - 1], vm[ky], ky < KY ? vm[ky + 1] : m));
                        }
                    }
                }
            }
            if (CW_FENCE_ALL) fence_proxy_async();  // Hy reads of the stage before the next TMA write
            CW_STAMP(5);  // C1
            __syncthreads();  // (2) T^ rows visible; the state stage is free
            CW_STAMP(6);  // barrier 2 wait
            if (yy + 1 < ye) issue(yy + 1, xb);
            if (CW_TBULK && !CW_MEMONLY && threadIdx.x == ISSUER) {  // the new T^ packet to HBM
                tma_store(a.that + pix * G::NTP * 32, tstage, G::SM_TSTAGE);
                tma_store_commit();
            }

            // ---------------- phase CD: lag contraction + partial argmax ----------------
            // score(ly, lx) = gy gx R^(ly, lx); stage 1 along kx (B(ky, lx)) for
            // this warp's lag columns, straight into stage 2 along ky and the pick.
            {
                float best = -INFINITY;
                int brk = 0x7fffffff;
                // T^(ky, kx) of the staged rows (row 0: kx >= 0, (0,0) real)
                auto tv = [&](int ky, int kx) -> cf {
                    if (ky == 0) {
                        const cf v = c2(tstage[(kx >= 0 ? kx : -kx) * 32 + lane]);
                        return kx >= 0 ? v : cconj(v);
                    }
                    return c2(tstage[(G::tpair(ky) + kx + KX) * 32 + lane]);
                };
                // stage 2 + in-column argmax for one column whose B values
                // are given: b0 = B(0, lx) (real), bq[ky] = B(ky, lx), ky >= 1
                auto column = [&](int lx, float b0, const cf *bq) {
                    if (NL && t.sym_y) {
                        // visit ly = 0, -1, +1, -2, +2, ...: ascending rank order within
                        // a column (|v|^2 grows with |ly|, then iy ascending); two
                        // interleaved chains (q odd / even) for ILP, each strict '>',
                        // merged by visit index -> the reference's tie winner
                        constexpr int C0 = NL / 2;
                        float ca = -INFINITY, cb = t.s2v[C0].gain * b0;
#pragma unroll
                        for (int k = 1; k <= KY; k++) cb = fmaf(t.s2v[C0].cs[k - 1].x, bq[k].r, cb);
                        int ia = 0x7fff, ib = 0;
#pragma unroll
                        for (int q = 1; q <= C0; q++) {
                            // (e, o) = (g b0 + sum c Re B, sum s Im B); (vm, vp) = e -+ o
                            cf eo = cmk(t.s2v[C0 + q].gain * b0, 0.f);
#pragma unroll
                            for (int k = 1; k <= KY; k++) eo = cfma2(c2(t.s2v[C0 + q].cs[k - 1]), bq[k], eo);
                            const cf v = cfma2(cf{eo.i, eo.i}, cf{-1.f, 1.f}, cf{eo.r, eo.r});
                            const float vm = v.r, vp = v.i;
                            if (q & 1) {
                                if (vm > ca) { ca = vm; ia = 2 * q - 1; }
                                if (vp > ca) { ca = vp; ia = 2 * q; }
                            } else {
                                if (vm > cb) { cb = vm; ib = 2 * q - 1; }
                                if (vp > cb) { cb = vp; ib = 2 * q; }
                            }
                        }
                        if (ca > cb || (ca == cb && ia < ib)) { cb = ca; ib = ia; }
                        const int ci = (ib == 0) ? C0 : ((ib & 1) ? C0 - ((ib + 1) >> 1) : C0 + (ib >> 1));
                        const int rk = srank[ci * nlx + lx];
                        if (better(cb, rk, best, brk)) { best = cb; brk = rk; }
                    } else {
                        for (int ly = 0; ly < nly; ly++) {
                            cf acc = cmk(t.s2v[ly].gain * b0, 0.f);
#pragma unroll
                            for (int k = 1; k <= KY; k++) acc = cfma2(c2(t.s2v[ly].cs[k - 1]), bq[k], acc);
                            const float v = acc.r + acc.i;
                            const int rk = srank[ly * nlx + lx];
                            if (better(v, rk, best, brk)) { best = v; brk = rk; }
                        }
                    }
                };
                if (CW_MEMONLY) {
                    best = 0.f;
                    brk = 0;
                } else if (NL && t.sym_x && t.sym_y) {
                    // Symmetric grids: lag column pairs C0 +- q, q = r + i NR, processed
                    // JQ at a time (stage 1 shares the T^ loads and A/D sums, stage 2
                    // the lag-table constants).  Columns are visited ly = 0, -1, +1,
                    // -2, +2, ... (ascending rank within a column, |v|^2 grows with
                    // |ly|, then iy ascending), so a strict '>' chain per column keeps
                    // the reference's tie winner; for a +-ly pair, max(e - o, e + o)
                    // = e + |o| (the same rounding), -ly on a tie (visited first).
                    constexpr int C0 = NL / 2;
                    constexpr int QPW = (C0 + NR) / NR;  // ceil((C0 + 1) / NR)
                    auto group = [&](auto jq, int q0) {
                        constexpr int JQ = decltype(jq)::value;
                        int qs[JQ];
                        float g[JQ];
                        float2 cs[JQ][KX];
#pragma unroll
                        for (int j = 0; j < JQ; j++) {
                            qs[j] = q0 + j * NR <= C0 ? q0 + j * NR : q0;  // past the grid: repeat q0
                            const LagRec &L = t.s1v[C0 + qs[j]];
                            g[j] = L.gain;
#pragma unroll
                            for (int kx = 0; kx < KX; kx++) cs[j][kx] = L.cs[kx];
                        }
                        // stage 1: B(ky, C0 +- q) for the JQ column pairs; column 2j is
                        // +q, 2j+1 is -q (for q = 0 both are the centre column)
                        float b0[2 * JQ];
                        cf bq[2 * JQ][KY + 1];
                        {   // row 0: T(0,-kx) = conj T(0,kx):
                            // B(0, +-lx) = g T00 + 2 sum c Re T -+ 2 sum s Im T
                            cf acc[JQ];
#pragma unroll
                            for (int j = 0; j < JQ; j++) acc[j] = cmk(0.f, 0.f);
#pragma unroll
                            for (int kx = 1; kx <= KX; kx++) {
                                const cf tv0 = tv(0, kx);
#pragma unroll
                                for (int j = 0; j < JQ; j++) acc[j] = cfma2(c2(cs[j][kx - 1]), tv0, acc[j]);
                            }
                            const float t00 = tv(0, 0).r;
#pragma unroll
                            for (int j = 0; j < JQ; j++) {
                                const float cp = fmaf(2.f, acc[j].r, g[j] * t00);
                                b0[2 * j] = fmaf(2.f, acc[j].i, cp);
                                b0[2 * j + 1] = fmaf(-2.f, acc[j].i, cp);
                            }
                        }
#pragma unroll
                        for (int ky = 1; ky <= KY; ky++) {
                            // P = (cr, ci) = g T0 + sum c A; Q = (sr, -si) = sum s (D.i, D.r)
                            cf P[JQ], Q[JQ];
                            const cf t0 = tv(ky, 0);
#pragma unroll
                            for (int j = 0; j < JQ; j++) {
                                P[j] = cmul2(cf{g[j], g[j]}, t0);
                                Q[j] = cmk(0.f, 0.f);
                            }
#pragma unroll
                            for (int kx = 1; kx <= KX; kx++) {
                                const cf tp = tv(ky, kx), tm = tv(ky, -kx);
                                const cf A = cadd(tp, tm), D = csub(tp, tm);
#pragma unroll
                                for (int j = 0; j < JQ; j++) {
                                    const float c = cs[j][kx - 1].x, sn = cs[j][kx - 1].y;
                                    P[j] = cfma2(cf{c, c}, A, P[j]);
                                    Q[j] = cfma2(cf{sn, sn}, cf{D.i, D.r}, Q[j]);
                                }
                            }
#pragma unroll
                            for (int j = 0; j < JQ; j++) {
                                bq[2 * j][ky] = cfma2(Q[j], cf{1.f, -1.f}, P[j]);      // (cr + sr, ci + si)
                                bq[2 * j + 1][ky] = cfma2(Q[j], cf{-1.f, 1.f}, P[j]);  // (cr - sr, ci - si)
                            }
                        }
                        // stage 2 + in-column argmax, all 2 JQ columns per ly pair
                        float cv[2 * JQ], co[2 * JQ];
                        int cpi[2 * JQ];
#pragma unroll
                        for (int c = 0; c < 2 * JQ; c++) {
                            float e = t.s2v[C0].gain * b0[c];
#pragma unroll
                            for (int k = 1; k <= KY; k++) e = fmaf(t.s2v[C0].cs[k - 1].x, bq[c][k].r, e);
                            cv[c] = e;
                            co[c] = 0.f;
                            cpi[c] = 0;
                        }
                        constexpr int PQU = NL > 17 ? CW_PQ_UNROLL_WIDE : (C0 > 0 ? C0 : 1);
#pragma unroll PQU
                        for (int pq = 1; pq <= C0; pq++) {
                            const LagRec &L2 = t.s2v[C0 + pq];
#pragma unroll
                            for (int c = 0; c < 2 * JQ; c++) {
                                    // (e, o) = (g b0 + sum c Re B, sum s Im B); scores e -+ o
                                cf eo = cmk(L2.gain * b0[c], 0.f);
                                if (CW_ARGMAX_ONLY) {  // diagnostic: the stage-2 FMAs left out (tensor-core bound)
                                    eo.i = L2.cs[0].y * bq[c][1 + (pq % KY)].i;
                                } else {
#pragma unroll
                                    for (int k = 1; k <= KY; k++) eo = cfma2(c2(L2.cs[k - 1]), bq[c][k], eo);
                                }
                                const float m = eo.r + fabsf(eo.i);
                                if (m > cv[c]) {
                                    cv[c] = m;
                                    cpi[c] = pq;
                                    co[c] = eo.i;
                                }
                            }
                        }
#pragma unroll
                        for (int c = 0; c < 2 * JQ; c++) {
                            const int lx = (c & 1) ? C0 - qs[c >> 1] : C0 + qs[c >> 1];
                            const int ci = co[c] > 0.f ? C0 + cpi[c] : C0 - cpi[c];
                            const int rk = srank[ci * nlx + lx];
                            if (better(cv[c], rk, best, brk)) { best = cv[c]; brk = rk; }
                        }
                    };
                    {
                        constexpr bool SMSP17 = CW_SMSP_17 && (NL == 17 || (CW_SMSP_9 && NL == 9));
                        constexpr int JW = NL > 17 ? CW_JQ_WIDE : (SMSP17 ? 1 : 2);
                        constexpr int NG2 = QPW / JW;
                        // (a group's first pair q0 is on the grid; JW = 1: the last
                        // round of q can run past it and is skipped)
                        constexpr SmspSched SS = smsp_sched(C0, NR);
                        if ((NL > 17 || SMSP17) && JW == 1 && CW_ROLL_WIDE && CW_SMSP_SCHED && SS.ok) {
                            // whole pairs dealt by scheduler load (smsp_sched)
                            unsigned int code = SS.code[0];
#pragma unroll
                            for (int w = 1; w < NR; w++)
                                if (r == w) code = SS.code[w];
#pragma unroll 1
                            for (; (code & 31u) != 31u; code >>= 5)
                                group(std::integral_constant<int, 1>{}, (int)(code & 31u));
                        } else if (NL > 17 && CW_ROLL_WIDE) {
#pragma unroll 1
                            for (int i = 0; i < NG2; i++)
                                if (JW == 2 || r + i * NR <= C0)
                                    group(std::integral_constant<int, JW>{}, r + JW * i * NR);
                        } else {
#pragma unroll
                            for (int i = 0; i < NG2; i++)
                                if (JW == 2 || r + i * NR <= C0)
                                    group(std::integral_constant<int, JW>{}, r + JW * i * NR);
                        }
                        if (JW == 2 && (QPW & 1)) {
                            const int q0 = r + (QPW - 1) * NR;
                            if (q0 <= C0) group(std::integral_constant<int, 1>{}, q0);
                        }
                    }
                } else {
                    for (int lx = r; lx < nlx; lx += NR) {
                        const LagRec &L = t.s1v[lx];
                        const float g = L.gain;
                        float b0;
                        cf bq[KY + 1];
                        {
                            float b = g * tv(0, 0).r;
#pragma unroll
                            for (int kx = 1; kx <= KX; kx++) {
                                const cf v = tv(0, kx);
                                b = fmaf(2.f * L.cs[kx - 1].x, v.r, b);
                                b = fmaf(2.f * L.cs[kx - 1].y, v.i, b);
                            }
                            b0 = b;
                        }
#pragma unroll
                        for (int ky = 1; ky <= KY; ky++) {
                            const cf t0 = tv(ky, 0);
                            float xr = g * t0.r, xi = g * t0.i;
#pragma unroll
                            for (int kx = 1; kx <= KX; kx++) {
                                const cf tp = tv(ky, kx), tm = tv(ky, -kx);
                                const cf A = cadd(tp, tm), D = csub(tp, tm);
                                const float c = L.cs[kx - 1].x, sn = L.cs[kx - 1].y;
                                xr = fmaf(c, A.r, fmaf(sn, D.i, xr));
                                xi = fmaf(c, A.i, fmaf(-sn, D.r, xi));
                            }
                            bq[ky] = cmk(xr, xi);
                        }
                        column(lx, b0, bq);
                    }
                }
                pbest[r * 32 + lane] = make_float2(best, __int_as_float(brk));
            }
            // warp KY (fewest lag columns, no PEF): x stage of yy+1 from the
            // row segment it prefetched in C1; barrier 3 orders it before any
            // consumer in the next phase B
            if (r == KY && yy + 1 < ye) {
                cp_async_wait_all();
                __syncwarp();
                xstage_s(ring_slot(yy + 1));
            }
            if (CW_FENCE_ALL) fence_proxy_async();  // T^ stage reads before the next TMA write
            CW_STAMP(7);  // CD
            __syncthreads();  // (3) partial maxima visible; the T^ stage is free
            CW_STAMP(8);  // barrier 3 wait
            if (yy + 1 < ye) issue_t(yy + 1, xb);

            // ---------------- phase E: final pick, PEF partials ----------------
            int vix = 0, viy = 0;
            if (r <= BY) {  // the PEF warps (warp 0 also stores the pair); warp KY goes straight on
                const float2 bv = pbest[lane];
                float best = bv.x;
                int brk = __float_as_int(bv.y);
#pragma unroll
                for (int w = 1; w < NR; w++) {
                    const float2 o = pbest[w * 32 + lane];
                    const int rk = __float_as_int(o.y);
                    if (better(o.x, rk, best, brk)) { best = o.x; brk = rk; }
                }
                if (a.forced_ix >= 0) {
                    vix = a.forced_ix;
                    viy = a.forced_iy;
                } else {
                    vix = srxy[2 * brk];
                    viy = srxy[2 * brk + 1];
                }
            }
            if (!CW_MEMONLY && r <= BY) {
                // PEF on the retained band (_kernels.py:330-342), folded to the
                // stored half space: pred = sum_j coef[v][j] . z+[j], two pairs
                // (one 16-byte coefficient load, one retained quad) per step
                const float4 *cp = reinterpret_cast<const float4 *>(a.coefP + (size_t)(viy * nlx + vix) * G::RETPP) +
                                   G::pquad(r);
                // retained pair q of row r: smem stage, or the state row in
                // L2 (row 0: pair q; rows >= 1: pair q + (KX - BX) MZ; the odd
                // pad pair has a zero coefficient and reads a real pair)
                const float2 *sr = G::PEF_L2
                    ? a.state + ((CW_L2ONLY ? (size_t)blockIdx.x : (size_t)yy * NXB + xb) * G::NSP + G::spair(r) +
                                 (r == 0 ? 0 : (KX - BX) * MZ)) * 32 + lane
                    : sret + 2 * G::pquad(r) * 32 + lane;
                cf acc[2] = {cmk(0.f, 0.f), cmk(0.f, 0.f)};  // packed (c.x z.x, c.y z.y) partial sums
                auto quad = [&](int k) {
                    const float4 c = ldg_coef4(cp + k);
                    const float2 z0 = sr[(2 * k) * 32], z1 = sr[(2 * k + 1) * 32];
                    acc[0] = cfma2(cmk(c.x, c.y), c2(z0), acc[0]);
                    acc[1] = cfma2(cmk(c.z, c.w), c2(z1), acc[1]);
                };
                if (r == 0) {
#pragma unroll
                    for (int k = 0; k < G::PROW0Q; k++) quad(k);
                } else {
#pragma unroll
                    for (int k = 0; k < G::PROWNQ; k++) quad(k);
                }
                const cf sum = cadd(acc[0], acc[1]);
                ppef[r * 32 + lane] = sum.r + sum.i;
            }
            if (r == 0 && colv) {
                uint8_t *vp = a.vidx + ((size_t)yy * W + x) * 2;
                *reinterpret_cast<uchar2 *>(vp) = make_uchar2((uint8_t)vix, (uint8_t)viy);
            }
            CW_STAMP(9);  // E
            // (4) PEF partials visible to warp 0 -- only the PEF warps 0..BY
            // meet here; warp KY runs on into the next row's phase B
            if (r <= BY) asm volatile("bar.sync 1, %0;" ::"n"((BY + 1) * 32) : "memory");
            CW_STAMP(10);  // barrier 4 wait

            // ---------------- phase F: residual (+ threshold epilogue) ----------------
            if (r == 0) {
                cp_async_wait_all();
                float rv = 0.f;
                if (anchor) {
                    float p = 0.f;
#pragma unroll
                    for (int k = 0; k <= BY; k++) p += ppef[k * 32 + lane];
                    const size_t o = (size_t)(yy - a.mhy) * W + (x - a.mhx);
                    rv = delbuf[lane] - p;
                    a.res[o] = rv;
                    if (a.pred) a.pred[o] = p;
                }
                if (a.det) detect_epilogue(a, anchor, x - a.mhx, yy - a.mhy, rv);
            }
        }
        u += ye - ys;
    }
    if (CW_TBULK && threadIdx.x == ISSUER) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (CW_SBULK && !G::PEF_L2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (a.done) {  // every thread's state / T^ / output stores before the flag
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) chain_publish(a.done + blockIdx.x, a.seq);
    }
#ifdef CW_PHASE_TIMING
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0)
        for (int k = 0; k < 11; k++) cw_phase_clk[threadIdx.x >> 5][k] += clk_acc[k];
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x < 1024) cw_cta_span[a.seq & 1][blockIdx.x][5] = cw_gtimer();
#endif
#undef XFR
}

}  // namespace cwb
