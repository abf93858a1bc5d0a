// cw_scene.cu -- counter-based synthetic scene generator.
//
// The reference's scene model (/root/reference/pkg/src/clutterwhiten/
// scenegen.py:152-209): a DC pedestal plus drifting cosines, an occluding
// Gaussian point target (inject_target, 102-129) and white Gaussian noise.
// The reference draws the noise from one numpy stream, row-major per frame
// (add_noise, 132-139), so a pixel's value depends on every pixel before it;
// a strip of a 4096^2 frame cannot be produced without the whole frame.
// Here every pixel is a pure function of (seed, t, y, x):
//
//   v = dc + sum_i amp_i cos(2 pi (fx_i (x - vx t) + fy_i (y - vy t) + ph_i / 2 pi))
//   v = blob  where the target blob peak exp(-r^2 / 2 sigma^2) >= truncation
//   v += sigma_n * sqrt(-2 ln u1) cos(2 pi u2),  (u1, u2) from
//        Philox4x32-10(counter = (x, y, t_lo, t_hi), key = seed)
//
// optionally with the config-C2 motion field v(x, y) = (vx + ax sin(2 pi y /
// H), vy + ay cos(2 pi x / W)).  Any row strip or crop equals
// the same pixels of the full frame bit for bit, for any split.
//
// The transcendental functions are evaluated here with IEEE-754 double
// +, -, *, / only (range reduction + fixed-degree polynomials, no FMA: this
// translation unit is compiled with -fmad=false), and sqrt / rint / frexp /
// ldexp, all exactly rounded.  scenegen.generate_counter restates the same
// operation sequence in numpy, so host crops equal device crops bit for bit.
#include "../../include/cw_b200.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

namespace {

constexpr int MAXCOMP = 64;

struct SceneArgs {
    int W, H;       // full frame
    int r0, c0;     // first row / column of the generated window
    int rows, cols; // window size
    long long t0;   // first frame
    int nt;
    int ncomp;
    double fx[MAXCOMP], fy[MAXCOMP], ph[MAXCOMP], amp[MAXCOMP];  // ph in turns (phase / 2 pi)
    double dc, vx, vy;
    int nonuniform;
    double ax, ay;
    int target;
    double tcx0, tcy0, tvx, tvy;  // centre(t) = (tcx0 + tvx (t - last), ...), t - last = t + tlast_neg
    long long last;
    double peak, two_s2, trunc, reach;
    double noise;
    unsigned int key0, key1;
};

#define HD __host__ __device__ __forceinline__

// cos(2 pi u): reduce to s in [-1/8, 1/8] turns, quadrant q, Taylor series
// of cos / sin on [-pi/4, pi/4] (degree 20 / 19: truncation < 2e-18).
HD double cos_turns(double u)
{
    const double r = u - rint(u);
    const double q = rint(4.0 * r);
    const double s = r - 0.25 * q;
    const double th = s * 6.283185307179586;
    const double t2 = th * th;
    double c = 1.0 / 2432902008176640000.0;  // 1/20!
    c = c * t2 - 1.0 / 6402373705728000.0;   // 1/18!
    c = c * t2 + 1.0 / 20922789888000.0;     // 1/16!
    c = c * t2 - 1.0 / 87178291200.0;        // 1/14!
    c = c * t2 + 1.0 / 479001600.0;          // 1/12!
    c = c * t2 - 1.0 / 3628800.0;            // 1/10!
    c = c * t2 + 1.0 / 40320.0;              // 1/8!
    c = c * t2 - 1.0 / 720.0;                // 1/6!
    c = c * t2 + 1.0 / 24.0;
    c = c * t2 - 0.5;
    c = c * t2 + 1.0;
    double sn = -1.0 / 121645100408832000.0;  // -1/19!
    sn = sn * t2 + 1.0 / 355687428096000.0;   // 1/17!
    sn = sn * t2 - 1.0 / 1307674368000.0;     // 1/15!
    sn = sn * t2 + 1.0 / 6227020800.0;        // 1/13!
    sn = sn * t2 - 1.0 / 39916800.0;          // 1/11!
    sn = sn * t2 + 1.0 / 362880.0;            // 1/9!
    sn = sn * t2 - 1.0 / 5040.0;              // 1/7!
    sn = sn * t2 + 1.0 / 120.0;
    sn = sn * t2 - 1.0 / 6.0;
    sn = sn * t2 + 1.0;
    sn = sn * th;
    // cos(theta + q pi / 2), q in {-2, -1, 0, 1, 2}
    if (q == 0.0) return c;
    if (q == 1.0) return -sn;
    if (q == -1.0) return sn;
    return -c;
}

// exp(x) for x <= 0 (0 below -700): x = k ln2 + r, |r| <= ln2 / 2, Taylor
// degree 17, scaled by 2^k.
HD double exp_nonpos(double x)
{
    if (x < -700.0) return 0.0;
    const double k = rint(x * 1.4426950408889634);
    const double r = (x - k * 6.93147180369123816490e-01) - k * 1.90821492927058770002e-10;
    double p = 1.0 / 355687428096000.0;  // 1/17!
    p = p * r + 1.0 / 20922789888000.0;
    p = p * r + 1.0 / 1307674368000.0;
    p = p * r + 1.0 / 87178291200.0;
    p = p * r + 1.0 / 6227020800.0;
    p = p * r + 1.0 / 479001600.0;
    p = p * r + 1.0 / 39916800.0;
    p = p * r + 1.0 / 3628800.0;
    p = p * r + 1.0 / 362880.0;
    p = p * r + 1.0 / 40320.0;
    p = p * r + 1.0 / 5040.0;
    p = p * r + 1.0 / 720.0;
    p = p * r + 1.0 / 120.0;
    p = p * r + 1.0 / 24.0;
    p = p * r + 1.0 / 6.0;
    p = p * r + 0.5;
    p = p * r + 1.0;
    p = p * r + 1.0;
    return ldexp(p, (int)k);
}

// ln(u) for u in (0, 1]: u = m 2^e, m in [sqrt(1/2), sqrt(2)), atanh series
// in s = (m - 1) / (m + 1), |s| <= 0.1716 (12 terms: truncation < 1e-19).
HD double log_unit(double u)
{
    int e;
    double m = frexp(u, &e);
    if (m < 0.70710678118654752440) {
        m = m * 2.0;
        e = e - 1;
    }
    const double s = (m - 1.0) / (m + 1.0);
    const double s2 = s * s;
    double p = 1.0 / 23.0;
    p = p * s2 + 1.0 / 21.0;
    p = p * s2 + 1.0 / 19.0;
    p = p * s2 + 1.0 / 17.0;
    p = p * s2 + 1.0 / 15.0;
    p = p * s2 + 1.0 / 13.0;
    p = p * s2 + 1.0 / 11.0;
    p = p * s2 + 1.0 / 9.0;
    p = p * s2 + 1.0 / 7.0;
    p = p * s2 + 1.0 / 5.0;
    p = p * s2 + 1.0 / 3.0;
    p = p * s2 + 1.0;
    const double de = (double)e;
    return de * 6.93147180369123816490e-01 + (2.0 * s * p + de * 1.90821492927058770002e-10);
}

HD void philox4x32_10(unsigned int c[4], unsigned int k0, unsigned int k1)
{
    for (int i = 0; i < 10; i++) {
        const unsigned long long p0 = 0xD2511F53ull * c[0], p1 = 0xCD9E8D57ull * c[2];
        const unsigned int hi0 = (unsigned int)(p0 >> 32), lo0 = (unsigned int)p0;
        const unsigned int hi1 = (unsigned int)(p1 >> 32), lo1 = (unsigned int)p1;
        const unsigned int n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0;
        c[1] = lo1;
        c[2] = n2;
        c[3] = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}

// one pixel of the scene (the whole model; the numpy twin follows this line
// by line: paper_1408_3526_b200/scenegen.py:generate_counter)
__device__ __forceinline__ float scene_pixel(const SceneArgs &a, long long t, int y, int x)
{
    const double xd = (double)x, yd = (double)y, td = (double)t;
    double vx = a.vx, vy = a.vy;
    if (a.nonuniform) {
        vx = vx + a.ax * cos_turns(yd / (double)a.H - 0.25);
        vy = vy + a.ay * cos_turns(xd / (double)a.W);
    }
    const double px = xd - vx * td, py = yd - vy * td;
    double acc = a.dc;
    for (int i = 0; i < a.ncomp; i++)
        acc = acc + a.amp[i] * cos_turns(a.fx[i] * px + a.fy[i] * py + a.ph[i]);
    if (a.target) {
        const double tl = (double)(t - a.last);
        const double cx = a.tcx0 + a.tvx * tl, cy = a.tcy0 + a.tvy * tl;
        const double dx = xd - cx, dy = yd - cy;
        if (fabs(dx) <= a.reach && fabs(dy) <= a.reach) {
            const double blob = a.peak * exp_nonpos(-(dx * dx + dy * dy) / a.two_s2);
            if (blob >= a.trunc) acc = blob;
        }
    }
    if (a.noise > 0.0) {
        unsigned int c[4] = {(unsigned int)x, (unsigned int)y, (unsigned int)(unsigned long long)t,
                             (unsigned int)((unsigned long long)t >> 32)};
        philox4x32_10(c, a.key0, a.key1);
        const double u1 = ((double)(c[0] >> 5) * 67108864.0 + (double)(c[1] >> 6) + 1.0) * 1.1102230246251565e-16;
        const double u2 = ((double)(c[2] >> 5) * 67108864.0 + (double)(c[3] >> 6)) * 1.1102230246251565e-16;
        const double z = sqrt(-2.0 * log_unit(u1)) * cos_turns(u2);
        acc = acc + a.noise * z;
    }
    return (float)acc;
}

__global__ void __launch_bounds__(256) cw_scene_kernel(const __grid_constant__ SceneArgs a, float *__restrict__ out)
{
    const long long per = (long long)a.rows * a.cols;
    const long long n = per * a.nt;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const long long f = i / per, rem = i - f * per;
        const int r = (int)(rem / a.cols), c = (int)(rem - (long long)r * a.cols);
        out[i] = scene_pixel(a, a.t0 + f, a.r0 + r, a.c0 + c);
    }
}

thread_local std::string g_scene_err;

}  // namespace

extern "C" {

const char *cw_scene_last_error(void) { return g_scene_err.c_str(); }

int cw_scene_generate(const cw_scene *s, int64_t t0, int32_t n_frames, int32_t r0, int32_t r1, int32_t c0, int32_t c1,
                      float *out_dev, void *stream)
{
    if (!s || !out_dev || n_frames < 0 || r0 < 0 || r1 > s->height || r0 > r1 || c0 < 0 || c1 > s->width || c0 > c1 ||
        s->n_comp < 0 || s->n_comp > MAXCOMP || (s->n_comp && !s->comps) || t0 < 0) {
        g_scene_err = "bad scene window or component count (<= 64)";
        return CW_ERR_VALUE;
    }
    SceneArgs a;
    std::memset(&a, 0, sizeof a);
    a.W = s->width;
    a.H = s->height;
    a.r0 = r0;
    a.c0 = c0;
    a.rows = r1 - r0;
    a.cols = c1 - c0;
    a.t0 = t0;
    a.nt = n_frames;
    a.ncomp = s->n_comp;
    for (int i = 0; i < s->n_comp; i++) {
        a.fx[i] = s->comps[4 * i];
        a.fy[i] = s->comps[4 * i + 1];
        a.ph[i] = s->comps[4 * i + 2] / 6.283185307179586;
        a.amp[i] = s->comps[4 * i + 3];
    }
    a.dc = s->dc_offset;
    a.vx = s->clutter_vx;
    a.vy = s->clutter_vy;
    a.nonuniform = s->nonuniform;
    a.ax = s->motion_ax;
    a.ay = s->motion_ay;
    a.target = s->target;
    a.tcx0 = s->width / 2.0;
    a.tcy0 = s->height / 2.0;
    a.tvx = s->target_vx;
    a.tvy = s->target_vy;
    a.last = s->frame_count - 1;
    a.peak = s->target_peak;
    a.two_s2 = 2.0 * s->psf_sigma * s->psf_sigma;
    a.trunc = s->target_truncation;
    a.reach = s->target ? s->psf_sigma * std::sqrt(2.0 * std::log(s->target_peak / s->target_truncation)) + 1.0 : 0.0;
    a.noise = s->noise_sigma;
    a.key0 = (unsigned int)s->seed;
    a.key1 = (unsigned int)(s->seed >> 32);
    const long long n = (long long)a.rows * a.cols * a.nt;
    if (n == 0)
        return CW_OK;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long want = (n + 255) / 256;
    const int grid = (int)std::min<long long>(want, (long long)sms * 8);
    cw_scene_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a, out_dev);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_scene_err = std::string("cw_scene_kernel: ") + cudaGetErrorString(e);
        return CW_ERR_CUDA;
    }
    return CW_OK;
}

}  // extern "C"
