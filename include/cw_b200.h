/*
 * cw_b200.h -- C ABI of the B200-native per-pixel whitening pipeline
 * (arXiv 1408.3526; drop-in for the reference `clutterwhiten` hot path).
 *
 * The reference has no native boundary: its hot path is the Python call
 * `Pipeline.process_frame(frame) -> WhitenedOutput | None`
 * (/root/reference/pkg/src/clutterwhiten/pipeline.py:201-294), which drives
 * 13 numba kernels through `BlockExecutor.map_blocks(fn, n)`
 * (parallel.py:62-73, _kernels.py:31-342).  This library replaces that
 * whole operator layer (L0 + L1 in SURVEY.md §1) with one fused sm_100a
 * kernel per frame behind the entry points below; the Python host layer
 * (`paper_1408_3526_b200.pipeline.Pipeline`) binds them with ctypes and
 * keeps the reference's Python signature.  Plain pointers and sizes only:
 * no torch or C++ types cross this boundary, no exceptions, every call
 * returns a status (CW_OK == 0, < 0 on error; text via cw_last_error).
 */
#ifndef CW_B200_H
#define CW_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CW_ABI_VERSION 1

enum cw_status {
    CW_OK = 0,
    CW_ERR_PARAM = -1,     /* maps to ParamError (params.py:30) */
    CW_ERR_VALUE = -2,     /* maps to ValueError */
    CW_ERR_CUDA = -3,      /* CUDA runtime failure (no CPU fallback exists) */
    CW_ERR_NOMEM = -4,     /* device allocation failed */
    CW_ERR_UNSUPPORTED = -5 /* request outside the device path's limits (e.g. > 65535 lags) */
};

/* FilterParams (params.py:34-63); lags as float64 like the reference. */
typedef struct cw_params {
    int32_t kx, ky, kz;      /* half windows: M = 2K + 1 */
    int32_t bx, by;          /* half bandwidths, B < K */
    int32_t mhat[3];         /* group delay (mhat_x, mhat_y, mhat_z) */
    double alpha;            /* smoothing pole in (0, 1) */
    int32_t n_lag_x, n_lag_y;
    const double *lag_x;     /* strictly increasing fractional lags (px) */
    const double *lag_y;
} cw_params;

typedef struct cw_handle cw_handle;

/*
 * Create a stream pipeline for (width x height) frames on CUDA `device`.
 * `bank_c64` is FilterBank.coeffs (design.py:208-253) as interleaved
 * float32 (re, im) pairs, shape (Ly, Lx, retained); `retained` is
 * retained_bin_indices (design.py:195-205).  Replaces Pipeline.__init__
 * (pipeline.py:118-177) minus the host-side bank design.
 * `halo_rows` / `row_offset` describe a spatial strip (multi-GPU): the
 * first `halo_rows` local rows are input-only, and local row 0 is global
 * row `row_offset` (both 0 for a whole frame).
 */
int cw_create(const cw_params *params, int32_t width, int32_t height, int32_t device,
              const float *bank_c64, const int64_t *retained, int32_t n_retained,
              int32_t halo_rows, int32_t row_offset, cw_handle **out);

void cw_destroy(cw_handle *h);

/* Last error message of this handle (or of the failed create when h is NULL). */
const char *cw_last_error(const cw_handle *h);

/* Override every pixel's velocity with grid index (ix, iy); (-1, -1) clears.
 * Replaces the forced_velocity branch of pipeline.py:174-177, 260-265. */
int cw_set_forced_velocity(cw_handle *h, int32_t ix, int32_t iy);

/*
 * Push one frame: the whole SpectrumStream.push + conditioning + flow +
 * PEF chain of Pipeline.process_frame (pipeline.py:201-294).
 *  frame        : (H, W) float32, HOST memory (pinned gives async copies)
 *  residual     : (H, W) float32 host out, or NULL
 *  prediction   : (H, W) float32 host out, or NULL
 *  vidx         : (H, W, 2) uint8 host out [ix, iy] per anchor, or NULL
 *  ready        : 1 when an output frame was produced (frames_seen >= Mz)
 *  frame_index  : input index of the output frame (n - mhat_z)
 *  stream       : cudaStream_t to run on (NULL: the handle's own stream)
 * Synchronises `stream` before returning when any host output is given or
 * when `frame` is page-locked (pageable frames are staged before the call
 * returns), so the caller may reuse every buffer afterwards.
 * When every given output buffer is page-locked host memory (cudaHostAlloc,
 * torch pin_memory), the kernel writes the outputs into it directly while it
 * runs (no device-to-host copies after the kernel); the residual/prediction
 * border outside the valid region is zeroed on the host.
 */
int cw_push(cw_handle *h, const float *frame, float *residual, float *prediction, uint8_t *vidx,
            int32_t *ready, int64_t *frame_index, void *stream);

/* Same, with the frame already in device memory and outputs left on the
 * device (see cw_device_outputs); never synchronises. */
int cw_push_device(cw_handle *h, const float *frame_dev, int32_t *ready, int64_t *frame_index,
                   void *stream);

/* Device pointers of the latest outputs: residual (H,W) f32, prediction
 * (H,W) f32, vidx (H,W,2) u8.  Valid until the next push. */
int cw_device_outputs(cw_handle *h, float **residual, float **prediction, uint8_t **vidx);

/*
 * Pipelined streaming: enqueue frame n's upload, kernel
 * and result download on three streams and return at once; consecutive
 * frames overlap (H2D of n+1 and D2H of n-1 run under kernel n).  Host
 * buffers (pinned for true overlap) must stay valid until cw_wait(ticket)
 * returns; at most 8 tickets may be outstanding.
 */
int cw_submit(cw_handle *h, const float *frame, float *residual, float *prediction, uint8_t *vidx,
              int64_t *ticket);
int cw_wait(cw_handle *h, int64_t ticket, int32_t *ready, int64_t *frame_index);

/*
 * cw_submit for a frame already in device memory (a strip assembled from
 * NCCL halo receives, strips.py): the pipeline's stream waits for work
 * already enqueued on `producer` (a cudaStream_t; NULL = legacy default),
 * copies the frame into its ring slot, and `producer` is then ordered after
 * that copy, so the caller may refill `frame_dev` with work enqueued later
 * on `producer`.  Results download into the host buffers as cw_submit's;
 * collect them with cw_wait(ticket).
 */
int cw_submit_device(cw_handle *h, const float *frame_dev, float *residual, float *prediction, uint8_t *vidx,
                     int64_t *ticket, void *producer);

/*
 * cw_submit for a frame that is already complete in device memory and stays
 * unchanged until cw_wait(ticket) returns (resident inputs, e.g. a frame
 * buffer filled before the stream starts).  No producer stream is joined
 * and nothing is enqueued between frame kernels: the frame kernel reads
 * `frame_dev` directly, its ring slot (the delayed frame of a later kernel)
 * is filled by a copy-engine copy on the upload stream that the later
 * kernel waits for by a flag, and consecutive frame kernels are chained
 * (programmatic dependent launch; each CTA waits only for its own units of
 * the previous frame), so a frame's kernel starts in
 * the SM slots the previous frame's early CTAs free.  Host output buffers may be NULL (the
 * results stay on the device: cw_device_outputs after cw_wait).  Results are
 * bit-identical to cw_push_device's with the static work split.
 * (Not in the reference: its frames are host arrays, pipeline.py:201.)
 */
int cw_submit_resident(cw_handle *h, const float *frame_dev, float *residual, float *prediction, uint8_t *vidx,
                       int64_t *ticket);

/* Orders `stream` (a cudaStream_t) after every frame kernel submitted so far
 * (device-side join, e.g. to consume cw_device_outputs on the caller's
 * stream or to time a run of cw_submit_resident calls with events). */
int cw_join(cw_handle *h, void *stream);

/*
 * cw_submit for a frame in a sequence-file sample format (replaces the host
 * decode of read_sequence, seqio.py:172-204; the payloads of seqio.py:1-8):
 *   CW_FMT_F32LE: little-endian float32 (frames.f32), scale/offset ignored;
 *   CW_FMT_PGM16: P5 payload, big-endian uint16 q; the frame is
 *                 f32(f64(q) * scale + offset), byte-swapped and de-quantised
 *                 on the device (half the upload bytes of float32).
 * `samples` = H*W samples (the PGM payload after its header).
 */
#define CW_FMT_F32LE 0
#define CW_FMT_PGM16 1
int cw_submit_raw(cw_handle *h, const void *samples, int32_t format, double scale, double offset,
                  float *residual, float *prediction, uint8_t *vidx, int64_t *ticket);

/*
 * Fused detection epilogue ("final threshold"; the truth-free
 * metrics of cli.compute_metrics_row, cli.py:157-208).  cw_set_detection(h,
 * tau, cap): every valid output pixel with |residual| >= tau (tau <= 0: no
 * list) is appended (x, y, residual) to a per-frame list of capacity `cap`
 * (cap < 0 turns the epilogue off).  cw_detections(h, ticket, ...) for a
 * completed frame (ticket = cw_submit ticket, or the frame number n of a
 * synchronising push): *n_total = detections found (may exceed cap),
 * xyr = up to out_cap (x, y, residual) triples in arbitrary order, stats =
 * {peak |res|, peak x, peak y (first in row-major order on ties),
 *  sum res^2, n valid outputs}.
 */
int cw_set_detection(cw_handle *h, float tau, int32_t cap);
int cw_detections(cw_handle *h, int64_t ticket, int32_t *n_total, float *xyr, int32_t out_cap, double *stats);

/*
 * Checkpoint / resume: the complete stream state (observer state, smoothing
 * state T^, raw-frame ring, frame counter) as one host blob of
 * cw_snapshot_size() bytes.  cw_restore() into a pipeline of the same
 * geometry continues the stream exactly where the snapshot was taken (no
 * new warm-up; the reference can only restart, pipeline.py:245-247).
 */
int cw_snapshot_size(const cw_handle *h, size_t *bytes);
int cw_snapshot(cw_handle *h, void *dst, size_t bytes);
int cw_restore(cw_handle *h, const void *src, size_t bytes);

/* Synchronous device -> host copy (e.g. of cw_device_outputs buffers). */
int cw_copy_to_host(cw_handle *h, void *dst, const void *src_dev, size_t bytes);

/* Device pointer of the frame-ring slot the next push will use (for
 * producers that write frames in place, e.g. NCCL halo receives). */
int cw_next_frame_slot(cw_handle *h, float **slot);

/* Push the frame already written into cw_next_frame_slot(). */
int cw_push_inplace(cw_handle *h, int32_t *ready, int64_t *frame_index, void *stream);

int64_t cw_frames_seen(const cw_handle *h);

/* Bytes per velocity-index component: 1 (vidx is (H, W, 2) uint8), or 2
 * when a lag grid has more than 256 entries (vidx is (H, W, 2) uint16). */
int32_t cw_index_bytes(const cw_handle *h);

/* 1 when the handle runs the runtime-geometry kernels (parameters with no
 * compiled fused instance: any window / bandwidth / lag grid that
 * params.py:114-158 accepts), 0 for the fused kernel. */
int32_t cw_is_generic(const cw_handle *h);

/* Which kernel runs this handle: 0 = a fused instance compiled into the
 * library, 1 = a fused instance compiled at run time for this geometry
 * (NVRTC, cached as a cubin), 2 = the runtime-geometry kernels. */
int32_t cw_kernel_kind(const cw_handle *h);

/* Compile (NVRTC) the fused instance these parameters need into the cubin
 * cache directory `dir` unless it is there already (build-time prebuild;
 * the library looks in <package>/jit_cache).  CW_ERR_UNSUPPORTED when the
 * geometry is beyond the fused kernel or NVRTC is unavailable. */
int cw_jit_prebuild(const cw_params *params, const char *dir);

/* Spectrum backend (pipeline.py:139-142): 0 = recursive (sliding DFT +
 * deadbeat observer, default), 1 = naive: every pixel's spectrum evaluated
 * directly from its raw Mx x My x Mz window (spectrum.py:257-327), then the
 * same conditioning, flow and PEF.  Switch before the first push. */
int cw_set_backend(cw_handle *h, int32_t naive);

/*
 * Parity views (tests only), copied to host after synchronising:
 *  what = 0: spectrum S of the last frame, (H, W, Mz, My, Mx) complex128
 *            (reference SpectrumField.bins layout, spectrum.py:107-135),
 *            rebuilt from the stored observer state
 *  what = 1: smoothed kz-collapsed state T^ (H, W, My, Mx) complex128
 *            (R^ = autocorr of T^, flow.py:87-114)
 *  what = 2: raw observer state, float32, kernel layout
 * `bytes` must equal the view size; returns CW_ERR_VALUE otherwise.
 */
int cw_read_view(cw_handle *h, int32_t what, void *dst, size_t bytes);

/* Kernel-only timing support: number of CUDA kernels one push launches
 * and the grid/block shape of the frame kernel (bench.py bookkeeping). */
int cw_launch_info(const cw_handle *h, int32_t *kernels_per_push, int32_t *grid, int32_t *block,
                   int32_t *smem_bytes);

/* Per-launch device timing of the frame kernel: when on, every push
 * records a CUDA event pair around the kernel on the launch stream;
 * cw_kernel_time returns the summed kernel milliseconds and the number
 * of launches since the last call (and resets the record). */
int cw_set_timing(cw_handle *h, int32_t on);
int cw_kernel_time(cw_handle *h, double *total_ms, int64_t *launches);

/*
 * Counter-based synthetic scene (the model of the
 * reference generator, scenegen.py:152-209, with noise that is a pure
 * function of (seed, t, y, x) instead of one row-major numpy stream,
 * scenegen.py:132-139).  cw_scene_generate writes frames t0 .. t0+n-1,
 * rows [r0, r1), columns [c0, c1) of the (width x height) scene into
 * out_dev (n, r1-r0, c1-c0) float32 on the current device, on `stream`.
 * Any window equals the same pixels of the full frame bit for bit, and
 * scenegen.generate_counter computes the same bits on the host.
 */
typedef struct cw_scene {
    int32_t width, height;
    int64_t frame_count;        /* the target reaches the centre at frame_count - 1 */
    int32_t n_comp;             /* <= 64 drifting cosines */
    const double *comps;        /* host (n_comp, 4): fx, fy, phase, amplitude */
    double dc_offset, clutter_vx, clutter_vy;
    int32_t nonuniform;         /* config C2: v += (ax sin(2 pi y/H), ay cos(2 pi x/W)) */
    double motion_ax, motion_ay;
    int32_t target;             /* 0: no point target */
    double target_vx, target_vy, target_peak, psf_sigma, target_truncation;
    double noise_sigma;
    uint64_t seed;
} cw_scene;

int cw_scene_generate(const cw_scene *scene, int64_t t0, int32_t n_frames, int32_t r0, int32_t r1, int32_t c0,
                      int32_t c1, float *out_dev, void *stream);
const char *cw_scene_last_error(void);

/* Library/ABI identification. */
int32_t cw_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* CW_B200_H */
