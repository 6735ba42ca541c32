/*
 * fractal.h -- C ABI of libfractal, the B200 (sm_100a) escape-time engine for
 * arXiv 1611.03079 "Fractal Art Generation using GPUs".
 *
 * Citations: P:n = PAPER.md line n (the paper), S:n = SPEC.md line n; "reading c-k"
 * = the interpretation recorded in DESIGN.md §Readings.
 *
 * The problem as the paper states it: every pixel of a region is "scaled to
 * the complex plane" (the region-covering routine) and iterated under
 * Z_{n+1} = Z_n^2 + C until it diverges or an iteration limit is reached ("in our
 * implementation, that limit is 100"); pixels are then "assigned color levels
 * according to the number of iterations".  Julia frames fix C and take Z_0 from the
 * pixel; Mandelbrot parameter maps take C from the pixel with Z_0 = 0;
 * paths re-render the Julia frame as C moves.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  Count.   count = smallest n in [0, max_iter-1] with |Z_n|^2 > 4 (strict), else
 *           max_iter (readings c-1, c-2).  Stored as uint16.
 *  Map.     pixel (px, py) -> (re, im) with row 0 at the top (reading c-3):
 *             re = center_re + (2 px + 1 - W) * (half_w / W)
 *             im = center_im + (H - 1 - 2 py) * (half_h / H)
 *           evaluated in binary64, each operation separately rounded, then rounded
 *           once to binary32 in the FP32 modes (reading c-8).
 *  Modes.   *_STRICT: the exact IEEE operation sequence of reading c-9, no
 *           contraction -> bit-identical counts to the CPU oracle.  *_FAST: FMA-
 *           contracted and rescaled; counts may differ from
 *           strict only at pixels within ~1 pixel of the set boundary (reading c-10).
 *  Layout.  counts: uint16, row-major [rows][width]; paths: frame-major
 *           [n_frames][rows][width] with 64-bit offsets.  rgba: 4 bytes per pixel
 *           (R, G, B, A), same order.  Little-endian.
 *  Memory.  Every pointer named *_dev / out_* is DEVICE memory owned by the caller;
 *           the library keeps no pointer after return.  c_host and the palette are
 *           HOST memory, consumed (copied into kernel parameters) before return.
 *           The library owns, per (device, stream), small scheduling workspaces
 *           (chunk counters, a 384-B queue header), the survivor buffer of the
 *           heavy-tailed two-phase path (one 16-B item per pixel, 24 B in fp64,
 *           grown on demand, frames up to 2^25 pixels) and, per device, a 1-KB
 *           device copy of each distinct palette.  They are created
 *           on first use (zeroed / uploaded in stream order on `stream`, which the
 *           call then synchronises once) and live until process exit; a buffer that
 *           has to grow is replaced, and the outgrown one is kept alive too, so a CUDA
 *           graph captured earlier never sees its memory freed.  Creation is not
 *           allowed inside CUDA graph capture (cudaErrorStreamCaptureUnsupported
 *           -> FR_ERR_CUDA), so make the first call of a kind on a stream outside
 *           capture.
 *  Graphs.  A captured graph uses the workspaces of the stream it was captured on.
 *           Replays of such graphs must be stream-ordered with each other and with
 *           eager calls on that stream (replay on the capture stream, or order the
 *           replay stream after it with events): the self-resetting counters of two
 *           overlapping launches sharing one workspace would race.
 *  Async.   Calls validate synchronously, enqueue on `stream` and return.  Outputs
 *           are valid once the caller synchronises the stream; device faults surface
 *           there.  On FR_ERR_INVALID_ARG / FR_ERR_TOO_LARGE / FR_ERR_UNSUPPORTED
 *           nothing has been launched.  On FR_ERR_CUDA (a failed launch or
 *           allocation) earlier kernels of the same call -- earlier chunks of a path,
 *           the first phase of a two-phase frame -- may already be enqueued: the
 *           output buffers are then undefined.  No C++ exception crosses the ABI.
 *           Calls are reentrant and thread-safe (the caches above are mutex-guarded;
 *           calls on one stream share its workspaces in stream order); apart from
 *           those caches the library holds only a monotonic launch counter
 *           (fr_launch_count).
 *  Overlap. Single-frame kernels use programmatic dependent launch: when the
 *           previous operation on `stream` is one of this library's single-frame
 *           kernels, the next one may start computing before it has finished, but
 *           touches no global memory until it has completed, so stream order holds
 *           for every memory effect (FRACTAL_PDL=0 in the environment disables it).
 *  Stream.  `stream` is a cudaStream_t (NULL = legacy default stream).
 */
#ifndef FRACTAL_H_
#define FRACTAL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fr_stream; /* == cudaStream_t */

/* A complex value ("values in the complex plane"). */
typedef struct {
    double re, im;
} fr_complex;

/* Region covered: centre and half extents in plane units. */
typedef struct {
    double center_re, center_im, half_w, half_h;
} fr_window;

typedef enum {
    FR_FP32_FAST = 0,
    FR_FP32_STRICT = 1,
    FR_FP64_FAST = 2, /* deep zoom: pixel pitch below binary32 resolution */
    FR_FP64_STRICT = 3
} fr_mode;

/* Colour levels (rule S:245, reading c-12): count == max_iter -> interior,
 * else rgba[4 * (count mod n) .. +3].  rgba is HOST memory, n in [2, 256]. */
typedef struct {
    const uint8_t* rgba;
    int32_t n;
    uint8_t interior[4];
} fr_palette;

/* Cyclic row bands: the frame's rows are cut into bands of
 * band_rows rows (the last may be short); global band b belongs to rank
 * b % n_ranks.  A rank's output holds its bands compacted in increasing global-row
 * order; band pixels use GLOBAL row indices, so they are bit-identical to the same
 * rows of the full render.  {0, 1, 0} = the whole frame. */
typedef struct {
    int32_t band_rows, n_ranks, rank;
} fr_bands;

typedef enum {
    FR_OK = 0,
    FR_ERR_INVALID_ARG = 1, /* bad size, non-finite value, null pointer, bad bands/palette */
    FR_ERR_TOO_LARGE = 2,   /* width*height > 2^31 pixels per frame */
    FR_ERR_UNSUPPORTED = 3, /* max_iter > 65535 (uint16 counts), unknown mode */
    FR_ERR_CUDA = 4         /* a CUDA launch/copy failed; see fr_last_cuda_error() */
} fr_status;

/* Julia frame of Z^2 + C, full frame, FR_FP32_FAST.
 *   c          the constant C (finite)
 *   win        region covered (finite, half_w > 0, half_h > 0)
 *   width, height >= 1, width*height <= 2^31;  1 <= max_iter <= 65535
 *   out_counts device uint16 [height][width] */
fr_status julia_render(fr_complex c, fr_window win, int32_t width, int32_t height,
                       int32_t max_iter, uint16_t* out_counts, fr_stream stream);

/* Julia frame with explicit mode, cyclic bands and optional fused colour levels.
 *   out_counts device uint16 [fr_band_local_rows(height, bands)][width]; a rank that holds
 *              no band (0 local rows) is a no-op returning FR_OK, null pointers allowed
 *   pal        NULL, or a palette (then out_rgba is required: device uint8 [rows][width][4]) */
fr_status julia_render_ex(fr_complex c, fr_window win, int32_t width, int32_t height,
                          int32_t max_iter, fr_mode mode, fr_bands bands, uint16_t* out_counts,
                          const fr_palette* pal, uint8_t* out_rgba, fr_stream stream);

/* Julia frames along a path of C values: frame k is exactly
 * julia_render_ex(c_host[k], ...) of the full frame.  n_frames == 0 is a no-op.
 *   c_host     HOST array of n_frames values, all finite (consumed before return)
 *   out_counts device uint16 [n_frames][height][width]
 *   out_rgba   device uint8 [n_frames][height][width][4] iff pal != NULL */
fr_status julia_render_path(const fr_complex* c_host, int32_t n_frames, fr_window win,
                            int32_t width, int32_t height, int32_t max_iter, fr_mode mode,
                            uint16_t* out_counts, const fr_palette* pal, uint8_t* out_rgba,
                            fr_stream stream);

/* As julia_render_path with uint8 counts (halves the bytes delivered to
 * rank 0 or to the host).  Requires max_iter <= 255 (else FR_ERR_UNSUPPORTED).
 *   out_counts8 device uint8 [n_frames][height][width] */
fr_status julia_render_path8(const fr_complex* c_host, int32_t n_frames, fr_window win,
                             int32_t width, int32_t height, int32_t max_iter, fr_mode mode,
                             uint8_t* out_counts8, const fr_palette* pal, uint8_t* out_rgba,
                             fr_stream stream);

/* As julia_render_path, with the counts delivered to HOST memory: frames are rendered
 * in chunks on `stream` into two device staging buffers and each chunk is copied
 * device->host on an internal stream while the next chunk renders.  SYNCHRONOUS: returns
 * once every count is in out_host (pinned host memory -- cudaMallocHost /
 * cudaHostRegister -- gives overlapped copies; pageable memory works, slower).
 *   bytes_per_count  2 (uint16) or 1 (uint8; requires max_iter <= 255)
 *   out_host         HOST [n_frames][height][width] of bytes_per_count each
 * Errors as julia_render_path; a bad bytes_per_count -> FR_ERR_INVALID_ARG. */
fr_status julia_render_path_host(const fr_complex* c_host, int32_t n_frames, fr_window win,
                                 int32_t width, int32_t height, int32_t max_iter, fr_mode mode,
                                 int32_t bytes_per_count, void* out_host, fr_stream stream);

/* Mandelbrot parameter map (C from the pixel, Z_0 = 0; deep zoom P:55). */
fr_status mandelbrot_param_map(fr_window win, int32_t width, int32_t height, int32_t max_iter,
                               fr_mode mode, fr_bands bands, uint16_t* out_counts,
                               const fr_palette* pal, uint8_t* out_rgba, fr_stream stream);

/* Other iteration maps (NEXT-3): the paper notes "many other functions yield fruitful
 * explorations" and shows one in Figure 4, printed garbled as
 * z^4 + (z^2+1)/(z^2+1) + c; it is read per SPEC S:35 (reading c-14). */
typedef enum {
    FR_FN_Z2 = 0,         /* z^2 + c (the main map) */
    FR_FN_Z4 = 1,         /* z^4 + c */
    FR_FN_Z4_RATIONAL = 2 /* z^4 + (z^2+1)/(z^2-1) + c; at the pole z^2 = 1, Z -> +inf */
} fr_function;

/* Julia frame of map `fn` (same count definition, bailout |Z|^2 > 4, map and layout as
 * julia_render_ex; full frame).  Both modes of a precision run the strict IEEE operation
 * sequence of reading c-14 (the FAST rescaling applies to z^2 + c only).
 * Errors as julia_render_ex; unknown fn -> FR_ERR_UNSUPPORTED. */
fr_status julia_render_fn(fr_function fn, fr_complex c, fr_window win, int32_t width,
                          int32_t height, int32_t max_iter, fr_mode mode, uint16_t* out_counts,
                          const fr_palette* pal, uint8_t* out_rgba, fr_stream stream);

/* Standalone colour levels over n_pixels counts.
 *   counts device uint16 [n_pixels], out_rgba device uint8 [n_pixels][4];
 *   n_pixels == 0 is a no-op; counts > max_iter are mapped by the same rule. */
fr_status colorize(const uint16_t* counts, int64_t n_pixels, int32_t max_iter,
                   const fr_palette* pal, uint8_t* out_rgba, fr_stream stream);

/* The paper's prescribed C-path: "the parameter moves clockwise along the cardioid
 * f(t) = ([2 cos t - cos 2t]/a, [2 sin t - sin 2t]/a), where a has the value 3.9"; a = 4
 * is the main-cardioid border; "if we let the size of the cardioid increase gradually
 * (by decreasing the values of a above), almost all relevant parameter values ... will be
 * traversed after a few trips".  Step rule (clockwise = decreasing t):
 * C_k = f(t_k, a_k); t_{k+1} = t_k - dt; when t_{k+1} <= -2 pi it wraps (+2 pi) and
 * a_{k+1} = max(a_k - da_per_rev, a_floor).  Host-only (no GPU work): fills out_host[n]
 * (HOST memory) for julia_render_path.  Errors: n < 0, non-finite inputs, a0 <= 0,
 * a_floor <= 0, dt < 0, da_per_rev < 0 -> FR_ERR_INVALID_ARG. */
fr_status fr_cardioid_path(double t0, double a0, double dt, double da_per_rev, double a_floor,
                           int32_t n, fr_complex* out_host);

/* Rows a rank holds under `bands` for a frame of `height` rows; -1 if invalid. */
int64_t fr_band_local_rows(int32_t height, fr_bands bands);

/* Global row of the rank's local row `local_row`; -1 if out of range/invalid. */
int64_t fr_band_global_row(int32_t height, fr_bands bands, int64_t local_row);

const char* fr_status_str(fr_status s);
/* The cudaError_t of the most recent FR_ERR_CUDA in this thread (0 if none). */
int32_t fr_last_cuda_error(void);
/* Diagnostics: when trace_dev (device, >= 3 uint64 per warp of the refill grid) is
 * non-null, the lane-refill kernel records per warp the %globaltimer (ns) at entry, at
 * chunk-supply exhaustion and at exit; NULL turns it off (the default).  Synchronous. */
fr_status fr_debug_refill_trace(void* trace_dev);

/* Number of kernels this library has launched in this process (monotonic). */
uint64_t fr_launch_count(void);
/* Library version string. */
const char* fr_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FRACTAL_H_ */
