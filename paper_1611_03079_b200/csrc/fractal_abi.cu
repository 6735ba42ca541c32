// fractal_abi.cu -- libfractal: the C ABI of include/fractal.h on top of the sm_100a
// kernels in escape_kernels.cuh.  Host side: validation, binary64 parameter
// derivation, chunking of C-paths into kernel parameters, dispatch.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>
#include <mutex>
#include <new>
#include <utility>
#include <type_traits>

#include "../../include/fractal.h"
#include "escape_kernels.cuh"

namespace {

std::atomic<uint64_t> g_launches{0};
thread_local int32_t g_last_cuda_error = 0;

constexpr int64_t kMaxFramePixels = int64_t(1) << 31;  // S:182 resource limit

// Tuning knobs read once from the environment (thread-safe: function-local statics are
// initialised exactly once).  Defaults are the measured best settings.
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}

// Vote block of the fast fp32 two-orbit loops in S2 and P1 (FRACTAL_VOTE_K: 2 default
// since the packed loop, 4 selectable).  Same box, round 2: cfg2 21.8 -> 20.6 us, cfg3
// 0.1695 -> 0.1653 ms (profiles/r02/ab_votek_*.txt); with the scalar loop of round 1,
// 4 was faster
int vote_k() {
  static const int v = env_int("FRACTAL_VOTE_K", 2);
  return v == 4 ? 4 : 2;
}

bool env_is(const char* name, const char* value) {
  const char* e = std::getenv(name);
  return e && !std::strcmp(e, value);
}

inline bool is_fin(double v) { return std::isfinite(v); }

fr_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FR_OK;
  g_last_cuda_error = (int32_t)e;
  return FR_ERR_CUDA;
}

fr_status check_frame(fr_window win, int32_t width, int32_t height, int32_t max_iter) {
  if (width < 1 || height < 1) return FR_ERR_INVALID_ARG;
  if (!(is_fin(win.center_re) && is_fin(win.center_im) && is_fin(win.half_w) &&
        is_fin(win.half_h)))
    return FR_ERR_INVALID_ARG;
  if (!(win.half_w > 0.0) || !(win.half_h > 0.0)) return FR_ERR_INVALID_ARG;
  if (max_iter < 1) return FR_ERR_INVALID_ARG;
  if (max_iter > 65535) return FR_ERR_UNSUPPORTED;
  if ((int64_t)width * (int64_t)height > kMaxFramePixels) return FR_ERR_TOO_LARGE;
  return FR_OK;
}

bool bands_valid(int32_t height, fr_bands b) {
  (void)height;
  return b.band_rows >= 0 && b.n_ranks >= 1 && b.rank >= 0 && b.rank < b.n_ranks &&
         (b.band_rows > 0 || (b.n_ranks == 1 && b.rank == 0));
}

int64_t local_rows(int32_t height, fr_bands b) {
  if (!bands_valid(height, b)) return -1;
  if (b.band_rows == 0) return height;
  const int64_t nb = ((int64_t)height + b.band_rows - 1) / b.band_rows;
  int64_t rows = 0;
  for (int64_t band = b.rank; band < nb; band += b.n_ranks) {
    const int64_t r0 = band * b.band_rows;
    const int64_t r1 = r0 + b.band_rows < height ? r0 + b.band_rows : height;
    rows += r1 - r0;
  }
  return rows;
}

// RGBA bytes as one little-endian word (R in the low byte: the in-memory byte order)
uint32_t rgba_word(uint8_t r, uint8_t g, uint8_t b, uint8_t a) {
  return (uint32_t)r | ((uint32_t)g << 8) | ((uint32_t)b << 16) | ((uint32_t)a << 24);
}

fr_status make_palette(const fr_palette* pal, fr::Palette* out) {
  std::memset(out, 0, sizeof(*out));
  if (!pal) return FR_OK;
  if (!pal->rgba || pal->n < 2 || pal->n > 256) return FR_ERR_INVALID_ARG;
  for (int i = 0; i < pal->n; ++i)
    out->e[i] = rgba_word(pal->rgba[4 * i], pal->rgba[4 * i + 1], pal->rgba[4 * i + 2],
                            pal->rgba[4 * i + 3]);
  out->interior = rgba_word(pal->interior[0], pal->interior[1], pal->interior[2],
                              pal->interior[3]);
  out->n = (uint32_t)pal->n;
  out->magic = (uint32_t)((((uint64_t)1 << 32) + (uint64_t)pal->n - 1) / (uint64_t)pal->n);
  return FR_OK;
}

// Device copies of palettes, cached per device by content (a 64-bit hash, confirmed by
// comparing the entries): kernels S2 and P1 read colours through L1 instead of staging
// the palette in shared memory behind a CTA barrier.  A new palette is uploaded once,
// outside any graph capture (like the workspaces).
struct DevPalette {
  std::vector<uint32_t> entries;
  uint32_t* ptr;
};
std::mutex g_pal_mutex;
std::map<std::pair<int, uint64_t>, std::vector<DevPalette>> g_pal_dev;

bool capturing(cudaStream_t s);

cudaError_t device_palette(fr::Palette& p, cudaStream_t s) {
  p.dev = nullptr;
  if (p.n == 0) return cudaSuccess;
  uint64_t h = 1469598103934665603ull;  // FNV-1a over the entries
  for (uint32_t i = 0; i < p.n; ++i) {
    for (int k = 0; k < 4; ++k) h = (h ^ ((p.e[i] >> (8 * k)) & 0xffu)) * 1099511628211ull;
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_pal_mutex);
  auto& bucket = g_pal_dev[std::make_pair(dev, h)];
  for (const DevPalette& d : bucket) {
    if (d.entries.size() == p.n &&
        std::memcmp(d.entries.data(), p.e, p.n * sizeof(uint32_t)) == 0) {
      p.dev = d.ptr;
      return cudaSuccess;
    }
  }
  if (capturing(s)) return cudaErrorStreamCaptureUnsupported;
  uint32_t* ptr = nullptr;
  e = cudaMalloc(&ptr, p.n * sizeof(uint32_t));
  if (e != cudaSuccess) return e;
  // stream-ordered upload on the caller's stream, then wait for it: the copy is shared
  // by later calls on any stream, which are not ordered after `s` (one-time cost)
  bucket.push_back(DevPalette{std::vector<uint32_t>(p.e, p.e + p.n), ptr});
  e = cudaMemcpyAsync(ptr, bucket.back().entries.data(), p.n * sizeof(uint32_t),
                      cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    bucket.pop_back();
    cudaFree(ptr);
    return e;
  }
  p.dev = ptr;
  return cudaSuccess;
}

fr::PalRef pal_ref(const fr::Palette& p) {
  fr::PalRef r;
  r.dev = p.dev;
  r.interior = p.interior;
  r.n = p.n;
  r.magic = p.magic;
  return r;
}

// Parameter derivation in binary64: hx = half_w / W, hy = half_h / H.
fr::Geom make_geom(fr_window win, int32_t width, int32_t height, int32_t max_iter,
                   fr_bands b, int64_t rows, uint16_t* counts, uint8_t* rgba) {
  fr::Geom g;
  g.cx = win.center_re;
  g.cy = win.center_im;
  g.hx = win.half_w / (double)width;
  g.hy = win.half_h / (double)height;
  g.W = width;
  g.H = height;
  g.rows = (int)rows;
  g.band_rows = b.band_rows;
  g.n_ranks = b.n_ranks;
  g.rank = b.rank;
  g.max_iter = max_iter;
  g.tiles_x = (width + fr::kTileW - 1) / fr::kTileW;
  g.frame_stride = rows * (int64_t)width;
  g.counts = counts;
  g.counts8 = nullptr;
  g.rgba = reinterpret_cast<uint32_t*>(rgba);
  g.grid2d = 0;
  return g;
}

// iterations per vote block of the static kernel (fp64: 8).  K = 2 for fp32 fast was
// measured slower on the bench workload (3.46 vs 3.44 ms).
constexpr int kStaticK = 4;
constexpr int kFramesPerCta = 32;  // frames of a path chunk rendered per CTA (static kernel); FRACTAL_FPC overrides

// Launch grid of kernels S/S2: (tiles_x, tiles_y, groups) when tiles_y fits grid y
// (kernel-side tile_of needs no division), else (tiles_x * tiles_y, groups, 1).
dim3 tile_grid(fr::Geom& g, int64_t tiles_y, int groups) {
  g.grid2d = tiles_y <= 65535 ? 1 : 0;
  if (g.grid2d) return dim3((unsigned)g.tiles_x, (unsigned)tiles_y, (unsigned)groups);
  return dim3((unsigned)((int64_t)g.tiles_x * tiles_y), (unsigned)groups, 1);
}

// Launch with programmatic dependent launch (PDL): the kernel may start
// while the previous kernel of the stream finishes; it calls pdl_wait() before touching
// global memory.  FRACTAL_PDL=0 launches plainly (A/B).
bool pdl_on() {
  static const bool on = !env_is("FRACTAL_PDL", "0");
  return on;
}
template <class... KArgs, class... Args>
cudaError_t launch_pdl_n(void (*kernel)(KArgs...), dim3 grid, unsigned threads, cudaStream_t s,
                         Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_on() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, cudaStream_t s, Args&&... args) {
  return launch_pdl_n(kernel, grid, fr::kThreads, s, std::forward<Args>(args)...);
}

template <class T, bool STRICT, bool MANDEL, bool COLOR, int NC>
cudaError_t launch_tiles_t(const fr::Geom& g0, const fr::Palette& pal, const fr::CList<T, NC>& cs,
                           int n_frames, int frame0, cudaStream_t s) {
  fr::Geom g = g0;
  static const int fpc_env = env_int("FRACTAL_FPC", 0);
  const int fpc_want = fpc_env > 0 ? fpc_env : kFramesPerCta;
  const int fpc = n_frames < fpc_want ? n_frames : fpc_want;
  // one frame, fp32 (either mode): two pixels per thread (kernel S2; FRACTAL_S2=0 disables)
  static const bool s2 = !env_is("FRACTAL_S2", "0");
  if constexpr (NC == 1 && std::is_same<T, float>::value) {
    if (s2 && g.counts8 == nullptr) {
      const dim3 grid2 =
          tile_grid(g, (g.rows + 2 * fr::kTileH - 1) / (2 * fr::kTileH) * (8 / FR_S2_WARPS), 1);
      auto k2 = fr::escape_tile2_kernel<STRICT, MANDEL, COLOR>;
      if constexpr (!STRICT) {
        if (vote_k() == 2) k2 = fr::escape_tile2_kernel<STRICT, MANDEL, COLOR, 2>;
      }
      const cudaError_t e =
          launch_pdl_n(k2, grid2, fr::kS2Threads, s, g, pal_ref(pal), cs.re[0], cs.im[0]);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return e;
    }
  }
  // C-path frames in FP32_FAST: kernel SX (x-adjacent pixel pairs, whole-sector count
  // stores; FRACTAL_SX=0 keeps kernel S's frame pairs)
  if constexpr (NC > 1 && !STRICT && !MANDEL && std::is_same<T, float>::value) {
    static const bool sx = !env_is("FRACTAL_SX", "0");
    if (sx) {
      fr::Geom gx = g;
      gx.tiles_x = (g.W + fr::kTileWX - 1) / fr::kTileWX;
      // 128 frames per CTA, one shared-memory C chunk (bench, 4-warp CTAs: 32/64/128/256
      // -> 2.347/2.296/2.289/2.449 ms, profiles/r02/ab_sx_fpc_w4.txt); FRACTAL_FPC overrides
      const int fpcx = fpc_env > 0 ? fpc : (n_frames < 128 ? n_frames : 128);
      const dim3 gridx =
          tile_grid(gx, (g.rows + fr::kSxRows - 1) / fr::kSxRows, (n_frames + fpcx - 1) / fpcx);
      // VEC: both pixels of every lane pair in or out together, pair stores aligned
      const int es = g.counts8 != nullptr ? 1 : 2;
      const uintptr_t base_c = g.counts8 != nullptr ? reinterpret_cast<uintptr_t>(g.counts8)
                                                    : reinterpret_cast<uintptr_t>(g.counts);
      const bool vec = (g.W % 2) == 0 && (g.frame_stride % 2) == 0 && base_c % (2 * es) == 0 &&
                       (!COLOR || reinterpret_cast<uintptr_t>(g.rgba) % 8 == 0);
      auto kx = g.counts8 != nullptr
                    ? (vec ? fr::escape_pathx_kernel<NC, 1, COLOR, true>
                           : fr::escape_pathx_kernel<NC, 1, COLOR, false>)
                    : (vec ? fr::escape_pathx_kernel<NC, 2, COLOR, true>
                           : fr::escape_pathx_kernel<NC, 2, COLOR, false>);
      kx<<<gridx, fr::kSxThreads, 0, s>>>(gx, pal_ref(pal), cs, frame0, n_frames, fpcx);
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return cudaGetLastError();
    }
  }
  const dim3 grid = tile_grid(g, (g.rows + fr::kTileH - 1) / fr::kTileH, (n_frames + fpc - 1) / fpc);
#ifndef FR_STATIC_K_FAST  // vote block of kernel S's fast fp32 frame pairs (A/B knob)
#define FR_STATIC_K_FAST kStaticK
#endif
  constexpr int KD = sizeof(T) == 8 ? 2 * kStaticK : (STRICT ? kStaticK : FR_STATIC_K_FAST);
  if (g.counts8 != nullptr) {  // uint8 counts: path chunks only (julia_render_path8)
    if constexpr (NC > 1 && !MANDEL)
      fr::escape_tile_kernel<T, STRICT, MANDEL, COLOR, KD, NC, 0, 1>
          <<<grid, fr::kThreads, 0, s>>>(g, pal, cs, frame0, n_frames, fpc);
    else
      return cudaErrorInvalidValue;
  } else if constexpr (NC == 1) {  // single frames: PDL (the kernel waits before storing)
    const cudaError_t e = launch_pdl(fr::escape_tile_kernel<T, STRICT, MANDEL, COLOR, KD, NC>,
                                     grid, s, g, pal, cs, frame0, n_frames, fpc);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return e;
  } else {
    fr::escape_tile_kernel<T, STRICT, MANDEL, COLOR, KD, NC>
        <<<grid, fr::kThreads, 0, s>>>(g, pal, cs, frame0, n_frames, fpc);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// C in the kernel's state representation (C_T = RN_T(C), on the host;
// FAST modes keep 2C, an exact doubling).
template <class T, bool STRICT>
T state_of(double v) {
  const T t = (T)v;  // round to nearest (default FP environment)
  return STRICT ? t : t + t;
}

template <class T, bool STRICT, bool MANDEL, bool COLOR, int NC>
cudaError_t launch_tiles_conv(const fr::Geom& g, const fr::Palette& pal, const fr_complex* c,
                              int n_frames, int frame0, cudaStream_t s) {
  if constexpr (NC == 1) {  // single frames: no heap round trip (small-frame latency)
    fr::CList<T, 1> one;
    one.re[0] = MANDEL ? T(0) : state_of<T, STRICT>(c[0].re);
    one.im[0] = MANDEL ? T(0) : state_of<T, STRICT>(c[0].im);
    return launch_tiles_t<T, STRICT, MANDEL, COLOR, 1>(g, pal, one, n_frames, frame0, s);
  }
  fr::CList<T, NC>* cs = new (std::nothrow) fr::CList<T, NC>;
  if (!cs) return cudaErrorMemoryAllocation;
  for (int k = 0; k < n_frames && !MANDEL; ++k) {
    cs->re[k] = state_of<T, STRICT>(c[k].re);
    cs->im[k] = state_of<T, STRICT>(c[k].im);
  }
  if (MANDEL) cs->re[0] = cs->im[0] = T(0);
  const cudaError_t e = launch_tiles_t<T, STRICT, MANDEL, COLOR, NC>(g, pal, *cs, n_frames, frame0, s);
  delete cs;
  return e;
}

template <bool MANDEL, bool COLOR, int NC>
cudaError_t launch_tiles_mode(fr_mode mode, const fr::Geom& g, const fr::Palette& pal,
                              const fr_complex* c, int n_frames, int frame0, cudaStream_t s) {
  switch (mode) {
    case FR_FP32_FAST:
      return launch_tiles_conv<float, false, MANDEL, COLOR, NC>(g, pal, c, n_frames, frame0, s);
    case FR_FP32_STRICT:
      return launch_tiles_conv<float, true, MANDEL, COLOR, NC>(g, pal, c, n_frames, frame0, s);
    case FR_FP64_FAST:
      return launch_tiles_conv<double, false, MANDEL, COLOR, NC>(g, pal, c, n_frames, frame0, s);
    case FR_FP64_STRICT:
      return launch_tiles_conv<double, true, MANDEL, COLOR, NC>(g, pal, c, n_frames, frame0, s);
  }
  return cudaErrorInvalidValue;
}

template <bool MANDEL, int NC>
cudaError_t launch_tiles(fr_mode mode, bool color, const fr::Geom& g, const fr::Palette& pal,
                         const fr_complex* c, int n_frames, int frame0, cudaStream_t s) {
  if (color) return launch_tiles_mode<MANDEL, true, NC>(mode, g, pal, c, n_frames, frame0, s);
  return launch_tiles_mode<MANDEL, false, NC>(mode, g, pal, c, n_frames, frame0, s);
}

// ---------------------------------------------------------------- refill kernel (R)
// Per-(device, stream) workspace holding the chunk counter.  Created (zeroed) on first
// use outside any graph capture; the kernel's last CTA resets it, so later launches on
// the same stream -- including CUDA-graph replays -- find it zeroed.
std::mutex g_ws_mutex;
std::map<std::pair<int, uintptr_t>, fr::Workspace*> g_ws;

// Lazily created per-stream device buffers cannot be created while the stream is being
// captured into a CUDA graph (cudaMalloc is not capturable): make the first call on a
// stream outside capture (tests/bench warm up first); during capture a missing buffer
// is reported as cudaErrorStreamCaptureUnsupported instead of breaking the capture.
bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st != cudaStreamCaptureStatusNone;
}

cudaError_t workspace_for(cudaStream_t s, fr::Workspace** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  auto key = std::make_pair(dev, (uintptr_t)s);
  auto it = g_ws.find(key);
  if (it != g_ws.end()) {
    *out = it->second;
    return cudaSuccess;
  }
  if (capturing(s)) return cudaErrorStreamCaptureUnsupported;
  fr::Workspace* w = nullptr;
  e = cudaMalloc(&w, sizeof(fr::Workspace));
  if (e != cudaSuccess) return e;
  // zeroed in stream order on `s` (the first kernel to use it runs on `s`); the host
  // waits once so that no later ordering question remains
  e = cudaMemsetAsync(w, 0, sizeof(fr::Workspace), s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFree(w);
    return e;
  }
  g_ws[key] = w;
  *out = w;
  return cudaSuccess;
}

// Library-owned device buffers cached per (device, stream), grown on demand and created
// outside any graph capture (like the workspace).
std::vector<void*> g_retired;  // outgrown buffers, kept alive for captured graphs
cudaError_t buffer_for(std::map<std::pair<int, uintptr_t>, std::pair<void*, size_t>>& g_cont,
                       cudaStream_t s, size_t bytes, void** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(g_ws_mutex);
  auto key = std::make_pair(dev, (uintptr_t)s);
  auto it = g_cont.find(key);
  if (it != g_cont.end() && it->second.second >= bytes) {
    *out = it->second.first;
    return cudaSuccess;
  }
  if (capturing(s)) return cudaErrorStreamCaptureUnsupported;
  if (it != g_cont.end()) {
    // Grown: the old buffer is NOT freed -- a CUDA graph captured earlier on this stream
    // may still hold its address and be replayed later -- but parked until process exit
    // (growth is rare: at most one step per frame size class).
    g_retired.push_back(it->second.first);
    g_cont.erase(it);
  }
  void* p = nullptr;
  e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return e;
  g_cont[key] = std::make_pair(p, bytes);
  *out = p;
  return cudaSuccess;
}

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
      sms <= 0)
    sms = 148;
  return sms;
}

// Chunks per CTA of the CTA-local refill grid; 0 = persistent grid with a global chunk
// counter.  Measured (B200): persistent is faster for heavy-tailed Julia frames (cfg3:
// 0.30 vs 0.36 ms), CTA-local for long uniform counts (cfg5: 641 vs 663 ms).
// FRACTAL_REFILL_CPC overrides.
int refill_cpc(bool amort) {
  static const int v = env_int("FRACTAL_REFILL_CPC", -1);
  if (v >= 0) return v;
  return amort ? 16 : 0;
}

template <class T, bool STRICT, bool MANDEL, bool COLOR, int K, int TH, bool AMORT = false>
cudaError_t launch_refill_t(const fr::Geom& g, const fr::Palette& pal, double2 c, cudaStream_t s) {
  const T jcr = MANDEL ? T(0) : state_of<T, STRICT>(c.x);
  const T jci = MANDEL ? T(0) : state_of<T, STRICT>(c.y);
  auto kern = fr::escape_refill_kernel<T, STRICT, MANDEL, COLOR, AMORT, K, TH>;
  const unsigned n_chunks =
      (unsigned)((int64_t)g.tiles_x * ((g.rows + fr::kTileH - 1) / fr::kTileH));
  const int cpc = refill_cpc(AMORT);
  cudaError_t e;
  if (cpc > 0) {
    const unsigned blocks = (n_chunks + cpc - 1) / cpc;
    kern<<<blocks, fr::kThreads, 0, s>>>(g, pal, jcr, jci, nullptr, n_chunks, (unsigned)cpc);
  } else {
    fr::Workspace* ws = nullptr;
    e = workspace_for(s, &ws);
    if (e != cudaSuccess) return e;
    static const int occ = [&] {  // per instantiation, computed once
      int o = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, fr::kThreads, 0) !=
              cudaSuccess || o <= 0)
        o = 1;
      return o;
    }();
    int64_t blocks = (int64_t)sm_count() * occ;
    const int64_t need = (n_chunks + fr::kThreads / 32 - 1) / (fr::kThreads / 32);
    if (blocks > need) blocks = need;
    if (blocks < 1) blocks = 1;
    kern<<<(unsigned)blocks, fr::kThreads, 0, s>>>(g, pal, jcr, jci, ws, n_chunks, 0u);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

// Two-phase kernels P1 + P2: the queue header (zeroed once per (device, stream), reset by
// P2's last warp) and an item buffer of one QItem per pixel of the call, grown on demand.
std::map<std::pair<int, uintptr_t>, std::pair<void*, size_t>> g_queue, g_items;
constexpr int64_t kTwoPhaseMaxPixels = int64_t(1) << 25;  // item buffer <= 1 GiB (fp64)

// P1's budget (FRACTAL_BUDGET, multiple of 4): 96 before an exact P2, 48 before the
// amortised P2, whose iterations are cheaper (cfg3 fast, 3 CTAs/SM, K 64: 48/64/96
// 0.1679/0.1685/0.1719 ms)
// fp64 fast with the amortised P1 (below): 64 (cfg3 FP64_FAST, KS 8, prefix 8: budget
// 32/40/48/64 0.2459/0.2442/0.2443/0.2433 ms; exact P1 at 48 0.2464)
// fp32 fast with the packed amortised P1 (round 2): 128 (cfg3, KS 8, prefix 8 / 16:
// budget 96/128/160/192/256 0.1647/0.1630-0.1637/0.1652/0.1670/0.1735 ms against the
// exact P1 at 48 0.1655; profiles/r02/ab_p1_packed_amort.txt)
int twophase_budget(bool amort, bool f64) {
  static const int b = env_int("FRACTAL_BUDGET", 0);
  const int v = b > 0 ? b : (amort ? (f64 ? 64 : 128) : 96);
  return v < 4 ? 4 : v - v % 4;
}

bool p2s_on() {  // experimental packed P2: off, slower than the one-orbit P2
  static const bool v = env_int("FRACTAL_P2S", 0) != 0;
  return v;
}


#ifndef FR_P1A_KS  // amortised P1 sub-block in fp32 (0 = exact per-iteration test)
#define FR_P1A_KS 8
#endif
#ifndef FR_P1A_PRE
#define FR_P1A_PRE 8
#endif
template <class T, bool STRICT, bool MANDEL, bool COLOR, int K, int TH, int KA, int THA>
cudaError_t launch_twophase_t(const fr::Geom& g0, const fr::Palette& pal, double2 c,
                              cudaStream_t s, bool amort) {
  fr::Geom g = g0;
  const T jcr = MANDEL ? T(0) : state_of<T, STRICT>(c.x);
  const T jci = MANDEL ? T(0) : state_of<T, STRICT>(c.y);
  const int64_t n = (int64_t)g.rows * g.W;
  void* qp = nullptr;
  bool fresh = false;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_ws_mutex);
    fresh = g_queue.find(std::make_pair(dev, (uintptr_t)s)) == g_queue.end();
  }
  cudaError_t e = buffer_for(g_queue, s, sizeof(fr::ContQueue), &qp);
  if (e != cudaSuccess) return e;
  if (fresh) {  // zeroed in stream order on `s`, before P1 appends to it
    e = cudaMemsetAsync(qp, 0, sizeof(fr::ContQueue), s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return e;
  }
  auto* q = static_cast<fr::ContQueue*>(qp);
  void* ip = nullptr;
  // (+ 128 positions per warp of the largest P2 grid: P2S reserves whole ranges)
  const size_t extra = (size_t)sm_count() * 8 * (fr::kThreads / 32) * 128;
  e = buffer_for(g_items, s, ((size_t)n + extra) * sizeof(fr::QItem<T>), &ip);
  if (e != cudaSuccess) return e;
  auto* items = static_cast<fr::QItem<T>*>(ip);
  // FRACTAL_P1_TILES=2: each P1 CTA renders two vertically adjacent tiles (exact P1 only)
  static const int p1nt = env_int("FRACTAL_P1_TILES", 1) == 2 ? 2 : 1;
  const dim3 grid1 = tile_grid(
      g, (g.rows + 2 * p1nt * fr::kTileH - 1) / (2 * p1nt * fr::kTileH) * (8 / FR_P1_WARPS), 1);
  const int budget = twophase_budget(amort, sizeof(T) == 8);
  // amortised P1 under the same precondition as the amortised P2 (FRACTAL_P1_AMORT:
  // 0 = exact test, else sub-blocks of 4 or 8 when the budget is a multiple of it)
  // FRACTAL_P1_PRE: exact prefix of 0 / 8 / 16 iterations before the amortised blocks
  // Defaults: exact P1 in fp32 (the amortised one is 3.5% slower there); in fp64 fast
  // sub-blocks of 8 after an exact prefix of 8 (cfg3 0.2464 -> 0.2433 ms with budget 64)
  static const int p1ks_env = env_int("FRACTAL_P1_AMORT", -1);
  static const int p1pre_env = env_int("FRACTAL_P1_PRE", -1);
  const int p1ks = p1ks_env >= 0 ? p1ks_env : (sizeof(T) == 8 ? 8 : FR_P1A_KS);
  const int p1pre = p1pre_env >= 0 ? p1pre_env : (sizeof(T) == 8 ? 8 : FR_P1A_PRE);
  auto kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR>;
  if constexpr (!STRICT && std::is_same<T, float>::value) {
    if (vote_k() == 2) kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 0, 0, 2>;
  }
  if constexpr (!STRICT) {
    if (amort && budget > p1pre && (budget - p1pre) % 8 == 0) {
      if (p1ks == 4 && p1pre == 0) kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 4>;
      if (p1ks == 8 && p1pre == 0) kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 8>;
      if (p1ks == 4 && p1pre == 8)
        kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 4, 8>;
      if (p1ks == 8 && p1pre == 8)
        kern1 = vote_k() == 2 && sizeof(T) == 4
                    ? fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 8, 8, 2>
                    : fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 8, 8>;
      if (p1ks == 4 && p1pre == 16)
        kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 4, 16>;
      if (p1ks == 8 && p1pre == 16)
        kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 8, 16>;
    }
  }
  // the two-tile CTA is the exact P1 alone (it overrides the other P1 knobs): its grid
  // covers half as many tile rows
  if (p1nt == 2) kern1 = fr::escape_budget_kernel<T, STRICT, MANDEL, COLOR, 0, 0, 4, 2>;
  kern1<<<grid1, fr::kP1Threads, 0, s>>>(g, pal_ref(pal), jcr, jci, budget, q, items);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  // FP32_FAST under the precondition: the packed two-slot P2 with stashes (P2S)
  // (FRACTAL_P2S=0 falls back; FRACTAL_P2S_K: block 16/32/64)
  if constexpr (!STRICT && std::is_same<T, float>::value) {
    if (amort && p2s_on()) {
      static const int ks = env_int("FRACTAL_P2S_K", 32);
      auto k2 = fr::escape_cont2s_kernel<MANDEL, COLOR, 32>;
      if (ks == 16) k2 = fr::escape_cont2s_kernel<MANDEL, COLOR, 16>;
      else if (ks == 64) k2 = fr::escape_cont2s_kernel<MANDEL, COLOR, 64>;
      static const int occs = [&] {
        int o = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k2, fr::kThreads, 0) !=
                cudaSuccess || o <= 0)
          o = 1;
        return o;
      }();
      static const int occ_env = env_int("FRACTAL_P2_OCC", 0);
      const int want = occ_env > 0 ? occ_env : 3;
      const int o2 = want < occs ? want : occs;
      k2<<<(unsigned)(sm_count() * o2), fr::kThreads, 0, s>>>(g, pal_ref(pal), jcr, jci, q,
                                                              items);
      e = cudaGetLastError();
      if (e != cudaSuccess) {
        cudaMemsetAsync(qp, 0, sizeof(fr::ContQueue), s);
        return e;
      }
      g_launches.fetch_add(1, std::memory_order_relaxed);
      return cudaSuccess;
    }
  }
  // P2 with the amortised block-end test when the escape-monotonicity precondition
  // holds (host-checked), else the exact per-iteration test
  // (strict modes never take the amortised kernel: it is not instantiated for them)
  auto kern = fr::escape_cont_kernel<T, STRICT, MANDEL, COLOR, K, TH, false>;
  if constexpr (!STRICT) {
    if (amort) kern = fr::escape_cont_kernel<T, STRICT, MANDEL, COLOR, KA, THA, true>;
  }
  static const int occ = [&] {
    int o = 0, oa = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &o, fr::escape_cont_kernel<T, STRICT, MANDEL, COLOR, K, TH, false>, fr::kThreads,
            0) != cudaSuccess || o <= 0)
      o = 1;
    oa = o;
    if constexpr (!STRICT) {
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
              &oa, fr::escape_cont_kernel<T, STRICT, MANDEL, COLOR, KA, THA, true>,
              fr::kThreads, 0) != cudaSuccess || oa <= 0)
        oa = 1;
    }
    return o < oa ? o : oa;
  }();
  // P2 runs 2 CTAs per SM (FRACTAL_P2_OCC), not the occupancy limit: a few warps per
  // SMSP already saturate issue for this loop, and every extra resident lane only adds
  // to the work still in flight when the queue runs dry (cfg3: 8 CTAs 0.273 ms, 3 CTAs
  // 0.1975, 2 CTAs 0.1965; strict 0.250 vs 0.246)
  // The amortised P2 issues fewer instructions per iteration and runs best at 3 CTAs/SM
  // (cfg3 fast, K 64: 2/3/4 CTAs 0.1704/0.1687/0.1715 ms)
  static const int occ_env = env_int("FRACTAL_P2_OCC", 0);
  const int occ_want = occ_env > 0 ? occ_env : (amort ? 3 : 2);
  const int occ2 = occ_want < occ ? occ_want : occ;
  kern<<<(unsigned)(sm_count() * occ2), fr::kThreads, 0, s>>>(g, pal, jcr, jci, q, items);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    // P2 resets the queue header when it finishes; if it never ran, reset it here so
    // the next call does not start from P1's stale tail
    cudaMemsetAsync(qp, 0, sizeof(fr::ContQueue), s);
    return e;
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaSuccess;
}

#ifndef FR_P2_K  // compile-time knobs for same-box A/B (tools/ab_build.sh)
#define FR_P2_K 32
#endif
#ifndef FR_P2_K_STRICT
#define FR_P2_K_STRICT 32
#endif
#ifndef FR_P2_TH
#define FR_P2_TH 8
#endif
#ifndef FR_P2A_K  // amortised P2 (block, service threshold): cfg3 fast sweep, DESIGN §5.1c
#define FR_P2A_K 64   // with checkpointed sub-blocks of FR_P2A_KS = 8 (escape_kernels.cuh)
#endif
#ifndef FR_P2A_TH
#define FR_P2A_TH 12
#endif
#ifndef FR_P2A_K_F64
#define FR_P2A_K_F64 32  // cfg3 FP64_FAST: 16,12 0.2566; 32,12 0.2467; 32,16 0.2523; 64,12 0.2473 ms
#endif
#ifndef FR_P2A_TH_F64
#define FR_P2A_TH_F64 12
#endif
template <bool MANDEL, bool COLOR>
cudaError_t launch_twophase_mode(fr_mode mode, const fr::Geom& g, const fr::Palette& pal,
                                 double2 c, cudaStream_t s, bool amort) {
  switch (mode) {
    // P2 blocks of 32, service threshold 8 (cfg3 sweep at 2 CTAs/SM with the dry-queue
    // drain: 32,8 0.1925 ms; 24,8 0.1926; 64,8 0.1929; 32,12 0.1937; 32,6 0.1940;
    // 16,8 0.1966; 32,4 0.1989; 16,4 0.2062; 8,8 0.2112.  Strict: 32 0.234, 16 0.241)
    case FR_FP32_FAST:
      return launch_twophase_t<float, false, MANDEL, COLOR, FR_P2_K, FR_P2_TH, FR_P2A_K,
                               FR_P2A_TH>(g, pal, c, s, amort);
    // strict: the replayed 7-op step makes the amortised P2 slower (cfg3 0.2417 vs 0.2339
    // ms at 32,16), so strict modes keep the exact per-iteration test
    case FR_FP32_STRICT:
      return launch_twophase_t<float, true, MANDEL, COLOR, FR_P2_K_STRICT, FR_P2_TH, FR_P2A_K,
                               FR_P2A_TH>(g, pal, c, s, false);
    case FR_FP64_FAST:
      return launch_twophase_t<double, false, MANDEL, COLOR, 16, 8, FR_P2A_K_F64, FR_P2A_TH_F64>(
          g, pal, c, s, amort);
    case FR_FP64_STRICT:
      return launch_twophase_t<double, true, MANDEL, COLOR, 16, 8, 16, 16>(g, pal, c, s, false);
  }
  return cudaErrorInvalidValue;
}

// Amortised P2 for the fast modes when the escape-monotonicity precondition holds
// (monotone_ok, below); FRACTAL_P2_AMORT=0 keeps the exact per-iteration test.
bool monotone_ok(bool mandel, fr_complex c, fr_window w);
bool p2_amort(fr_mode mode, bool mandel, fr_complex c, fr_window w) {
  static const bool on = env_int("FRACTAL_P2_AMORT", 1) != 0;
  return on && (mode == FR_FP32_FAST || mode == FR_FP64_FAST) && monotone_ok(mandel, c, w);
}

// Kernel R: blocks of 16, service threshold 8 (cfg3 sweep: K 8-32 and
// TH 1-24 all within 0.30-0.36 ms, 16,8 best).
template <bool MANDEL, bool COLOR>
cudaError_t launch_refill_mode(fr_mode mode, const fr::Geom& g, const fr::Palette& pal,
                               double2 c, cudaStream_t s) {
  switch (mode) {
    case FR_FP32_FAST: return launch_refill_t<float, false, MANDEL, COLOR, 16, 8>(g, pal, c, s);
    case FR_FP32_STRICT: return launch_refill_t<float, true, MANDEL, COLOR, 16, 8>(g, pal, c, s);
    case FR_FP64_FAST: return launch_refill_t<double, false, MANDEL, COLOR, 16, 8>(g, pal, c, s);
    case FR_FP64_STRICT: return launch_refill_t<double, true, MANDEL, COLOR, 16, 8>(g, pal, c, s);
  }
  return cudaErrorInvalidValue;
}

// Kernel A: blocks of 64, service threshold 4 (cfg5 fp64 fast sweep, DESIGN.md §5.3:
// 64,4 592 ms; 32,4 609; 128,4 597; 64,8 601; 16,1 641-663).
template <class T, bool STRICT, bool MANDEL, bool COLOR>
cudaError_t launch_amort_t(const fr::Geom& g, const fr::Palette& pal, double2 c, cudaStream_t s) {
  return launch_refill_t<T, STRICT, MANDEL, COLOR, 64, 4, true>(g, pal, c, s);
}

template <bool MANDEL, bool COLOR>
cudaError_t launch_amort_mode(fr_mode mode, const fr::Geom& g, const fr::Palette& pal,
                              double2 c, cudaStream_t s) {
  switch (mode) {
    case FR_FP32_FAST: return launch_amort_t<float, false, MANDEL, COLOR>(g, pal, c, s);
    case FR_FP32_STRICT: return launch_amort_t<float, true, MANDEL, COLOR>(g, pal, c, s);
    case FR_FP64_FAST: return launch_amort_t<double, false, MANDEL, COLOR>(g, pal, c, s);
    case FR_FP64_STRICT: return launch_amort_t<double, true, MANDEL, COLOR>(g, pal, c, s);
  }
  return cudaErrorInvalidValue;
}

// Escape-monotonicity precondition of the amortised kernel: every C of
// the frame satisfies |C| <= 1.989 (Julia: the constant; Mandelbrot: the window's
// corners bound every pixel centre).
bool monotone_ok(bool mandel, fr_complex c, fr_window w) {
  const double lim = 1.989;
  if (!mandel) return std::hypot(c.re, c.im) <= lim;
  for (int sx = -1; sx <= 1; sx += 2)
    for (int sy = -1; sy <= 1; sy += 2)
      if (std::hypot(w.center_re + sx * w.half_w, w.center_im + sy * w.half_h) > lim)
        return false;
  return true;
}

// Scheduling policy for single frames (DESIGN.md §5 dispatch table):
// FRACTAL_SCHED=static|refill|amort|twophase overrides; default static for max_iter <
// 256, kernel A for deep Mandelbrot maps under the monotonicity precondition, else the
// two phases (P1 + P2; kernel R for frames too large for the survivor buffer).
enum Sched { kStatic = 0, kRefill = 1, kAmort = 2, kTwoPhase = 3 };

Sched choose_sched(bool mandel, fr_complex c, fr_window w, int max_iter) {
  static const int forced = env_is("FRACTAL_SCHED", "static")   ? kStatic
                            : env_is("FRACTAL_SCHED", "refill") ? kRefill
                            : env_is("FRACTAL_SCHED", "amort")  ? kAmort
                            : env_is("FRACTAL_SCHED", "twophase") ? kTwoPhase
                                                                 : -1;
  const bool mono = monotone_ok(mandel, c, w);
  if (forced >= 0) return (forced == kAmort && !mono) ? kRefill : (Sched)forced;
  if (max_iter < 256) return kStatic;
  // Long, low-divergence counts (deep Mandelbrot zooms) amortise the escape test;
  // heavy-tailed frames keep the exact per-iteration test: a budgeted static pass then
  // lane refill over its survivors (P1 + P2), or plain lane refill (R) when the frame
  // is too large for the survivor buffer.
  if (mandel && mono && max_iter >= 1000) return kAmort;
  return kTwoPhase;
}

bool mode_valid(fr_mode m) {
  return m == FR_FP32_FAST || m == FR_FP32_STRICT || m == FR_FP64_FAST || m == FR_FP64_STRICT;
}

fr_status render_frame(bool mandel, fr_complex c, fr_window win, int32_t width, int32_t height,
                       int32_t max_iter, fr_mode mode, fr_bands bands, uint16_t* out_counts,
                       const fr_palette* pal, uint8_t* out_rgba, fr_stream stream) {
  fr_status st = check_frame(win, width, height, max_iter);
  if (st != FR_OK) return st;
  if (!mode_valid(mode)) return FR_ERR_UNSUPPORTED;
  if (!mandel && !(is_fin(c.re) && is_fin(c.im))) return FR_ERR_INVALID_ARG;
  const int64_t rows = local_rows(height, bands);
  if (rows < 0) return FR_ERR_INVALID_ARG;
  fr::Palette p;
  st = make_palette(pal, &p);
  if (st != FR_OK) return st;
  if (rows == 0) return FR_OK;  // this rank holds no band: nothing to write (null ok)
  if (!out_counts) return FR_ERR_INVALID_ARG;
  if ((pal != nullptr) != (out_rgba != nullptr)) return FR_ERR_INVALID_ARG;
  const fr::Geom g = make_geom(win, width, height, max_iter, bands, rows, out_counts, out_rgba);
  cudaError_t e;
  if (pal != nullptr && (e = device_palette(p, stream)) != cudaSuccess) return cuda_status(e);
  const Sched sched = choose_sched(mandel, c, win, max_iter);
  if (sched != kStatic) {
    const double2 cc = make_double2(c.re, c.im);
    const bool col = pal != nullptr;
    if (sched == kAmort) {
      if (mandel)
        e = col ? launch_amort_mode<true, true>(mode, g, p, cc, stream)
                : launch_amort_mode<true, false>(mode, g, p, cc, stream);
      else
        e = col ? launch_amort_mode<false, true>(mode, g, p, cc, stream)
                : launch_amort_mode<false, false>(mode, g, p, cc, stream);
    } else if (sched == kTwoPhase &&
               max_iter > twophase_budget(p2_amort(mode, mandel, c, win),
                                          mode == FR_FP64_FAST || mode == FR_FP64_STRICT) &&
               (int64_t)g.rows * g.W <= kTwoPhaseMaxPixels) {
      const bool am = p2_amort(mode, mandel, c, win);
      if (mandel)
        e = col ? launch_twophase_mode<true, true>(mode, g, p, cc, stream, am)
                : launch_twophase_mode<true, false>(mode, g, p, cc, stream, am);
      else
        e = col ? launch_twophase_mode<false, true>(mode, g, p, cc, stream, am)
                : launch_twophase_mode<false, false>(mode, g, p, cc, stream, am);
    } else if (mandel) {
      e = col ? launch_refill_mode<true, true>(mode, g, p, cc, stream)
              : launch_refill_mode<true, false>(mode, g, p, cc, stream);
    } else {
      e = col ? launch_refill_mode<false, true>(mode, g, p, cc, stream)
              : launch_refill_mode<false, false>(mode, g, p, cc, stream);
    }
    return cuda_status(e);
  }
  e = mandel ? launch_tiles<true, 1>(mode, pal != nullptr, g, p, &c, 1, 0, stream)
             : launch_tiles<false, 1>(mode, pal != nullptr, g, p, &c, 1, 0, stream);
  return cuda_status(e);
}

template <class T, int FN, bool COLOR>
cudaError_t launch_fn_t(const fr::Geom& g0, const fr::Palette& pal, fr_complex c, cudaStream_t s) {
  fr::Geom g = g0;
  fr::CList<T, 1> cs;
  cs.re[0] = state_of<T, true>(c.re);
  cs.im[0] = state_of<T, true>(c.im);
#ifndef FR_FN2  // z^4 + c on the two-pixel S2 layout (escape_fn2_kernel; the rational map
#define FR_FN2 1  // measured slower there: profiles/r02/ab_fig4_fn2.txt)
#endif
  cudaError_t e;
  if constexpr (FR_FN2 && FN == 1) {
    const dim3 grid2 = tile_grid(g, (g.rows + 2 * fr::kTileH - 1) / (2 * fr::kTileH), 1);
    e = launch_pdl(fr::escape_fn2_kernel<T, FN, COLOR>, grid2, s, g, pal, cs.re[0], cs.im[0]);
  } else {
    const dim3 grid = tile_grid(g, (g.rows + fr::kTileH - 1) / fr::kTileH, 1);
    e = launch_pdl(fr::escape_tile_kernel<T, true, false, COLOR, 4, 1, FN>, grid, s, g, pal, cs,
                   0, 1, 1);
  }
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return e;
}

template <int FN>
cudaError_t launch_fn(fr_mode mode, bool color, const fr::Geom& g, const fr::Palette& pal,
                      fr_complex c, cudaStream_t s) {
  const bool f64 = (mode == FR_FP64_FAST || mode == FR_FP64_STRICT);
  if (f64) return color ? launch_fn_t<double, FN, true>(g, pal, c, s)
                        : launch_fn_t<double, FN, false>(g, pal, c, s);
  return color ? launch_fn_t<float, FN, true>(g, pal, c, s) : launch_fn_t<float, FN, false>(g, pal, c, s);
}

}  // namespace

extern "C" {

fr_status julia_render(fr_complex c, fr_window win, int32_t width, int32_t height,
                       int32_t max_iter, uint16_t* out_counts, fr_stream stream) {
  return render_frame(false, c, win, width, height, max_iter, FR_FP32_FAST, fr_bands{0, 1, 0},
                      out_counts, nullptr, nullptr, stream);
}

fr_status julia_render_ex(fr_complex c, fr_window win, int32_t width, int32_t height,
                          int32_t max_iter, fr_mode mode, fr_bands bands, uint16_t* out_counts,
                          const fr_palette* pal, uint8_t* out_rgba, fr_stream stream) {
  return render_frame(false, c, win, width, height, max_iter, mode, bands, out_counts, pal,
                      out_rgba, stream);
}

fr_status mandelbrot_param_map(fr_window win, int32_t width, int32_t height, int32_t max_iter,
                               fr_mode mode, fr_bands bands, uint16_t* out_counts,
                               const fr_palette* pal, uint8_t* out_rgba, fr_stream stream) {
  return render_frame(true, fr_complex{0.0, 0.0}, win, width, height, max_iter, mode, bands,
                      out_counts, pal, out_rgba, stream);
}

fr_status julia_render_fn(fr_function fn, fr_complex c, fr_window win, int32_t width,
                          int32_t height, int32_t max_iter, fr_mode mode, uint16_t* out_counts,
                          const fr_palette* pal, uint8_t* out_rgba, fr_stream stream) {
  if (fn == FR_FN_Z2)
    return julia_render_ex(c, win, width, height, max_iter, mode, fr_bands{0, 1, 0}, out_counts,
                           pal, out_rgba, stream);
  fr_status st = check_frame(win, width, height, max_iter);
  if (st != FR_OK) return st;
  if (!mode_valid(mode) || (fn != FR_FN_Z4 && fn != FR_FN_Z4_RATIONAL)) return FR_ERR_UNSUPPORTED;
  if (!(is_fin(c.re) && is_fin(c.im))) return FR_ERR_INVALID_ARG;
  if (!out_counts) return FR_ERR_INVALID_ARG;
  if ((pal != nullptr) != (out_rgba != nullptr)) return FR_ERR_INVALID_ARG;
  fr::Palette p;
  st = make_palette(pal, &p);
  if (st != FR_OK) return st;
  const fr::Geom g =
      make_geom(win, width, height, max_iter, fr_bands{0, 1, 0}, height, out_counts, out_rgba);
  const cudaError_t e = fn == FR_FN_Z4 ? launch_fn<1>(mode, pal != nullptr, g, p, c, stream)
                                       : launch_fn<2>(mode, pal != nullptr, g, p, c, stream);
  return cuda_status(e);
}

static fr_status render_path_impl(const fr_complex* c_host, int32_t n_frames, fr_window win,
                                  int32_t width, int32_t height, int32_t max_iter, fr_mode mode,
                                  uint16_t* out16, uint8_t* out8, const fr_palette* pal,
                                  uint8_t* out_rgba, fr_stream stream) {
  if (n_frames < 0) return FR_ERR_INVALID_ARG;
  fr_status st = check_frame(win, width, height, max_iter);
  if (st != FR_OK) return st;
  if (!mode_valid(mode)) return FR_ERR_UNSUPPORTED;
  if (out8 && max_iter > 255) return FR_ERR_UNSUPPORTED;
  if (n_frames == 0) return FR_OK;
  if (!c_host || (!out16 && !out8)) return FR_ERR_INVALID_ARG;
  if ((pal != nullptr) != (out_rgba != nullptr)) return FR_ERR_INVALID_ARG;
  for (int32_t k = 0; k < n_frames; ++k)
    if (!(is_fin(c_host[k].re) && is_fin(c_host[k].im))) return FR_ERR_INVALID_ARG;
  fr::Palette p;
  st = make_palette(pal, &p);
  if (st != FR_OK) return st;
  fr::Geom g = make_geom(win, width, height, max_iter, fr_bands{0, 1, 0}, height, out16,
                         out_rgba);
  g.counts8 = out8;
  cudaError_t e = cudaSuccess;
  // kernel SX reads colours from the device copy of the palette
  if (pal != nullptr && (e = device_palette(p, stream)) != cudaSuccess) return cuda_status(e);
  for (int32_t f0 = 0; f0 < n_frames && e == cudaSuccess; f0 += fr::kMaxPathChunk) {
    const int nf = n_frames - f0 < fr::kMaxPathChunk ? n_frames - f0 : fr::kMaxPathChunk;
    e = launch_tiles<false, fr::kMaxPathChunk>(mode, pal != nullptr, g, p, c_host + f0, nf, f0,
                                               stream);
  }
  return cuda_status(e);
}

fr_status julia_render_path(const fr_complex* c_host, int32_t n_frames, fr_window win,
                            int32_t width, int32_t height, int32_t max_iter, fr_mode mode,
                            uint16_t* out_counts, const fr_palette* pal, uint8_t* out_rgba,
                            fr_stream stream) {
  if (n_frames > 0 && !out_counts) return FR_ERR_INVALID_ARG;
  return render_path_impl(c_host, n_frames, win, width, height, max_iter, mode, out_counts,
                          nullptr, pal, out_rgba, stream);
}

fr_status julia_render_path8(const fr_complex* c_host, int32_t n_frames, fr_window win,
                             int32_t width, int32_t height, int32_t max_iter, fr_mode mode,
                             uint8_t* out_counts8, const fr_palette* pal, uint8_t* out_rgba,
                             fr_stream stream) {
  if (n_frames > 0 && !out_counts8) return FR_ERR_INVALID_ARG;
  return render_path_impl(c_host, n_frames, win, width, height, max_iter, mode, nullptr,
                          out_counts8, pal, out_rgba, stream);
}

fr_status julia_render_path_host(const fr_complex* c_host, int32_t n_frames, fr_window win,
                                 int32_t width, int32_t height, int32_t max_iter, fr_mode mode,
                                 int32_t bytes_per_count, void* out_host, fr_stream stream) {
  if (n_frames < 0) return FR_ERR_INVALID_ARG;
  if (bytes_per_count != 1 && bytes_per_count != 2) return FR_ERR_INVALID_ARG;
  fr_status st = check_frame(win, width, height, max_iter);
  if (st != FR_OK) return st;
  if (!mode_valid(mode)) return FR_ERR_UNSUPPORTED;
  if (bytes_per_count == 1 && max_iter > 255) return FR_ERR_UNSUPPORTED;
  if (n_frames == 0) return FR_OK;
  if (!c_host || !out_host) return FR_ERR_INVALID_ARG;
  for (int32_t k = 0; k < n_frames; ++k)
    if (!(is_fin(c_host[k].re) && is_fin(c_host[k].im))) return FR_ERR_INVALID_ARG;
  const size_t frame_bytes = (size_t)width * (size_t)height * (size_t)bytes_per_count;
  // staging: two buffers of up to 128 MiB (at least one frame each)
  int32_t chunk = (int32_t)((size_t)(128u << 20) / frame_bytes);
  if (chunk < 1) chunk = 1;
  if (chunk > n_frames) chunk = n_frames;
  cudaStream_t s = stream, cs = nullptr;
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t rendered[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
  cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
  {
    // stream-ordered staging from the device's default pool; keep freed staging
    // memory in the pool between calls instead of returning it at every sync
    static std::once_flag once;
    std::call_once(once, [] {
      int dev = 0;
      cudaMemPool_t pool;
      if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = 1ull << 30;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    });
  }
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = cudaMallocAsync(&buf[b], frame_bytes * (size_t)chunk, s);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&rendered[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming);
  }
  fr_status rs = FR_OK;
  // the first chunk's render is the only one not hidden behind a copy: keep it small
  const int32_t first = chunk / 8 > 0 ? chunk / 8 : 1;
  for (int32_t f0 = 0, i = 0, nf = 0; f0 < n_frames && e == cudaSuccess && rs == FR_OK;
       f0 += nf, ++i) {
    const int b = i & 1;
    const int32_t want = i == 0 ? first : chunk;
    nf = n_frames - f0 < want ? n_frames - f0 : want;
    if (i >= 2) e = cudaStreamWaitEvent(s, copied[b], 0);  // buffer b's copy is done
    if (e != cudaSuccess) break;
    rs = bytes_per_count == 2
             ? render_path_impl(c_host + f0, nf, win, width, height, max_iter, mode,
                                static_cast<uint16_t*>(buf[b]), nullptr, nullptr, nullptr,
                                stream)
             : render_path_impl(c_host + f0, nf, win, width, height, max_iter, mode, nullptr,
                                static_cast<uint8_t*>(buf[b]), nullptr, nullptr, stream);
    if (rs != FR_OK) break;
    e = cudaEventRecord(rendered[b], s);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, rendered[b], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(static_cast<char*>(out_host) + (size_t)f0 * frame_bytes, buf[b],
                          frame_bytes * (size_t)nf, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaEventRecord(copied[b], cs);
  }
  if (cs) {
    const cudaError_t e2 = cudaStreamSynchronize(cs);
    if (e == cudaSuccess) e = e2;
  }
  const cudaError_t e3 = cudaStreamSynchronize(s);  // the renders (and any fault) are done
  if (e == cudaSuccess) e = e3;
  for (int b = 0; b < 2; ++b) {
    if (buf[b]) cudaFreeAsync(buf[b], s);
    if (rendered[b]) cudaEventDestroy(rendered[b]);
    if (copied[b]) cudaEventDestroy(copied[b]);
  }
  if (cs) cudaStreamDestroy(cs);
  if (rs != FR_OK) return rs;
  return cuda_status(e);
}

#ifndef FR_COLORIZE_V2  // warp-contiguous stores (colorize_kernel2); 0 = the first kernel
#define FR_COLORIZE_V2 1
#endif
fr_status colorize(const uint16_t* counts, int64_t n_pixels, int32_t max_iter,
                   const fr_palette* pal, uint8_t* out_rgba, fr_stream stream) {
  if (n_pixels < 0 || max_iter < 1) return FR_ERR_INVALID_ARG;
  if (max_iter > 65535) return FR_ERR_UNSUPPORTED;
  if (!pal) return FR_ERR_INVALID_ARG;
  fr::Palette p;
  fr_status st = make_palette(pal, &p);
  if (st != FR_OK) return st;
  if (n_pixels == 0) return FR_OK;
  if (!counts || !out_rgba) return FR_ERR_INVALID_ARG;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const bool aligned = ((uintptr_t)counts % 16 == 0) && ((uintptr_t)out_rgba % 16 == 0);
  const int64_t work = aligned ? (n_pixels >> 3) : n_pixels;
  int64_t blocks = (work + fr::kThreads - 1) / fr::kThreads;
  // grid cap: 512 CTAs per SM of the warp-contiguous kernel (1.06e9 pixels: 8/64/256/512/
  // 1024 -> 0.83/0.96/0.995/1.00/0.93 of the HBM copy peak, profiles/r02/ab_colorize.txt;
  // the old kernel at 8: 0.79); FRACTAL_COLORIZE_CTAS overrides (tests force grid strides)
  static const int ctas_env = env_int("FRACTAL_COLORIZE_CTAS", 0);
  const int64_t cap = (int64_t)sms * (ctas_env > 0 ? ctas_env : (FR_COLORIZE_V2 ? 512 : 8));
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  uint32_t* o = reinterpret_cast<uint32_t*>(out_rgba);
  if (aligned && FR_COLORIZE_V2)
    fr::colorize_kernel2<<<(unsigned)blocks, fr::kThreads, 0, stream>>>(counts, n_pixels,
                                                                         max_iter, p, o);
  else if (aligned)
    fr::colorize_kernel<<<(unsigned)blocks, fr::kThreads, 0, stream>>>(counts, n_pixels,
                                                                        max_iter, p, o);
  else
    fr::colorize_scalar_kernel<<<(unsigned)blocks, fr::kThreads, 0, stream>>>(
        counts, n_pixels, max_iter, p, o);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

fr_status fr_cardioid_path(double t0, double a0, double dt, double da_per_rev, double a_floor,
                           int32_t n, fr_complex* out_host) {
  if (n < 0) return FR_ERR_INVALID_ARG;
  if (!(is_fin(t0) && is_fin(a0) && is_fin(dt) && is_fin(da_per_rev) && is_fin(a_floor)))
    return FR_ERR_INVALID_ARG;
  if (!(a0 > 0.0) || !(a_floor > 0.0) || dt < 0.0 || da_per_rev < 0.0) return FR_ERR_INVALID_ARG;
  if (n == 0) return FR_OK;
  if (!out_host) return FR_ERR_INVALID_ARG;
  const double two_pi = 6.283185307179586476925286766559;
  double t = t0, a = a0;
  for (int32_t k = 0; k < n; ++k) {
    const double re = (2.0 * std::cos(t) - std::cos(2.0 * t)) / a;
    const double im = (2.0 * std::sin(t) - std::sin(2.0 * t)) / a;
    out_host[k].re = re;
    out_host[k].im = im;
    t = t - dt;
    if (t <= -two_pi) {
      t += two_pi;
      a = a - da_per_rev > a_floor ? a - da_per_rev : a_floor;
    }
  }
  return FR_OK;
}

int64_t fr_band_local_rows(int32_t height, fr_bands bands) {
  if (height < 1) return -1;
  return local_rows(height, bands);
}

int64_t fr_band_global_row(int32_t height, fr_bands b, int64_t local_row) {
  const int64_t rows = fr_band_local_rows(height, b);
  if (rows < 0 || local_row < 0 || local_row >= rows) return -1;
  if (b.band_rows == 0) return local_row;
  const int64_t band = local_row / b.band_rows;
  const int64_t w = local_row - band * b.band_rows;
  return (band * b.n_ranks + b.rank) * b.band_rows + w;
}

const char* fr_status_str(fr_status s) {
  switch (s) {
    case FR_OK: return "FR_OK";
    case FR_ERR_INVALID_ARG: return "FR_ERR_INVALID_ARG: invalid argument";
    case FR_ERR_TOO_LARGE: return "FR_ERR_TOO_LARGE: frame exceeds 2^31 pixels";
    case FR_ERR_UNSUPPORTED: return "FR_ERR_UNSUPPORTED: unsupported mode or max_iter > 65535";
    case FR_ERR_CUDA: return "FR_ERR_CUDA: CUDA launch or copy failed";
  }
  return "FR_ERR_UNKNOWN";
}

int32_t fr_last_cuda_error(void) { return g_last_cuda_error; }

fr_status fr_debug_refill_trace(void* trace_dev) {
  unsigned long long* p = static_cast<unsigned long long*>(trace_dev);
  return cuda_status(cudaMemcpyToSymbol(fr::g_refill_trace, &p, sizeof(p)));
}

uint64_t fr_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char* fr_version(void) { return "libfractal 0.1 (sm_100a)"; }

}  // extern "C"
