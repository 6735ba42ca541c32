// escape_kernels.cuh -- sm_100a device code for the escape-time hot path.
//
// Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, "reading c-k" = DESIGN.md
// §Readings.  Nothing here is shared with oracle/ (which is plain C, test-only).
//
// Kernels (DESIGN.md §5 has the dispatch table and the measurements):
//   escape_tile_kernel    S   static tiles; frame groups of a C-path, two frames per lane
//   escape_tile2_kernel   S2  one fp32 frame, two pixels per thread
//   escape_budget_kernel  P1  heavy-tailed frames: static pass up to a budget (fp32 fast:
//                             packed amortised sub-blocks), survivors appended to a queue
//   escape_cont_kernel    P2  persistent lane refill over P1's survivors; fast modes with
//                             |C| <= 1.989 amortise the escape test (block-end test,
//                             checkpointed sub-blocks, exact replay of one sub-block)
//   escape_refill_kernel  R / A  persistent lane refill over pixel chunks; A amortises
//                             the escape test (block-end test + exact replay)
//   escape_pathx_kernel   SX  C-path frames, FP32_FAST: two x-adjacent pixels per lane
//                             (packed FFMA2 loop), whole-sector count stores; the
//                             frame-independent first iteration hoisted (sx_pre), the
//                             uint16 frame loop as one PTX block (sx_frames_u16)
//   escape_cont2s_kernel  P2S experimental packed P2 (two orbits per lane, stashes, batched
//                             in-warp replay; off by default)
//   colorize_kernel           count -> RGBA colour levels (HBM-bound)
// All iteration goes through Iter<T, STRICT>::step / core, the packed fast_core2 and the
// PTX vote loops, which implement the same operation sequences (FAST: doubled state,
// FMA-contracted -- packed FFMA2 halves are separately rounded fused ops; STRICT:
// reading c-9's sequence, scalar), so counts do not depend on the kernel.
#pragma once
#include <cstdint>
#include <type_traits>
#include <cuda_runtime.h>

#ifndef FR_P2A_KS  // amortised P2: iterations per checkpointed sub-block
#define FR_P2A_KS 8
#endif

namespace fr {

constexpr int kThreads = 256;      // 8 warps per CTA
constexpr int kTileW = 32;         // CTA tile: 32 x 8 pixels, one pixel per thread
constexpr int kTileH = 8;
constexpr int kWarpW = 8;          // warp tile: 8 x 4 pixels (2-D for orbit coherence)
constexpr int kWarpH = 4;
constexpr int kMaxPathChunk = 1024;  // C values per launch, carried in kernel params
constexpr unsigned kFull = 0xffffffffu;

// Programmatic dependent launch (sm_90+): a kernel launched with the PDL attribute may
// start while the previous kernel of its stream is still finishing.  pdl_trigger() lets
// the NEXT kernel's CTAs start launching; pdl_wait() blocks until the previous kernel
// has completed and its memory is visible -- every kernel that uses them calls
// pdl_wait() before its first global-memory access other than its parameters, so the
// overlap covers only work that touches nothing the previous kernel writes.  Both are
// no-ops when the kernel was launched without the attribute.
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }


// ----------------------------------------------------------------------------------
// Parameters (passed by value; the path chunk's C values ride in param space).
// ----------------------------------------------------------------------------------
// Colours are RGBA bytes packed in 32-bit words (R in the low byte: the byte order of
// an RGBA image in memory), so a colour moves and selects as one register.
struct Palette {
  uint32_t e[256];
  uint32_t interior;
  uint32_t n;      // entries, 2..256
  uint32_t magic;  // ceil(2^32 / n): count mod n = c - n * umulhi(c, magic) for c < 2^16
  const uint32_t* dev;  // the n entries in device memory (short-lived CTAs read it through
                        // L1 instead of staging e[] in shared memory behind a CTA barrier)
};

struct Geom {
  double cx, cy;  // window centre
  double hx, hy;  // half_w / W, half_h / H (rounded once on the host, reading c-3)
  int W, H;       // full-frame size
  int rows;       // rows held by this call (bands) -- output has rows x W per frame
  int band_rows, n_ranks, rank;  // cyclic bands (band_rows == 0: rows == H, identity)
  int max_iter;
  int tiles_x;    // ceil(W / kTileW)
  int64_t frame_stride;  // rows * W
  uint16_t* counts;
  uint8_t* counts8;  // uint8 counts instead (max_iter <= 255; static kernel only), else null
  uint32_t* rgba;  // packed RGBA words; nullptr unless colour levels are fused
  int grid2d;     // kernels S/S2: tiles on grid x/y (frame groups on z), else tiles on x
};

// Tile (and frame group) of this CTA for kernels S/S2.  With grid2d the launch is
// (tiles_x, tiles_y, groups) and no division is needed; otherwise (tiles_y > 65535)
// tiles are linear on x and groups on y.
__device__ __forceinline__ void tile_of(const Geom& g, int& tx, int& ty, int& grp) {
  if (g.grid2d) {
    tx = blockIdx.x;
    ty = blockIdx.y;
    grp = blockIdx.z;
  } else {
    ty = blockIdx.x / g.tiles_x;
    tx = blockIdx.x - ty * g.tiles_x;
    grp = blockIdx.y;
  }
}

// Julia C values of a path chunk, already in the kernel's state representation
// (rounded once to T on the host; doubled in FAST modes -- exact), so the kernel does no
// per-frame conversion.
template <class T, int NC>
struct CList {
  T re[NC];
  T im[NC];
};

// ----------------------------------------------------------------------------------
// Region-covering map, reading c-3: pixel centres, row 0 at the top, binary64
// with each operation separately rounded (explicit _rn intrinsics: no contraction).
// ----------------------------------------------------------------------------------
// The integer k = 2 px + 1 - W (H - 1 - 2 gy) is formed directly in binary64: every
// operand and every intermediate is an integer below 2^33, so the doubling and the
// addition are exact and k is the same double as the integer computed in 64 bits and
// converted (a shorter dependency chain in the kernels' prologue than 64-bit integer
// arithmetic; no fused operation, so the strict kernels' no-FMA guard still holds).
__device__ __forceinline__ double pixel_re(const Geom& g, int px) {
  const double k = __dadd_rn(__dmul_rn(2.0, (double)px), (double)(1 - g.W));
  return __dadd_rn(g.cx, __dmul_rn(k, g.hx));
}
__device__ __forceinline__ double pixel_im(const Geom& g, int gy) {
  const double k = __dadd_rn((double)(g.H - 1), __dmul_rn(-2.0, (double)gy));
  return __dadd_rn(g.cy, __dmul_rn(k, g.hy));
}

// Local output row -> global frame row under cyclic bands.
__device__ __forceinline__ int global_row(const Geom& g, int ly) {
  if (g.band_rows == 0) return ly;
  const int b = ly / g.band_rows;
  const int w = ly - b * g.band_rows;
  return (b * g.n_ranks + g.rank) * g.band_rows + w;
}

// ----------------------------------------------------------------------------------
// Sticky "alive" predicate + predicated count increment, one FSETP/DSETP and one
// predicated IADD per iteration (the SASS is FSETP.LE.AND P, PT, m, lim, P and
// @P IADD3).  cnt ends as the number of leading iterations n with |Z_n|^2 <= 4,
// which is the escape count when the loop ran >= max_iter iterations (clamped).
// ----------------------------------------------------------------------------------
__device__ __forceinline__ void alive_step_f32(unsigned& alive, int& cnt, float m, float lim) {
  asm("{\n\t.reg .pred pa, pb;\n\t"
      "setp.ne.u32 pa, %1, 0;\n\t"
      "setp.le.and.f32 pb, %2, %3, pa;\n\t"
      "selp.u32 %1, 1, 0, pb;\n\t"
      "@pb add.s32 %0, %0, 1;\n\t}"
      : "+r"(cnt), "+r"(alive)
      : "f"(m), "f"(lim));
}
__device__ __forceinline__ void alive_step_f64(unsigned& alive, int& cnt, double m, double lim) {
  asm("{\n\t.reg .pred pa, pb;\n\t"
      "setp.ne.u32 pa, %1, 0;\n\t"
      "setp.le.and.f64 pb, %2, %3, pa;\n\t"
      "selp.u32 %1, 1, 0, pb;\n\t"
      "@pb add.s32 %0, %0, 1;\n\t}"
      : "+r"(cnt), "+r"(alive)
      : "d"(m), "d"(lim));
}

// ----------------------------------------------------------------------------------
// One iteration Z <- Z^2 + C with the escape test on Z (before the update).
//
// STRICT (reading c-9): exactly the oracle's sequence
//   xx = x*x; yy = y*y; m = xx + yy; [m > 4 ?]; xy = x*y; x = (xx - yy) + cr;
//   y = (xy + xy) + ci
// with every op separately rounded (_rn intrinsics forbid contraction).
//
// FAST: state rescaled by 2, X = 2x, Y = 2y, with
// CR2 = 2cr, CI2 = 2ci, so that
//   Y' = 2(2xy + ci) = X*Y + CI2                 (one FFMA)
//   X' = 2(x^2 - y^2 + cr) = (X^2 - Y^2)/2 + CR2 (FMUL, FFMA, FFMA-by-0.5)
//   |Z|^2 > 4  <=>  X^2 + Y^2 > 16               (one FFMA)
// i.e. 5 FP-pipe instructions per iteration instead of 6 unscaled.
// ----------------------------------------------------------------------------------
template <class T, bool STRICT>
struct Iter;

template <>
struct Iter<float, true> {
  static constexpr float kLim = 4.0f;
  __device__ __forceinline__ static float mag(float x, float y) {
    return __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));
  }
  __device__ __forceinline__ static void core(float& x, float& y, float cr, float ci) {
    const float xx = __fmul_rn(x, x);
    const float yy = __fmul_rn(y, y);
    const float xy = __fmul_rn(x, y);
    const float t = __fsub_rn(xx, yy);
    const float s = __fadd_rn(xy, xy);
    x = __fadd_rn(t, cr);
    y = __fadd_rn(s, ci);
  }
  __device__ __forceinline__ static void step(float& x, float& y, float cr, float ci,
                                              unsigned& alive, int& cnt) {
    const float xx = __fmul_rn(x, x);
    const float yy = __fmul_rn(y, y);
    const float m = __fadd_rn(xx, yy);
    alive_step_f32(alive, cnt, m, kLim);
    const float xy = __fmul_rn(x, y);
    const float t = __fsub_rn(xx, yy);
    const float s = __fadd_rn(xy, xy);
    x = __fadd_rn(t, cr);
    y = __fadd_rn(s, ci);
  }
};

template <>
struct Iter<float, false> {
  static constexpr float kLim = 16.0f;
  __device__ __forceinline__ static float mag(float X, float Y) {
    return __fmaf_rn(X, X, __fmul_rn(Y, Y));
  }
  __device__ __forceinline__ static void core(float& X, float& Y, float CR2, float CI2) {
    const float YY = __fmul_rn(Y, Y);
    const float Tm = __fmaf_rn(X, X, -YY);
    const float Yn = __fmaf_rn(X, Y, CI2);
    X = __fmaf_rn(Tm, 0.5f, CR2);
    Y = Yn;
  }
  __device__ __forceinline__ static void step(float& X, float& Y, float CR2, float CI2,
                                              unsigned& alive, int& cnt) {
    const float YY = __fmul_rn(Y, Y);
    const float M = __fmaf_rn(X, X, YY);
    alive_step_f32(alive, cnt, M, kLim);
    const float Tm = __fmaf_rn(X, X, -YY);
    const float Yn = __fmaf_rn(X, Y, CI2);
    X = __fmaf_rn(Tm, 0.5f, CR2);
    Y = Yn;
  }
};

template <>
struct Iter<double, true> {
  static constexpr double kLim = 4.0;
  __device__ __forceinline__ static double mag(double x, double y) {
    return __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
  }
  __device__ __forceinline__ static void core(double& x, double& y, double cr, double ci) {
    const double xx = __dmul_rn(x, x);
    const double yy = __dmul_rn(y, y);
    const double xy = __dmul_rn(x, y);
    const double t = __dsub_rn(xx, yy);
    const double s = __dadd_rn(xy, xy);
    x = __dadd_rn(t, cr);
    y = __dadd_rn(s, ci);
  }
  __device__ __forceinline__ static void step(double& x, double& y, double cr, double ci,
                                              unsigned& alive, int& cnt) {
    const double xx = __dmul_rn(x, x);
    const double yy = __dmul_rn(y, y);
    const double m = __dadd_rn(xx, yy);
    alive_step_f64(alive, cnt, m, kLim);
    const double xy = __dmul_rn(x, y);
    const double t = __dsub_rn(xx, yy);
    const double s = __dadd_rn(xy, xy);
    x = __dadd_rn(t, cr);
    y = __dadd_rn(s, ci);
  }
};

template <>
struct Iter<double, false> {
  static constexpr double kLim = 16.0;
  __device__ __forceinline__ static double mag(double X, double Y) {
    return __fma_rn(X, X, __dmul_rn(Y, Y));
  }
  __device__ __forceinline__ static void core(double& X, double& Y, double CR2, double CI2) {
    const double YY = __dmul_rn(Y, Y);
    const double Tm = __fma_rn(X, X, -YY);
    const double Yn = __fma_rn(X, Y, CI2);
    X = __fma_rn(Tm, 0.5, CR2);
    Y = Yn;
  }
  __device__ __forceinline__ static void step(double& X, double& Y, double CR2, double CI2,
                                              unsigned& alive, int& cnt) {
    const double YY = __dmul_rn(Y, Y);
    const double M = __fma_rn(X, X, YY);
    alive_step_f64(alive, cnt, M, kLim);
    const double Tm = __fma_rn(X, X, -YY);
    const double Yn = __fma_rn(X, Y, CI2);
    X = __fma_rn(Tm, 0.5, CR2);
    Y = Yn;
  }
};

// Packed-float helpers (sm_100 FFMA2 / FMUL2: two separately rounded operations).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fneg2(float2 a) { return make_float2(-a.x, -a.y); }
// One FAST step on both halves (the doubled FMA sequence of Iter<float, false>::core).
__device__ __forceinline__ void fast_core2(float2& X, float2& Y, const float2 CR, const float2 CI) {
  const float2 YY = fmul2(Y, Y);
  const float2 T = ffma2(X, X, fneg2(YY));
  const float2 Yn = ffma2(X, Y, CI);
  X = ffma2(T, make_float2(0.5f, 0.5f), CR);
  Y = Yn;
}
__device__ __forceinline__ float2 fast_mag2(const float2 X, const float2 Y) {
  return ffma2(X, X, fmul2(Y, Y));
}

// NEXT-3 iteration maps (Figure 4, reading c-14), strict op sequence in
// both modes, identical to the oracle's: w = z^2 = (xx - yy, xy + xy); z^4 = w^2;
// rational term q = (w + 1)/(w - 1) = ((a c + b d) + i (b c - a d))/(c^2 + d^2) with
// a = wx + 1, c = wx - 1, b = d = wy; pole (c^2 + d^2 == 0) -> Z_{n+1} = +inf.
template <class T>
struct Ops;
template <>
struct Ops<float> {
  __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static float div(float a, float b) { return __fdiv_rn(a, b); }
  __device__ __forceinline__ static void alive(unsigned& al, int& cnt, float m) {
    alive_step_f32(al, cnt, m, 4.0f);
  }
  __device__ __forceinline__ static float inf() { return __int_as_float(0x7f800000); }
};
template <>
struct Ops<double> {
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
  __device__ __forceinline__ static void alive(unsigned& al, int& cnt, double m) {
    alive_step_f64(al, cnt, m, 4.0);
  }
  __device__ __forceinline__ static double inf() { return __longlong_as_double(0x7ff0000000000000ll); }
};

#ifndef FR_FN_FREEZE
#define FR_FN_FREEZE 1
#endif
template <class T, int FN>
struct FnIter {
  __device__ __forceinline__ static void step(T& x, T& y, T cr, T ci, unsigned& alive, int& cnt) {
    using O = Ops<T>;
    const T xx = O::mul(x, x);
    const T yy = O::mul(y, y);
    O::alive(alive, cnt, O::add(xx, yy));
    // the rational map: an escaped lane stops here -- its count is final, and its orbit
    // would run to inf / NaN within a few iterations, where every IEEE division of the
    // warp takes the slow path (FR_FN_FREEZE=0 keeps iterating, for the A/B)
    if (FN == 2 && FR_FN_FREEZE && !alive) return;
    const T xy = O::mul(x, y);
    const T wx = O::sub(xx, yy);
    const T wy = O::add(xy, xy);
    const T u = O::mul(wx, wx);
    const T v = O::mul(wy, wy);
    const T pp = O::mul(wx, wy);
    T fx = O::sub(u, v);
    T fy = O::add(pp, pp);
    if (FN == 2) {
      const T a = O::add(wx, T(1));
      const T c = O::sub(wx, T(1));
      const T den = O::add(O::mul(c, c), O::mul(wy, wy));
      if (den == T(0)) {
        x = O::inf();
        y = T(0);
        return;
      }
      const T qx = O::div(O::add(O::mul(a, c), O::mul(wy, wy)), den);
      const T qy = O::div(O::sub(O::mul(wy, c), O::mul(a, wy)), den);
      fx = O::add(fx, qx);
      fy = O::add(fy, qy);
    }
    x = O::add(fx, cr);
    y = O::add(fy, ci);
  }
};

// Initial state for a pixel: STRICT keeps (x, y, cr, ci); FAST keeps the doubled
// values (exact scaling by 2).  For binary32 the binary64 map value and C are rounded
// once to nearest (reading c-8).
template <class T, bool STRICT>
__device__ __forceinline__ T to_state(double v) {
  const T t = (T)v;  // cvt.rn
  return STRICT ? t : t + t;
}

// Count -> colour level: interior if count == max_iter, else
// palette[count mod n].
__device__ __forceinline__ uint32_t colour_of(const uint32_t* spal, const Palette& p, int cnt,
                                              int max_iter) {
  if (cnt == max_iter) return p.interior;
  const unsigned c = (unsigned)cnt;
  const unsigned q = __umulhi(c, p.magic);
  return spal[c - q * p.n];
}

// What the kernels that read colours from the device copy need of a palette (S2, SX,
// P1, P2S): 24 bytes of kernel parameters instead of the 1.1-KB Palette (the launch
// copies every parameter byte; it matters for small frames).
struct PalRef {
  const uint32_t* dev;
  uint32_t interior;
  uint32_t n;
  uint32_t magic;
};

// The same colour level from the device copy of the palette (read-only path).
__device__ __forceinline__ uint32_t colour_dev(const PalRef& p, int cnt, int max_iter) {
  if (cnt == max_iter) return p.interior;
  const unsigned c = (unsigned)cnt;
  const unsigned q = __umulhi(c, p.magic);
  return __ldg(p.dev + (c - q * p.n));
}

// ----------------------------------------------------------------------------------
// Whole vote loop of the FAST fp32 iteration in one PTX block: the sticky alive
// predicate stays a predicate across blocks (no predicate<->register round trip), and
// the loop test is one vote + one compare.  Runs blocks of K iterations while any lane
// of the warp is alive and fewer than `kfull` (a multiple of K) iterations have run.
// Returns the number of iterations run (warp-uniform); cnt / alive updated per lane.
// ----------------------------------------------------------------------------------
#define FR_FAST_STEP                                 \
  "mul.rn.f32 yy, %1, %1;\n\t"                       \
  "fma.rn.f32 m, %0, %0, yy;\n\t"                    \
  "setp.le.and.f32 pa, m, 0f41800000, pa;\n\t"       \
  "@pa add.s32 %2, %2, 1;\n\t"                       \
  "neg.f32 yy, yy;\n\t"                              \
  "fma.rn.f32 t, %0, %0, yy;\n\t"                    \
  "fma.rn.f32 %1, %0, %1, %7;\n\t"                   \
  "fma.rn.f32 %0, t, 0f3F000000, %6;\n\t"

template <int K>
__device__ __forceinline__ int fast_vote_loop_f32(float& x, float& y, int& cnt, unsigned& alive,
                                                  float cr2, float ci2, int kfull);

template <>
__device__ __forceinline__ int fast_vote_loop_f32<2>(float& x, float& y, int& cnt,
                                                     unsigned& alive, float cr2, float ci2,
                                                     int kfull) {
  int n;
  asm volatile(
      "{\n\t.reg .pred pa, pm;\n\t.reg .f32 yy, m, t;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\tmov.u32 %4, 0;\n\t"
      "setp.gt.s32 pm, %5, 0;\n\t@!pm bra FR_K2_DONE;\n"
      "FR_K2_LOOP:\n\t" FR_FAST_STEP FR_FAST_STEP
      "add.s32 %4, %4, 2;\n\t"
      "vote.sync.any.pred pm, pa, 0xffffffff;\n\t"
      "setp.lt.and.s32 pm, %4, %5, pm;\n\t"
      "@pm bra FR_K2_LOOP;\n"
      "FR_K2_DONE:\n\t"
      "selp.u32 %3, 1, 0, pa;\n\t}"
      : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n)
      : "r"(kfull), "f"(cr2), "f"(ci2));
  return n;
}

template <>
__device__ __forceinline__ int fast_vote_loop_f32<4>(float& x, float& y, int& cnt,
                                                     unsigned& alive, float cr2, float ci2,
                                                     int kfull) {
  int n;
  asm volatile(
      "{\n\t.reg .pred pa, pm;\n\t.reg .f32 yy, m, t;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\tmov.u32 %4, 0;\n\t"
      "setp.gt.s32 pm, %5, 0;\n\t@!pm bra FR_K4_DONE;\n"
      "FR_K4_LOOP:\n\t" FR_FAST_STEP FR_FAST_STEP FR_FAST_STEP FR_FAST_STEP
      "add.s32 %4, %4, 4;\n\t"
      "vote.sync.any.pred pm, pa, 0xffffffff;\n\t"
      "setp.lt.and.s32 pm, %4, %5, pm;\n\t"
      "@pm bra FR_K4_LOOP;\n"
      "FR_K4_DONE:\n\t"
      "selp.u32 %3, 1, 0, pa;\n\t}"
      : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n)
      : "r"(kfull), "f"(cr2), "f"(ci2));
  return n;
}
#undef FR_FAST_STEP

// Two independent orbits per lane (same pixel, two frames of a path): instruction-level
// parallelism for the FP pipe and one vote per block for both.
#define FR_FAST_STEP2                                \
  "mul.rn.f32 yy, %1, %1;\n\t"                       \
  "mul.rn.f32 yy2, %6, %6;\n\t"                      \
  "fma.rn.f32 m, %0, %0, yy;\n\t"                    \
  "fma.rn.f32 m2, %5, %5, yy2;\n\t"                  \
  "setp.le.and.f32 pa, m, 0f41800000, pa;\n\t"       \
  "setp.le.and.f32 pb, m2, 0f41800000, pb;\n\t"      \
  "@pa add.s32 %2, %2, 1;\n\t"                       \
  "@pb add.s32 %7, %7, 1;\n\t"                       \
  "neg.f32 yy, yy;\n\t"                              \
  "neg.f32 yy2, yy2;\n\t"                            \
  "fma.rn.f32 t, %0, %0, yy;\n\t"                    \
  "fma.rn.f32 t2, %5, %5, yy2;\n\t"                  \
  "fma.rn.f32 %1, %0, %1, %13;\n\t"                  \
  "fma.rn.f32 %6, %5, %6, %15;\n\t"                  \
  "fma.rn.f32 %0, t, 0f3F000000, %12;\n\t"           \
  "fma.rn.f32 %5, t2, 0f3F000000, %14;\n\t"

// Packed form (sm_100 FFMA2 / FMUL2): the two orbits are the two halves of 64-bit
// register pairs X = (x, x2), Y = (y, y2), CR = (cr, crb), CI = (ci, cib); one packed
// instruction runs the same correctly rounded fused operation on both halves, so the
// counts are bit-identical to the scalar loop.  The packed FP instructions keep the FMA
// pipe busy two cycles each while the escape tests (FSETP) and predicated count
// increments issue in between: 5 packed + 4 scalar + 1/K vote issue slots per pair of
// pixel-iterations instead of 10 + 4 (microbenchmark: 1.33x, profiles/r02/).
// -YY is formed by unpack + neg + repack, which ptxas folds into an FFMA2 operand
// modifier (no instruction).
#define FR_FAST_STEP2X                               \
  "mul.rn.f32x2 yy, Y, Y;\n\t"                       \
  "fma.rn.f32x2 m, X, X, yy;\n\t"                    \
  "mov.b64 {m1, m2}, m;\n\t"                         \
  "setp.le.and.f32 pa, m1, 0f41800000, pa;\n\t"      \
  "setp.le.and.f32 pb, m2, 0f41800000, pb;\n\t"      \
  "@pa add.s32 %2, %2, 1;\n\t"                       \
  FR_COUNT_B                                         \
  "mov.b64 {n1, n2}, yy;\n\t"                        \
  "neg.f32 n1, n1;\n\t"                              \
  "neg.f32 n2, n2;\n\t"                              \
  "mov.b64 nyy, {n1, n2};\n\t"                       \
  "fma.rn.f32x2 t, X, X, nyy;\n\t"                   \
  "fma.rn.f32x2 Y, X, Y, CI;\n\t"                    \
  "fma.rn.f32x2 X, t, HALF, CR;\n\t"

#ifndef FR_FFMA2
#define FR_FFMA2 1  // 0: the scalar two-orbit loop (same-box A/B)
#endif
// FR_FCOUNT: the second orbit's count kept as a float and incremented with a predicated
// FADD, which issues to the FMA pipe, instead of an IADD on the ALU pipe -- the packed
// loop is ALU-bound, so this moves one instruction per iteration to
// the pipe with room.  Exact: counts <= 65535 < 2^24.
#ifndef FR_FCOUNT
#define FR_FCOUNT 0
#endif
#if FR_FCOUNT
#define FR_COUNT_B "@pb add.f32 cbf, cbf, 0f3F800000;\n\t"
#define FR_COUNT_B_DECL ".reg .f32 cbf;\n\tcvt.rn.f32.s32 cbf, %7;\n\t"
#define FR_COUNT_B_OUT "cvt.rzi.s32.f32 %7, cbf;\n\t"
#else
#define FR_COUNT_B "@pb add.s32 %7, %7, 1;\n\t"
#define FR_COUNT_B_DECL ""
#define FR_COUNT_B_OUT ""
#endif

template <int K>
__device__ __forceinline__ int fast_vote_loop2_f32(float& x, float& y, int& cnt, unsigned& alive,
                                                   float& x2, float& y2, int& cnt2,
                                                   unsigned& alive2, float cr2, float ci2,
                                                   float cr2b, float ci2b, int kfull);

template <int K>
__device__ __forceinline__ int fast_vote_loop2x_f32(float& x, float& y, int& cnt,
                                                    unsigned& alive, float& x2, float& y2,
                                                    int& cnt2, unsigned& alive2, float cr2,
                                                    float ci2, float cr2b, float ci2b,
                                                    int kfull) {
  static_assert(K == 1 || K == 2 || K == 4, "vote blocks of 1, 2 or 4");
  int n;
  if constexpr (K == 1) {
    asm volatile(
        "{\n\t.reg .pred pa, pb, pm;\n\t.reg .b64 X, Y, CR, CI, HALF, yy, m, nyy, t;\n\t"
        ".reg .f32 m1, m2, n1, n2;\n\t" FR_COUNT_B_DECL
        "mov.b64 X, {%0, %5};\n\tmov.b64 Y, {%1, %6};\n\t"
        "mov.b64 CR, {%12, %14};\n\tmov.b64 CI, {%13, %15};\n\t"
        "mov.b64 HALF, {0f3F000000, 0f3F000000};\n\t"
        "setp.ne.u32 pa, %3, 0;\n\tsetp.ne.u32 pb, %8, 0;\n\tmov.u32 %4, 0;\n\t"
        "setp.gt.s32 pm, %9, 0;\n\t@!pm bra FR_X1B_DONE;\n"
        "FR_X1B_LOOP:\n\t" FR_FAST_STEP2X
        "add.s32 %4, %4, 1;\n\t"
        "or.pred pm, pa, pb;\n\t"
        "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
        "setp.lt.and.s32 pm, %4, %9, pm;\n\t"
        "@pm bra FR_X1B_LOOP;\n"
        "FR_X1B_DONE:\n\t"
        "mov.b64 {%0, %5}, X;\n\tmov.b64 {%1, %6}, Y;\n\t"
        FR_COUNT_B_OUT "selp.u32 %3, 1, 0, pa;\n\tselp.u32 %8, 1, 0, pb;\n\t}"
        : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n), "+f"(x2), "+f"(y2), "+r"(cnt2),
          "+r"(alive2)
        : "r"(kfull), "r"(0), "r"(0), "f"(cr2), "f"(ci2), "f"(cr2b), "f"(ci2b));
  } else if constexpr (K == 4) {
    asm volatile(
        "{\n\t.reg .pred pa, pb, pm;\n\t.reg .b64 X, Y, CR, CI, HALF, yy, m, nyy, t;\n\t"
        ".reg .f32 m1, m2, n1, n2;\n\t" FR_COUNT_B_DECL
        "mov.b64 X, {%0, %5};\n\tmov.b64 Y, {%1, %6};\n\t"
        "mov.b64 CR, {%12, %14};\n\tmov.b64 CI, {%13, %15};\n\t"
        "mov.b64 HALF, {0f3F000000, 0f3F000000};\n\t"
        "setp.ne.u32 pa, %3, 0;\n\tsetp.ne.u32 pb, %8, 0;\n\tmov.u32 %4, 0;\n\t"
        "setp.gt.s32 pm, %9, 0;\n\t@!pm bra FR_X4B_DONE;\n"
        "FR_X4B_LOOP:\n\t" FR_FAST_STEP2X FR_FAST_STEP2X FR_FAST_STEP2X FR_FAST_STEP2X
        "add.s32 %4, %4, 4;\n\t"
        "or.pred pm, pa, pb;\n\t"
        "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
        "setp.lt.and.s32 pm, %4, %9, pm;\n\t"
        "@pm bra FR_X4B_LOOP;\n"
        "FR_X4B_DONE:\n\t"
        "mov.b64 {%0, %5}, X;\n\tmov.b64 {%1, %6}, Y;\n\t"
        FR_COUNT_B_OUT "selp.u32 %3, 1, 0, pa;\n\tselp.u32 %8, 1, 0, pb;\n\t}"
        : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n), "+f"(x2), "+f"(y2), "+r"(cnt2),
          "+r"(alive2)
        : "r"(kfull), "r"(0), "r"(0), "f"(cr2), "f"(ci2), "f"(cr2b), "f"(ci2b));
  } else {
    asm volatile(
        "{\n\t.reg .pred pa, pb, pm;\n\t.reg .b64 X, Y, CR, CI, HALF, yy, m, nyy, t;\n\t"
        ".reg .f32 m1, m2, n1, n2;\n\t" FR_COUNT_B_DECL
        "mov.b64 X, {%0, %5};\n\tmov.b64 Y, {%1, %6};\n\t"
        "mov.b64 CR, {%12, %14};\n\tmov.b64 CI, {%13, %15};\n\t"
        "mov.b64 HALF, {0f3F000000, 0f3F000000};\n\t"
        "setp.ne.u32 pa, %3, 0;\n\tsetp.ne.u32 pb, %8, 0;\n\tmov.u32 %4, 0;\n\t"
        "setp.gt.s32 pm, %9, 0;\n\t@!pm bra FR_X2B_DONE;\n"
        "FR_X2B_LOOP:\n\t" FR_FAST_STEP2X FR_FAST_STEP2X
        "add.s32 %4, %4, 2;\n\t"
        "or.pred pm, pa, pb;\n\t"
        "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
        "setp.lt.and.s32 pm, %4, %9, pm;\n\t"
        "@pm bra FR_X2B_LOOP;\n"
        "FR_X2B_DONE:\n\t"
        "mov.b64 {%0, %5}, X;\n\tmov.b64 {%1, %6}, Y;\n\t"
        FR_COUNT_B_OUT "selp.u32 %3, 1, 0, pa;\n\tselp.u32 %8, 1, 0, pb;\n\t}"
        : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n), "+f"(x2), "+f"(y2), "+r"(cnt2),
          "+r"(alive2)
        : "r"(kfull), "r"(0), "r"(0), "f"(cr2), "f"(ci2), "f"(cr2b), "f"(ci2b));
  }
  return n;
}
// Kernel SX's frame loop (§5.3c).  Every frame of a C-path starts its pixels from the
// same state (X0, Y0), so the first iteration's squares, its escape test and
// T0 = X0*X0 - Y0*Y0 do not depend on the frame: sx_pre computes them once per lane,
// and per frame only Y1 = fma(X0, Y0, CI) and X1 = fma(T0, 1/2, CR) remain of the first
// iteration; the second iteration follows, then the K = 2 vote loop is entered at its
// vote.  Same operations on the same values as fast_vote_loop2x_f32<2>: bit-identical.
struct SxPre {
  uint64_t X0, Y0, T0;  // packed pairs (x, x2), (y, y2), (t, t2) of the first iteration
  int c0, c1;           // counts after the first iteration (1 = passed its escape test)
};
__device__ __forceinline__ SxPre sx_pre(float re0, float re1, float im, bool in0, bool in1) {
  SxPre p;
  asm("{\n\t.reg .pred pa, pb;\n\t.reg .b64 yy, m, nyy;\n\t.reg .f32 m1, m2, n1, n2;\n\t"
      "mov.b64 %0, {%5, %6};\n\tmov.b64 %1, {%7, %7};\n\t"
      "mul.rn.f32x2 yy, %1, %1;\n\t"
      "fma.rn.f32x2 m, %0, %0, yy;\n\t"
      "mov.b64 {m1, m2}, m;\n\t"
      "setp.ne.u32 pa, %8, 0;\n\tsetp.ne.u32 pb, %9, 0;\n\t"
      "setp.le.and.f32 pa, m1, 0f41800000, pa;\n\t"
      "setp.le.and.f32 pb, m2, 0f41800000, pb;\n\t"
      "selp.u32 %3, 1, 0, pa;\n\tselp.u32 %4, 1, 0, pb;\n\t"
      "mov.b64 {n1, n2}, yy;\n\tneg.f32 n1, n1;\n\tneg.f32 n2, n2;\n\t"
      "mov.b64 nyy, {n1, n2};\n\t"
      "fma.rn.f32x2 %2, %0, %0, nyy;\n\t}"
      : "=l"(p.X0), "=l"(p.Y0), "=l"(p.T0), "=r"(p.c0), "=r"(p.c1)
      : "f"(re0), "f"(re1), "f"(im), "r"((unsigned)in0), "r"((unsigned)in1));
  return p;
}
#define FR_SX_STEP                                   \
  "mul.rn.f32x2 yy, Y, Y;\n\t"                       \
  "fma.rn.f32x2 m, X, X, yy;\n\t"                    \
  "mov.b64 {m1, m2}, m;\n\t"                         \
  "setp.le.and.f32 pa, m1, 0f41800000, pa;\n\t"      \
  "setp.le.and.f32 pb, m2, 0f41800000, pb;\n\t"      \
  "@pa add.s32 %0, %0, 1;\n\t"                       \
  "@pb add.s32 %1, %1, 1;\n\t"                       \
  "mov.b64 {n1, n2}, yy;\n\t"                        \
  "neg.f32 n1, n1;\n\t"                              \
  "neg.f32 n2, n2;\n\t"                              \
  "mov.b64 nyy, {n1, n2};\n\t"                       \
  "fma.rn.f32x2 t, X, X, nyy;\n\t"                   \
  "fma.rn.f32x2 Y, X, Y, CI;\n\t"                    \
  "fma.rn.f32x2 X, t, HALF, CR;\n\t"
// one frame: counts of the lane's two pixels for C = (cr, ci); kfull even and >= 2
__device__ __forceinline__ void sx_frame(const SxPre& p, float cr, float ci, int kfull,
                                         int& cnt, int& cnt2) {
  asm volatile(
      "{\n\t.reg .pred pa, pb, pm;\n\t.reg .b64 X, Y, CR, CI, HALF, yy, m, nyy, t;\n\t"
      ".reg .f32 m1, m2, n1, n2;\n\t.reg .s32 n;\n\t"
      "mov.b64 CR, {%5, %5};\n\tmov.b64 CI, {%6, %6};\n\t"
      "mov.b64 HALF, {0f3F000000, 0f3F000000};\n\t"
      "mov.u32 %0, %7;\n\tmov.u32 %1, %8;\n\t"
      "setp.ne.u32 pa, %7, 0;\n\tsetp.ne.u32 pb, %8, 0;\n\t"
      "fma.rn.f32x2 Y, %2, %3, CI;\n\t"
      "fma.rn.f32x2 X, %4, HALF, CR;\n\t" FR_SX_STEP
      "mov.u32 n, 2;\n\t"
      "bra.uni FR_SXF_CHECK;\n"
      "FR_SXF_LOOP:\n\t" FR_SX_STEP FR_SX_STEP
      "add.s32 n, n, 2;\n"
      "FR_SXF_CHECK:\n\t"
      "or.pred pm, pa, pb;\n\t"
      "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
      "setp.lt.and.s32 pm, n, %9, pm;\n\t"
      "@pm bra FR_SXF_LOOP;\n\t}"
      : "=r"(cnt), "=r"(cnt2)
      : "l"(p.X0), "l"(p.Y0), "l"(p.T0), "f"(cr), "f"(ci), "r"(p.c0), "r"(p.c1), "r"(kfull));
}
#define FR_SX_STEP_C                                 \
  "mul.rn.f32x2 yy, Y, Y;\n\t"                       \
  "fma.rn.f32x2 m, X, X, yy;\n\t"                    \
  "mov.b64 {m1, m2}, m;\n\t"                         \
  "setp.le.and.f32 pa, m1, 0f41800000, pa;\n\t"      \
  "setp.le.and.f32 pb, m2, 0f41800000, pb;\n\t"      \
  "@pa add.s32 %%c0, %%c0, 1;\n\t"                   \
  "@pb add.s32 %%c1, %%c1, 1;\n\t"                   \
  "mov.b64 {n1, n2}, yy;\n\t"                        \
  "neg.f32 n1, n1;\n\t"                              \
  "neg.f32 n2, n2;\n\t"                              \
  "mov.b64 nyy, {n1, n2};\n\t"                       \
  "fma.rn.f32x2 t, X, X, nyy;\n\t"                   \
  "fma.rn.f32x2 Y, X, Y, CI;\n\t"                    \
  "fma.rn.f32x2 X, t, HALF, CR;\n\t"
// The whole frame loop of kernel SX in one PTX block (uint16 counts, whole pairs, no
// colour): per frame one shared-memory load of C, the hoisted first iteration, the vote
// loop, one 4-byte store and the pointer bump.  cbase: shared-memory address of the
// group's (cr, ci) pairs; out: the lane's pair address in the group's first frame.
__device__ __forceinline__ void sx_frames_u16(const SxPre& p, uint32_t cbase, int nfr,
                                              uint32_t* out, int64_t stride_bytes, int kfull,
                                              bool in0) {
  asm volatile(
      "{\n\t.reg .pred pa, pb, pm, pin, pf;\n\t.reg .b64 X, Y, CR, CI, HALF, yy, m, nyy, t, P;\n\t"
      ".reg .f32 m1, m2, n1, n2, cr, ci;\n\t.reg .s32 n, %%c0, %%c1, f;\n\t.reg .u32 v, ca;\n\t"
      "mov.b64 HALF, {0f3F000000, 0f3F000000};\n\t"
      "setp.ne.u32 pin, %10, 0;\n\t"
      "mov.u64 P, %6;\n\tmov.u32 ca, %5;\n\tmov.u32 f, 0;\n"
      "FR_SXA_FRAME:\n\t"
      "ld.shared.v2.f32 {cr, ci}, [ca];\n\t"
      "mov.b64 CR, {cr, cr};\n\tmov.b64 CI, {ci, ci};\n\t"
      "mov.u32 %%c0, %3;\n\tmov.u32 %%c1, %4;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\tsetp.ne.u32 pb, %4, 0;\n\t"
      "fma.rn.f32x2 Y, %0, %1, CI;\n\t"
      "fma.rn.f32x2 X, %2, HALF, CR;\n\t" FR_SX_STEP_C
      "mov.u32 n, 2;\n\t"
      "bra.uni FR_SXA_CHECK;\n"
      "FR_SXA_LOOP:\n\t" FR_SX_STEP_C FR_SX_STEP_C
      "add.s32 n, n, 2;\n"
      "FR_SXA_CHECK:\n\t"
      "or.pred pm, pa, pb;\n\t"
      "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
      "setp.lt.and.s32 pm, n, %9, pm;\n\t"
      "@pm bra FR_SXA_LOOP;\n\t"
      "prmt.b32 v, %%c0, %%c1, 0x5410;\n\t"
      "@pin st.global.u32 [P], v;\n\t"
      "add.s64 P, P, %7;\n\t"
      "add.u32 ca, ca, 8;\n\t"
      "add.s32 f, f, 1;\n\t"
      "setp.lt.s32 pf, f, %8;\n\t"
      "@pf bra FR_SXA_FRAME;\n\t}"
      :
      : "l"(p.X0), "l"(p.Y0), "l"(p.T0), "r"(p.c0), "r"(p.c1), "r"(cbase), "l"(out),
        "l"(stride_bytes), "r"(nfr), "r"(kfull), "r"((unsigned)in0)
      : "memory");
}
#undef FR_SX_STEP_C
#undef FR_SX_STEP
#undef FR_FAST_STEP2X

template <>
__device__ __forceinline__ int fast_vote_loop2_f32<4>(float& x, float& y, int& cnt,
                                                      unsigned& alive, float& x2, float& y2,
                                                      int& cnt2, unsigned& alive2, float cr2,
                                                      float ci2, float cr2b, float ci2b,
                                                      int kfull) {
  int n;
  asm volatile(
      "{\n\t.reg .pred pa, pb, pm;\n\t.reg .f32 yy, m, t, yy2, m2, t2;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\tsetp.ne.u32 pb, %8, 0;\n\tmov.u32 %4, 0;\n\t"
      "setp.gt.s32 pm, %9, 0;\n\t@!pm bra FR_K4B_DONE;\n"
      "FR_K4B_LOOP:\n\t" FR_FAST_STEP2 FR_FAST_STEP2 FR_FAST_STEP2 FR_FAST_STEP2
      "add.s32 %4, %4, 4;\n\t"
      "or.pred pm, pa, pb;\n\t"
      "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
      "setp.lt.and.s32 pm, %4, %9, pm;\n\t"
      "@pm bra FR_K4B_LOOP;\n"
      "FR_K4B_DONE:\n\t"
      "selp.u32 %3, 1, 0, pa;\n\tselp.u32 %8, 1, 0, pb;\n\t}"
      : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n), "+f"(x2), "+f"(y2), "+r"(cnt2),
        "+r"(alive2)
      : "r"(kfull), "r"(0), "r"(0), "f"(cr2), "f"(ci2), "f"(cr2b), "f"(ci2b));
  return n;
}
template <>
__device__ __forceinline__ int fast_vote_loop2_f32<2>(float& x, float& y, int& cnt,
                                                      unsigned& alive, float& x2, float& y2,
                                                      int& cnt2, unsigned& alive2, float cr2,
                                                      float ci2, float cr2b, float ci2b,
                                                      int kfull) {
  int n;
  asm volatile(
      "{\n\t.reg .pred pa, pb, pm;\n\t.reg .f32 yy, m, t, yy2, m2, t2;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\tsetp.ne.u32 pb, %8, 0;\n\tmov.u32 %4, 0;\n\t"
      "setp.gt.s32 pm, %9, 0;\n\t@!pm bra FR_K2B_DONE;\n"
      "FR_K2B_LOOP:\n\t" FR_FAST_STEP2 FR_FAST_STEP2
      "add.s32 %4, %4, 2;\n\t"
      "or.pred pm, pa, pb;\n\t"
      "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
      "setp.lt.and.s32 pm, %4, %9, pm;\n\t"
      "@pm bra FR_K2B_LOOP;\n"
      "FR_K2B_DONE:\n\t"
      "selp.u32 %3, 1, 0, pa;\n\tselp.u32 %8, 1, 0, pb;\n\t}"
      : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n), "+f"(x2), "+f"(y2), "+r"(cnt2),
        "+r"(alive2)
      : "r"(kfull), "r"(0), "r"(0), "f"(cr2), "f"(ci2), "f"(cr2b), "f"(ci2b));
  return n;
}
// STRICT fp32, two orbits: the exact IEEE sequence of reading c-9 (every operation
// separately rounded, no contraction -- explicit .rn), same operand layout and vote loop
// as the fast version, so the sticky predicates stay predicates across blocks.
#define FR_STRICT_STEP2                              \
  "mul.rn.f32 xx, %0, %0;\n\t"                       \
  "mul.rn.f32 xx2, %5, %5;\n\t"                      \
  "mul.rn.f32 yy, %1, %1;\n\t"                       \
  "mul.rn.f32 yy2, %6, %6;\n\t"                      \
  "add.rn.f32 m, xx, yy;\n\t"                        \
  "add.rn.f32 m2, xx2, yy2;\n\t"                     \
  "setp.le.and.f32 pa, m, 0f40800000, pa;\n\t"       \
  "setp.le.and.f32 pb, m2, 0f40800000, pb;\n\t"      \
  "@pa add.s32 %2, %2, 1;\n\t"                       \
  "@pb add.s32 %7, %7, 1;\n\t"                       \
  "mul.rn.f32 xy, %0, %1;\n\t"                       \
  "mul.rn.f32 xy2, %5, %6;\n\t"                      \
  "sub.rn.f32 t, xx, yy;\n\t"                        \
  "sub.rn.f32 t2, xx2, yy2;\n\t"                     \
  "add.rn.f32 s, xy, xy;\n\t"                        \
  "add.rn.f32 s2, xy2, xy2;\n\t"                     \
  "add.rn.f32 %0, t, %12;\n\t"                       \
  "add.rn.f32 %5, t2, %14;\n\t"                      \
  "add.rn.f32 %1, s, %13;\n\t"                       \
  "add.rn.f32 %6, s2, %15;\n\t"

__device__ __forceinline__ int strict_vote_loop2_f32(float& x, float& y, int& cnt,
                                                     unsigned& alive, float& x2, float& y2,
                                                     int& cnt2, unsigned& alive2, float cr,
                                                     float ci, float crb, float cib, int kfull) {
  int n;
  asm volatile(
      "{\n\t.reg .pred pa, pb, pm;\n\t"
      ".reg .f32 xx, yy, m, xy, t, s, xx2, yy2, m2, xy2, t2, s2;\n\t"
      "setp.ne.u32 pa, %3, 0;\n\tsetp.ne.u32 pb, %8, 0;\n\tmov.u32 %4, 0;\n\t"
      "setp.gt.s32 pm, %9, 0;\n\t@!pm bra FR_S4B_DONE;\n"
      "FR_S4B_LOOP:\n\t" FR_STRICT_STEP2 FR_STRICT_STEP2 FR_STRICT_STEP2 FR_STRICT_STEP2
      "add.s32 %4, %4, 4;\n\t"
      "or.pred pm, pa, pb;\n\t"
      "vote.sync.any.pred pm, pm, 0xffffffff;\n\t"
      "setp.lt.and.s32 pm, %4, %9, pm;\n\t"
      "@pm bra FR_S4B_LOOP;\n"
      "FR_S4B_DONE:\n\t"
      "selp.u32 %3, 1, 0, pa;\n\tselp.u32 %8, 1, 0, pb;\n\t}"
      : "+f"(x), "+f"(y), "+r"(cnt), "+r"(alive), "=r"(n), "+f"(x2), "+f"(y2), "+r"(cnt2),
        "+r"(alive2)
      : "r"(kfull), "r"(0), "r"(0), "f"(cr), "f"(ci), "f"(crb), "f"(cib));
  return n;
}
#undef FR_STRICT_STEP2

// Two-orbit PTX vote loop of either fp32 mode (blocks of 4).
// KV: vote block of the fast loop (4, or 2 for the FRACTAL_VOTE_K=2 experiment; strict
// always 4); kfull must be a multiple of it
template <bool STRICT, int KV = 4>
__device__ __forceinline__ int vote_loop2_f32(float& x, float& y, int& cnt, unsigned& alive,
                                              float& x2, float& y2, int& cnt2, unsigned& alive2,
                                              float cr, float ci, float crb, float cib,
                                              int kfull) {
  if constexpr (STRICT)
    return strict_vote_loop2_f32(x, y, cnt, alive, x2, y2, cnt2, alive2, cr, ci, crb, cib, kfull);
  else
    return FR_FFMA2 ? fast_vote_loop2x_f32<KV>(x, y, cnt, alive, x2, y2, cnt2, alive2, cr, ci, crb,
                                               cib, kfull)
                    : fast_vote_loop2_f32<KV>(x, y, cnt, alive, x2, y2, cnt2, alive2, cr, ci, crb,
                                              cib, kfull);
}

#undef FR_FAST_STEP2

template <class T, bool STRICT, int K>
constexpr bool kAsmLoop = std::is_same<T, float>::value && !STRICT && (K == 2 || K == 4);
// two-orbit PTX loops: fp32, both modes (strict: the exact sequence), blocks of 4 (fast
// also 2)
template <class T, bool STRICT, int K>
constexpr bool kAsmPair = std::is_same<T, float>::value && (K == 4 || (!STRICT && K == 2));

// ----------------------------------------------------------------------------------
// Static-tile kernel (S): one pixel per thread, 8x4 warp tiles in a 32x8 CTA tile.  The
// CTA computes its tile's axis values once (32 re + 8 im, binary64 -> state type) into
// shared memory and then renders a GROUP of frames of the path chunk for that tile
// (frames [blockIdx.y * fpc, ...)), so the per-pixel map cost is amortised over the
// group.  Iteration runs in unrolled blocks of K with a warp-vote (__any_sync) exit; the
// count is exact per iteration (sticky alive predicate + predicated increment).
// MANDEL takes C from the pixel and Z_0 = 0.
// ----------------------------------------------------------------------------------
template <class T, bool STRICT, bool MANDEL, bool COLOR, int K, int NC, int FN = 0, int ES = 2>
__global__ void __launch_bounds__(kThreads)
escape_tile_kernel(const Geom g, const Palette pal, const CList<T, NC> cs, int frame0,
                   int n_frames, int fpc) {
  static_assert(FN == 0 || (STRICT && !MANDEL), "map variants: strict Julia frames");
  if constexpr (NC == 1) pdl_trigger();
  static_assert(ES == 1 || ES == 2, "counts are uint16 (ES 2) or uint8 (ES 1)");
  using CountT = typename std::conditional<ES == 2, uint16_t, uint8_t>::type;
  __shared__ uint32_t spal[COLOR ? 256 : 1];
  int tx, ty, grp;
  tile_of(g, tx, ty, grp);
  if (COLOR) {
    spal[threadIdx.x] = pal.e[threadIdx.x];
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int cx = (warp & 3) * kWarpW + (lane & 7);
  const int cy = (warp >> 2) * kWarpH + (lane >> 3);
  const int px = tx * kTileW + cx;
  const int ly = ty * kTileH + cy;
  const bool inside = (px < g.W) && (ly < g.rows);
  // this thread's pixel in the plane (binary64 map, one rounding to T); no CTA barrier:
  // the cost is amortised over the frame group
  const T are = to_state<T, STRICT>(pixel_re(g, min(px, g.W - 1)));
  const T aim = to_state<T, STRICT>(pixel_im(g, global_row(g, min(ly, g.rows - 1))));
  const int max_iter = g.max_iter;
  const int kfull = max_iter - max_iter % K;  // iterations run in whole K-blocks
  const int f0 = grp * fpc;
  const int f1 = min(f0 + fpc, n_frames);
  const int64_t stride = g.frame_stride;
  const int64_t pix0 = (int64_t)(frame0 + f0) * stride + (int64_t)ly * g.W + px;
  CountT* outp = (ES == 2 ? reinterpret_cast<CountT*>(g.counts)
                          : reinterpret_cast<CountT*>(g.counts8)) + pix0;
  uint32_t* outc = COLOR ? g.rgba + pix0 : nullptr;
  // Output sectors: with 8x4 warp tiles each 32-B sector of a count row is written half
  // by one warp and half by its neighbour, and over a frame group the two warps drift
  // apart in frames; a sector evicted from L2 half-written costs a DRAM read-modify-write
  // (measured: +0.4 GB reads per cfg4 launch).  FR_COUNT_STORE (compile time) picks the
  // count store: 1 (default) L2 evict_last policy, so a half-written line tends to stay
  // until its other half arrives; 2 stage the frame group in shared memory and write
  // whole 16-B row segments after a CTA barrier (path chunks); 0 plain stores.
  // DESIGN.md §5 has the measurements.
#ifndef FR_COUNT_STORE
#define FR_COUNT_STORE 1
#endif
  constexpr bool kStaged = FR_COUNT_STORE == 2 && NC > 1;
  constexpr int kStageFrames = 32;
  __shared__ __align__(16) CountT stage[kStaged ? kStageFrames * kThreads : 1];
  const bool staged = kStaged && (f1 - f0) <= kStageFrames;
  CountT* sp = stage + cy * kTileW + cx;
  uint64_t l2pol = 0;
  if (FR_COUNT_STORE == 1)
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(l2pol));
  auto put = [&](CountT* q, int v, int dk) {  // dk: frame offset of q from outp (0 or 1)
    if (kStaged && staged) {
      sp[dk * kThreads] = (CountT)v;
    } else if constexpr (FR_COUNT_STORE == 1 && ES == 2) {
      asm volatile("st.global.L2::cache_hint.u16 [%0], %1, %2;" ::"l"(q),
                   "h"((unsigned short)v), "l"(l2pol) : "memory");
    } else if constexpr (FR_COUNT_STORE == 1) {
      asm volatile("st.global.L2::cache_hint.u8 [%0], %1, %2;" ::"l"(q), "r"(v), "l"(l2pol)
                   : "memory");
    } else {
      *q = (CountT)v;
    }
  };

  int f = f0;
  if constexpr (FN == 0 && kAsmPair<T, STRICT, K> && !MANDEL && NC > 1) {
    // two frames per lane (ILP); the remaining odd frame goes through the loop below
    for (; f + 1 < f1; f += 2) {
      float x = are, y = aim, x2 = are, y2 = aim;
      unsigned alive = inside ? 1u : 0u, alive2 = alive;
      int cnt = 0, cnt2 = 0;
      // C values through a shuffle: they then live in per-thread registers, so the FFMA
      // X' = T * 0.5 + CR2 keeps 0.5 as an immediate (a uniform-register C forces ptxas
      // to rematerialise 0.5 with an extra ALU move every iteration: +18% instructions)
      int n;
      if constexpr (STRICT)
        n = strict_vote_loop2_f32(x, y, cnt, alive, x2, y2, cnt2, alive2,
                                  __shfl_sync(kFull, cs.re[f], lane),
                                  __shfl_sync(kFull, cs.im[f], lane),
                                  __shfl_sync(kFull, cs.re[f + 1], lane),
                                  __shfl_sync(kFull, cs.im[f + 1], lane), kfull);
      else
        n = vote_loop2_f32<false, K>(x, y, cnt, alive, x2, y2, cnt2, alive2,
                                     __shfl_sync(kFull, cs.re[f], lane),
                                     __shfl_sync(kFull, cs.im[f], lane),
                                     __shfl_sync(kFull, cs.re[f + 1], lane),
                                     __shfl_sync(kFull, cs.im[f + 1], lane), kfull);
      if (kfull != max_iter && n == kfull && __any_sync(kFull, alive | alive2)) {
        for (; n < max_iter; ++n) {
          Iter<T, STRICT>::step(x, y, cs.re[f], cs.im[f], alive, cnt);
          Iter<T, STRICT>::step(x2, y2, cs.re[f + 1], cs.im[f + 1], alive2, cnt2);
        }
      }
      if (inside) {
        // counts need no clamp: one increment at most per executed iteration, and the
        // loops execute exactly max_iter iterations at most
        const int c1 = cnt, c2 = cnt2;
        put(outp, c1, 0);
        put(outp + stride, c2, 1);
        if (COLOR) {
          outc[0] = colour_of(spal, pal, c1, max_iter);
          outc[stride] = colour_of(spal, pal, c2, max_iter);
        }
      }
      outp += 2 * stride;
      if (kStaged) sp += 2 * kThreads;
      if (COLOR) outc += 2 * stride;
    }
  }
  for (; f < f1; ++f) {
    T x, y, cr, ci;
    if (MANDEL) {
      x = T(0);
      y = T(0);
      cr = are;
      ci = aim;
    } else {
      x = are;
      y = aim;
      cr = cs.re[NC == 1 ? 0 : f];
      ci = cs.im[NC == 1 ? 0 : f];
    }
    unsigned alive = inside ? 1u : 0u;
    int cnt = 0;
    int n;
    using It = typename std::conditional<FN == 0, Iter<T, STRICT>, FnIter<T, FN>>::type;
    if constexpr (FN == 0 && kAsmLoop<T, STRICT, K>) {
      n = fast_vote_loop_f32<K>(x, y, cnt, alive, cr, ci, kfull);
    } else {
      n = 0;
      while (n < kfull) {
#pragma unroll
        for (int j = 0; j < K; ++j) It::step(x, y, cr, ci, alive, cnt);
        n += K;
        if (!__any_sync(kFull, alive)) break;
      }
    }
    if (kfull != max_iter && n == kfull && __any_sync(kFull, alive)) {
      for (; n < max_iter; ++n) It::step(x, y, cr, ci, alive, cnt);
    }
    if constexpr (NC == 1) pdl_wait();  // single frames are launched with PDL
    if (inside) {
      const int count = cnt;  // <= max_iter (see above)
      put(outp, count, 0);
      if (COLOR) *outc = colour_of(spal, pal, count, max_iter);
    }
    outp += stride;
    if (kStaged) sp += kThreads;
    if (COLOR) outc += stride;
  }
  if constexpr (kStaged) {
    if (staged) {
      // flush: thread = (row, 8-pixel group) segment, frames 8 apart; vector store when
      // the segment is whole and aligned in every frame, else per pixel in bounds
      __syncthreads();
      const int t = threadIdx.x, r = (t >> 2) & 7, col = (t & 3) * 8, fl0 = t >> 5;
      const int row = ty * kTileH + r, x0 = tx * kTileW + col;
      if (row < g.rows && x0 < g.W) {
        CountT* q = (ES == 2 ? reinterpret_cast<CountT*>(g.counts)
                             : reinterpret_cast<CountT*>(g.counts8)) +
                    ((int64_t)(frame0 + f0 + fl0) * stride + (int64_t)row * g.W + x0);
        const CountT* src = stage + fl0 * kThreads + r * kTileW + col;
        constexpr unsigned kVec = 8 * ES;  // bytes per segment
        const bool vec = x0 + 8 <= g.W && (reinterpret_cast<uintptr_t>(q) % kVec) == 0 &&
                         ((stride * ES) % kVec) == 0;
        for (int fl = fl0; fl < f1 - f0; fl += 8, q += 8 * stride, src += 8 * kThreads) {
          if (vec) {
            if constexpr (ES == 2) *reinterpret_cast<uint4*>(q) = *reinterpret_cast<const uint4*>(src);
            else *reinterpret_cast<uint2*>(q) = *reinterpret_cast<const uint2*>(src);
          } else {
            for (int i = 0; i < min(8, g.W - x0); ++i) q[i] = src[i];
          }
        }
      }
    }
  }
}

// ----------------------------------------------------------------------------------
// Kernel SX: C-path frames in FP32_FAST (Julia), two x-adjacent pixels per lane.  CTA tile
// 64 x 8 pixels, warp tile 16 x 4: lane l holds pixels (2 (l & 7), l >> 3) and
// (2 (l & 7) + 1, l >> 3) of its warp tile as the two halves of the packed FFMA2 vote
// loop, both with the frame's C.  A warp row is then 16 pixels = one whole 32-byte
// sector of uint16 counts, written by one 4-byte store per lane: no sector is shared
// between warps, so no partially written sector is ever evicted from L2 (with 8 x 4
// warp tiles every sector was split between two warps that drift apart over the frame
// group: +0.4 GB of DRAM read-modify-write per bench launch).
// The CTA renders a group of `fpc` frames of the path chunk for its tile (pixel map
// amortised over the group), one frame at a time.
// ----------------------------------------------------------------------------------
#ifndef FR_SX_WARPS  // warps per CTA of kernel SX (see kSxThreads below)
#define FR_SX_WARPS 4
#endif
constexpr int kSxWarpsX = FR_SX_WARPS < 4 ? FR_SX_WARPS : 4;  // warp tiles side by side
constexpr int kTileWX = 16 * kSxWarpsX;                          // CTA tile width
#ifndef FR_SX_UNROLL  // unroll the frame loop of kernel SX by 4 (A/B knob)
#define FR_SX_UNROLL 0
#endif
#ifndef FR_SX_K  // vote block of kernel SX (A/B knob)
#define FR_SX_K 2  // same box: 2.629 vs 2.734 ms per bench step (profiles/r02/ab_sx_votek.txt)
#endif
#ifndef FR_SX_PEEL  // first iteration hoisted out of the frame loop (A/B knob)
#define FR_SX_PEEL 1
#endif
#ifndef FR_SX_ASM  // the whole frame loop as one PTX block (uint16, no colour; A/B knob)
#define FR_SX_ASM 1
#endif
constexpr int kSxChunk = 128;  // frames per shared-memory C chunk
// VEC (host-checked): even width and frame stride, aligned outputs -- both pixels of a
// lane are in or out together and every pair store is aligned
// warps per CTA of kernel SX: 4 (CTA tile 64 x 4; bench 2.322 -> 2.293 ms against 8,
// profiles/r02/ab_sx_warps.txt), 8 (64 x 8) or 2 (32 x 4)
constexpr int kSxThreads = 32 * FR_SX_WARPS;
constexpr int kSxRows = 4 * (FR_SX_WARPS / kSxWarpsX);  // CTA tile rows
static_assert(FR_SX_WARPS == 8 || FR_SX_WARPS == 4 || FR_SX_WARPS == 2,
              "kernel SX: 2, 4 or 8 warps per CTA");
template <int NC, int ES, bool COLOR, bool VEC>
__global__ void __launch_bounds__(kSxThreads)
escape_pathx_kernel(const Geom g, const PalRef pal, const CList<float, NC> cs, int frame0,
                    int n_frames, int fpc) {
  using CountT = typename std::conditional<ES == 2, uint16_t, uint8_t>::type;
  int tx, ty, grp;
  tile_of(g, tx, ty, grp);  // g.tiles_x counts 64-pixel tiles here
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int px = tx * kTileWX + (warp % kSxWarpsX) * 16 + (lane & 7) * 2;
  const int ly = ty * kSxRows + (warp / kSxWarpsX) * 4 + (lane >> 3);
  const bool in0 = px < g.W && ly < g.rows;
  const bool in1 = px + 1 < g.W && ly < g.rows;
  const float re0 = to_state<float, false>(pixel_re(g, min(px, g.W - 1)));
  const float re1 = to_state<float, false>(pixel_re(g, min(px + 1, g.W - 1)));
  const float im = to_state<float, false>(pixel_im(g, global_row(g, min(ly, g.rows - 1))));
  const int max_iter = g.max_iter;
  const int kfull = max_iter - max_iter % FR_SX_K;
  const int f0 = grp * fpc;
  const int f1 = min(f0 + fpc, n_frames);
  const int64_t stride = g.frame_stride;
  const int64_t pix0 = (int64_t)(frame0 + f0) * stride + (int64_t)ly * g.W + px;
  CountT* outp = (ES == 2 ? reinterpret_cast<CountT*>(g.counts)
                          : reinterpret_cast<CountT*>(g.counts8)) + pix0;
  uint32_t* outc = COLOR ? g.rgba + pix0 : nullptr;
  // one store for both counts when the pair is whole and aligned in every frame
  const uintptr_t base_c = ES == 2 ? reinterpret_cast<uintptr_t>(g.counts)
                                   : reinterpret_cast<uintptr_t>(g.counts8);
  const bool vec = VEC || (in1 && ((g.W & 1) == 0) && ((stride & 1) == 0) &&
                           (base_c % (2 * ES)) == 0 &&
                           (!COLOR || (reinterpret_cast<uintptr_t>(g.rgba) & 7) == 0));
  // one frame; TAIL: max_iter is not a multiple of the vote block (hoisted out of the
  // frame loop: the per-frame checks of the tail cost instructions on every frame)
  const SxPre pre = sx_pre(re0, re1, im, in0, in1);
  auto frame = [&](const int f, auto tail_tag) {
    constexpr bool TAIL = decltype(tail_tag)::value == 1;
    constexpr bool PEEL = decltype(tail_tag)::value == 2;
    float x = re0, y = im, x2 = re1, y2 = im;
    unsigned alive = in0 ? 1u : 0u, alive2 = in1 ? 1u : 0u;
    int cnt = 0, cnt2 = 0;
    const float cr = cs.re[f], ci = cs.im[f];
    if constexpr (PEEL) {
      sx_frame(pre, cr, ci, kfull, cnt, cnt2);
    } else {
    int n = fast_vote_loop2x_f32<FR_SX_K>(x, y, cnt, alive, x2, y2, cnt2, alive2, cr, ci, cr,
                                          ci, kfull);
    if constexpr (TAIL) {
      if (n == kfull && __any_sync(kFull, alive | alive2)) {
        for (; n < max_iter; ++n) {
          Iter<float, false>::step(x, y, cr, ci, alive, cnt);
          Iter<float, false>::step(x2, y2, cr, ci, alive2, cnt2);
        }
      }
    } else {
      (void)n;
    }
    }
    if (VEC) {
      if (in0) {
        if constexpr (ES == 2)
          *reinterpret_cast<uint32_t*>(outp) = (uint32_t)cnt | ((uint32_t)cnt2 << 16);
        else
          *reinterpret_cast<uint16_t*>(outp) = (uint16_t)(cnt | (cnt2 << 8));
        if (COLOR) {
          *reinterpret_cast<uint2*>(outc) =
              make_uint2(colour_dev(pal, cnt, max_iter), colour_dev(pal, cnt2, max_iter));
        }
      }
    } else if (vec) {
      if constexpr (ES == 2)
        *reinterpret_cast<uint32_t*>(outp) = (uint32_t)cnt | ((uint32_t)cnt2 << 16);
      else
        *reinterpret_cast<uint16_t*>(outp) = (uint16_t)(cnt | (cnt2 << 8));
      if (COLOR) {
        *reinterpret_cast<uint2*>(outc) =
            make_uint2(colour_dev(pal, cnt, max_iter), colour_dev(pal, cnt2, max_iter));
      }
    } else {
      if (in0) {
        outp[0] = (CountT)cnt;
        if (COLOR) outc[0] = colour_dev(pal, cnt, max_iter);
      }
      if (in1) {
        outp[1] = (CountT)cnt2;
        if (COLOR) outc[1] = colour_dev(pal, cnt2, max_iter);
      }
    }
    outp += stride;
    if (COLOR) outc += stride;
  };
  if constexpr (FR_SX_ASM && ES == 2 && !COLOR && VEC) {
    if (FR_SX_PEEL && FR_SX_K == 2 && kfull == max_iter && kfull >= 2) {
      // the frame loop in one PTX block, C staged in shared memory per chunk of frames
      __shared__ float2 sc[kSxChunk];
      for (int c0 = f0; c0 < f1; c0 += kSxChunk) {
        const int nc = min(kSxChunk, f1 - c0);
        __syncthreads();
        for (int i = threadIdx.x; i < nc; i += kSxThreads) sc[i] = make_float2(cs.re[c0 + i], cs.im[c0 + i]);
        __syncthreads();
        sx_frames_u16(pre, static_cast<uint32_t>(__cvta_generic_to_shared(sc)), nc,
                      reinterpret_cast<uint32_t*>(outp), stride * 2, kfull, in0);
        outp += (int64_t)nc * stride;
      }
      return;
    }
  }
  if (FR_SX_PEEL && FR_SX_K == 2 && kfull == max_iter && kfull >= 2) {
#pragma unroll 1
    for (int f = f0; f < f1; ++f) frame(f, std::integral_constant<int, 2>{});
  } else if (kfull == max_iter) {
#if FR_SX_UNROLL
#pragma unroll 4
#else
#pragma unroll 1
#endif
    for (int f = f0; f < f1; ++f) frame(f, std::integral_constant<int, 0>{});
  } else {
#pragma unroll 1
    for (int f = f0; f < f1; ++f) frame(f, std::integral_constant<int, 1>{});
  }
}

// ----------------------------------------------------------------------------------
// Static-tile kernel for ONE frame, fp32 (fast or strict), two pixels per thread (S2): CTA tile
// 32x16, each thread iterates the pixels of rows ly and ly + 8 of its 8x4-lane warp
// tile together in the two-orbit PTX vote loop (ILP for the FP pipe, one vote for
// both, half the per-pixel overhead).  Julia frames share C; Mandelbrot maps take each
// orbit's C from its pixel (Z_0 = 0).  Bit-identical to kernel S (same arithmetic).
// ----------------------------------------------------------------------------------
#ifndef FR_S2_WARPS  // warps per CTA of kernel S2: 8 (tile 32 x 16) or 4 (half of one; cfg2
                     // 17.5 -> 17.9 us per call, profiles/r02/ab_s2_warps.txt)
#define FR_S2_WARPS 8
#endif
constexpr int kS2Threads = 32 * FR_S2_WARPS;
static_assert(FR_S2_WARPS == 8 || FR_S2_WARPS == 4, "kernel S2: 4 or 8 warps per CTA");
template <bool STRICT, bool MANDEL, bool COLOR, int KV = 4>
__global__ void __launch_bounds__(kS2Threads)
escape_tile2_kernel(const Geom g, const PalRef pal, const float jcr2, const float jci2) {
  // jcr2/jci2: the Julia C in the state representation (doubled in FAST, plain in STRICT)
  // colours from the device palette (no CTA barrier in these short-lived CTAs)
  pdl_trigger();  // the next frame's CTAs may start while this frame's last wave runs
  int tx, ty, grp;
  tile_of(g, tx, ty, grp);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // 4-warp CTAs: grid rows count half tiles; the low bit picks the warp-tile row
  const int wy = FR_S2_WARPS == 8 ? (warp >> 2) : (ty & 1);
  if (FR_S2_WARPS == 4) ty >>= 1;
  const int cx = (warp & 3) * kWarpW + (lane & 7);
  const int cy = wy * kWarpH + (lane >> 3);
  const int px = tx * kTileW + cx;
  const int ly0 = ty * (2 * kTileH) + cy;
  const int ly1 = ly0 + kTileH;
  const bool in0 = (px < g.W) && (ly0 < g.rows);
  const bool in1 = (px < g.W) && (ly1 < g.rows);
  const float re = to_state<float, STRICT>(pixel_re(g, min(px, g.W - 1)));
  const float im0 = to_state<float, STRICT>(pixel_im(g, global_row(g, min(ly0, g.rows - 1))));
  const float im1 = to_state<float, STRICT>(pixel_im(g, global_row(g, min(ly1, g.rows - 1))));
  float x, y, x2, y2, cr, ci, cr2, ci2;
  if (MANDEL) {
    x = y = x2 = y2 = 0.0f;
    cr = re;
    ci = im0;
    cr2 = re;
    ci2 = im1;
  } else {
    x = re;
    y = im0;
    x2 = re;
    y2 = im1;
    cr = cr2 = jcr2;
    ci = ci2 = jci2;
  }
  unsigned alive = in0 ? 1u : 0u, alive2 = in1 ? 1u : 0u;
  int cnt = 0, cnt2 = 0;
  const int max_iter = g.max_iter;
  {
    const int kfull = max_iter - max_iter % KV;
    int n = vote_loop2_f32<STRICT, KV>(x, y, cnt, alive, x2, y2, cnt2, alive2, cr, ci, cr2,
                                       ci2, kfull);
    if (kfull != max_iter && n == kfull && __any_sync(kFull, alive | alive2)) {
      for (; n < max_iter; ++n) {
        Iter<float, STRICT>::step(x, y, cr, ci, alive, cnt);
        Iter<float, STRICT>::step(x2, y2, cr2, ci2, alive2, cnt2);
      }
    }
  }
  pdl_wait();  // stores (and palette reads) only after the previous kernel completed
  if (in0) {
    const int64_t off = (int64_t)ly0 * g.W + px;
    const int c0 = cnt;  // <= max_iter: at most one increment per executed iteration
    g.counts[off] = (uint16_t)c0;
    if (COLOR) g.rgba[off] = colour_dev(pal, c0, max_iter);
  }
  if (in1) {
    const int64_t off = (int64_t)ly1 * g.W + px;
    const int c1 = cnt2;
    g.counts[off] = (uint16_t)c1;
    if (COLOR) g.rgba[off] = colour_dev(pal, c1, max_iter);
  }
}

// ----------------------------------------------------------------------------------
// Figure 4 maps (FnIter, the strict sequence; NEXT-3) on the S2 layout: CTA tile 32 x 16,
// two pixels per thread (rows y and y + 8) iterated together for instruction-level
// parallelism across the long dependent chain of the rational map's divisions.
// ----------------------------------------------------------------------------------
template <class T, int FN, bool COLOR>
__global__ void __launch_bounds__(kThreads)
escape_fn2_kernel(const Geom g, const Palette pal, const T jcr, const T jci) {
  __shared__ uint32_t spal[COLOR ? 256 : 1];
  if (COLOR) {
    spal[threadIdx.x] = pal.e[threadIdx.x];
    __syncthreads();
  }
  pdl_trigger();
  int tx, ty, grp;
  tile_of(g, tx, ty, grp);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int px = tx * kTileW + (warp & 3) * kWarpW + (lane & 7);
  const int ly0 = ty * (2 * kTileH) + (warp >> 2) * kWarpH + (lane >> 3);
  const int ly1 = ly0 + kTileH;
  const bool in0 = (px < g.W) && (ly0 < g.rows);
  const bool in1 = (px < g.W) && (ly1 < g.rows);
  T x = to_state<T, true>(pixel_re(g, min(px, g.W - 1)));
  T y = to_state<T, true>(pixel_im(g, global_row(g, min(ly0, g.rows - 1))));
  T x2 = x;
  T y2 = to_state<T, true>(pixel_im(g, global_row(g, min(ly1, g.rows - 1))));
  unsigned alive = in0 ? 1u : 0u, alive2 = in1 ? 1u : 0u;
  int cnt = 0, cnt2 = 0;
  const int max_iter = g.max_iter;
  const int kfull = max_iter - max_iter % 4;
  using It = FnIter<T, FN>;
  int n = 0;
  while (n < kfull) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      It::step(x, y, jcr, jci, alive, cnt);
      It::step(x2, y2, jcr, jci, alive2, cnt2);
    }
    n += 4;
    if (!__any_sync(kFull, alive | alive2)) break;
  }
  if (kfull != max_iter && n == kfull && __any_sync(kFull, alive | alive2)) {
    for (; n < max_iter; ++n) {
      It::step(x, y, jcr, jci, alive, cnt);
      It::step(x2, y2, jcr, jci, alive2, cnt2);
    }
  }
  pdl_wait();
  if (in0) {
    const int64_t off = (int64_t)ly0 * g.W + px;
    g.counts[off] = (uint16_t)cnt;
    if (COLOR) g.rgba[off] = colour_of(spal, pal, cnt, max_iter);
  }
  if (in1) {
    const int64_t off = (int64_t)ly1 * g.W + px;
    g.counts[off] = (uint16_t)cnt2;
    if (COLOR) g.rgba[off] = colour_of(spal, pal, cnt2, max_iter);
  }
}

// Optional per-warp timeline of kernels R and P2 (diagnostics; null in normal operation):
// [warp][0] = %globaltimer at entry, [1] = at chunk-supply exhaustion, [2] = at exit.
__device__ unsigned long long* g_refill_trace = nullptr;

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ----------------------------------------------------------------------------------
// Two-phase rendering of heavy-tailed single frames (kernels P1 + P2).  Most pixels of a
// heavy-tailed frame escape within a few iterations (cfg3: p50 = 2) while most of the
// WORK is in the few long orbits (cfg3: 20% of pixels survive 32 iterations and carry 83%
// of the iterations).  One kernel serves both badly: small vote blocks waste issue on the
// long orbits, large refill blocks waste most of a block on every short one.
//   P1: static tiles, two pixels per thread (the S2 layout), vote blocks of 4, stop at a
//       budget of B iterations.
//       Pixels that escaped store their count (and colour); survivors append their
//       state (Z_B, B, pixel index) to a queue, one atomic per warp that has any.
//   P2: persistent lane refill over the queue (blocks of K, service threshold TH):
//       warps take 32 items per atomic, the next grab prefetched.  The orbit continues
//       from Z_B with the same arithmetic, so counts are bit-identical to one pass.
// ----------------------------------------------------------------------------------
// 16-byte aligned for binary32 so a whole item moves in one 128-bit load / store
template <class T>
struct alignas(sizeof(T) == 4 ? 16 : 8) QItem {
  T x, y;        // state after the phase-1 budget (kernel representation)
  int cnt;       // iterations done (= the budget)
  unsigned idx;  // pixel index row * W + px within the call's rows
};

struct ContQueue {
  unsigned tail;  // items appended by P1 (its survivors)
  unsigned pad0[31];
  unsigned head;  // items taken by P2
  unsigned pad1[31];
  unsigned done_warps;
  unsigned pad2[31];
  unsigned left;  // reserved (0)
  unsigned pad3[31];
  unsigned head2;  // reserved (0)
  unsigned pad4[31];
};

// KS > 0 (fast modes, under the escape-monotonicity precondition of kernel A / the
// amortised P2): sub-blocks of KS bare Z^2+C steps with one |Z|^2 test at the sub-block
// end; each orbit keeps the start state of its current sub-block until an end state has
// escaped, and escaped orbits recover their exact index by one replay of <= KS steps
// with the per-iteration test after the loop (P1's lanes are never refilled, so one
// replay per orbit, deferred to the end).
// PRE > 0: the first PRE iterations run the exact vote loop (counts of the orbits that
// end there are final); the amortised sub-blocks continue the rest from PRE.
#ifndef FR_P1_WARPS  // warps per CTA of kernel P1: 4 (half of a 32 x 16 tile; cfg3 0.1554 ->
#define FR_P1_WARPS 4  // 0.1544 ms against 8, profiles/r02/ab_p1_warps.txt) or 8
#endif
constexpr int kP1Threads = 32 * FR_P1_WARPS;
template <class T, bool STRICT, bool MANDEL, bool COLOR, int KS, int PRE, int KV>
__device__ __forceinline__ void budget_tile(const Geom& g, const PalRef& pal, const T jcr,
                                            const T jci, int budget, ContQueue* q,
                                            QItem<T>* items, const int tx, const int ty) {
  // CTA tile 32x16: each thread iterates the pixels of rows ly and ly + 8 of its 8x4-lane
  // warp tile together (two orbits, one vote per block of 4; the S2 layout).  Colours come
  // from the device palette: no CTA barrier in these short-lived CTAs.
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // 4-warp CTAs (FR_P1_WARPS): the tile-row index counts half tiles, its low bit the row
  const int wy = FR_P1_WARPS == 8 ? (warp >> 2) : (ty & 1);
  const int tyt = FR_P1_WARPS == 8 ? ty : (ty >> 1);
  const int px = tx * kTileW + (warp & 3) * kWarpW + (lane & 7);
  const int ly0 = tyt * (2 * kTileH) + wy * kWarpH + (lane >> 3);
  const int ly1 = ly0 + kTileH;
  const bool in0 = (px < g.W) && (ly0 < g.rows);
  const bool in1 = (px < g.W) && (ly1 < g.rows);
  const T re = to_state<T, STRICT>(pixel_re(g, min(px, g.W - 1)));
  const T im0 = to_state<T, STRICT>(pixel_im(g, global_row(g, min(ly0, g.rows - 1))));
  const T im1 = to_state<T, STRICT>(pixel_im(g, global_row(g, min(ly1, g.rows - 1))));
  T x, y, x2, y2, cr, ci, cr2, ci2;
  if (MANDEL) {
    x = y = x2 = y2 = T(0);
    cr = re;
    ci = im0;
    cr2 = re;
    ci2 = im1;
  } else {
    x = re;
    y = im0;
    x2 = re;
    y2 = im1;
    cr = cr2 = jcr;
    ci = ci2 = jci;
  }
  unsigned alive = in0 ? 1u : 0u, alive2 = in1 ? 1u : 0u;
  int cnt = 0, cnt2 = 0;
  // budget is a multiple of 4 (of KS when KS > 0) and < max_iter (host)
  if constexpr (KS > 0) {
    static_assert(!STRICT && KS % 2 == 0, "amortised P1: fast modes, pairs of replay steps");
    using It = Iter<T, STRICT>;
    // exact prefix of PRE iterations (most orbits of a heavy-tailed frame end there)
    int n0 = 0;
    if constexpr (PRE > 0) {
      if constexpr (kAsmPair<T, STRICT, 4>) {
        n0 = vote_loop2_f32<STRICT, KV>(x, y, cnt, alive, x2, y2, cnt2, alive2, cr, ci, cr2,
                                        ci2, PRE);
      } else {
        for (; n0 < PRE; n0 += 4) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            Iter<T, STRICT>::step(x, y, cr, ci, alive, cnt);
            Iter<T, STRICT>::step(x2, y2, cr2, ci2, alive2, cnt2);
          }
          if (!__any_sync(kFull, alive | alive2)) break;
        }
      }
    }
    // p: still running after the prefix (its count is final otherwise)
    const bool p0 = alive != 0u, p1 = alive2 != 0u;
    // d: the end state of some sub-block escaped (sticky; NaN/inf count as escaped);
    // (xc, yc) = start state of the first such sub-block, cnt = its first index
    bool d0 = !p0, d1 = !p1;
    if (!__any_sync(kFull, p0 || p1)) n0 = budget;
    if constexpr (std::is_same<T, float>::value) {
      // binary32: both orbits in packed registers (FFMA2/FMUL2)
      float2 X = make_float2(x, x2), Y = make_float2(y, y2);
      const float2 CRp = make_float2(cr, cr2), CIp = make_float2(ci, ci2);
      float2 XC = X, YC = Y;
      for (int n = n0; n < budget; n += KS) {
        if (!d0) {
          XC.x = X.x;
          YC.x = Y.x;
          cnt = n;
        }
        if (!d1) {
          XC.y = X.y;
          YC.y = Y.y;
          cnt2 = n;
        }
#pragma unroll
        for (int j = 0; j < KS; ++j) fast_core2(X, Y, CRp, CIp);
        const float2 M = fast_mag2(X, Y);
        d0 = d0 || !(M.x <= 16.0f);
        d1 = d1 || !(M.y <= 16.0f);
        if (__all_sync(kFull, d0 && d1)) break;
      }
      if (!d0) cnt = budget;
      if (!d1) cnt2 = budget;
      alive = !d0 ? 1u : 0u;
      alive2 = !d1 ? 1u : 0u;
      const bool q0 = p0 && d0, q1 = p1 && d1;
      bool ra = q0, rb = q1;
      int rc = 0, rc2 = 0;
#pragma unroll 1
      for (int j = 0; j < KS; ++j) {
        if (!__any_sync(kFull, ra || rb)) break;
        const float2 m = fast_mag2(XC, YC);
        ra = ra && (m.x <= 16.0f);
        rb = rb && (m.y <= 16.0f);
        if (ra) ++rc;
        if (rb) ++rc2;
        fast_core2(XC, YC, CRp, CIp);
      }
      if (q0) cnt += rc;
      if (q1) cnt2 += rc2;
      x = X.x;
      y = Y.x;
      x2 = X.y;
      y2 = Y.y;
    } else {
    T xc = x, yc = y, xc2 = x2, yc2 = y2;
    for (int n = n0; n < budget; n += KS) {
      if (!d0) {
        xc = x;
        yc = y;
        cnt = n;
      }
      if (!d1) {
        xc2 = x2;
        yc2 = y2;
        cnt2 = n;
      }
#pragma unroll
      for (int j = 0; j < KS; ++j) {
        It::core(x, y, cr, ci);
        It::core(x2, y2, cr2, ci2);
      }
      d0 = d0 || !(It::mag(x, y) <= It::kLim);
      d1 = d1 || !(It::mag(x2, y2) <= It::kLim);
      if (__all_sync(kFull, d0 && d1)) break;
    }
    // survivors: |Z_budget|^2 <= 4, so (monotonicity) every earlier state passed too
    if (!d0) cnt = budget;
    if (!d1) cnt2 = budget;
    alive = !d0 ? 1u : 0u;
    alive2 = !d1 ? 1u : 0u;
    // exact index of the orbits that escaped after the prefix: replay their sub-block
    // from its checkpoint; rc tests passed before the first escaping state (rc == KS:
    // the end state)
    const bool q0 = p0 && d0, q1 = p1 && d1;
    unsigned ra = q0 ? 1u : 0u, rb = q1 ? 1u : 0u;
    int rc = 0, rc2 = 0;
    if (__any_sync(kFull, ra | rb)) {
      for (int j = 0; j < KS; j += 2) {
        It::step(xc, yc, cr, ci, ra, rc);
        It::step(xc2, yc2, cr2, ci2, rb, rc2);
        It::step(xc, yc, cr, ci, ra, rc);
        It::step(xc2, yc2, cr2, ci2, rb, rc2);
        if (!__any_sync(kFull, ra | rb)) break;
      }
    }
    if (q0) cnt += rc;
    if (q1) cnt2 += rc2;
    }
  } else if constexpr (kAsmPair<T, STRICT, 4>) {
    vote_loop2_f32<STRICT, KV>(x, y, cnt, alive, x2, y2, cnt2, alive2, cr, ci, cr2, ci2,
                               budget);
  } else {
    for (int n = 0; n < budget; n += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        Iter<T, STRICT>::step(x, y, cr, ci, alive, cnt);
        Iter<T, STRICT>::step(x2, y2, cr2, ci2, alive2, cnt2);
      }
      if (!__any_sync(kFull, alive | alive2)) break;
    }
  }
  // |Z_n|^2 <= 4 for every n < budget: survivor; else the count is final
  const bool s0 = in0 && alive, s1 = in1 && alive2;
  const unsigned i0 = (unsigned)ly0 * (unsigned)g.W + (unsigned)px;
  const unsigned i1 = (unsigned)ly1 * (unsigned)g.W + (unsigned)px;
  if (in0 && !s0) {
    g.counts[i0] = (uint16_t)cnt;
    if (COLOR) g.rgba[i0] = colour_dev(pal, cnt, g.max_iter);
  }
  if (in1 && !s1) {
    g.counts[i1] = (uint16_t)cnt2;
    if (COLOR) g.rgba[i1] = colour_dev(pal, cnt2, g.max_iter);
  }
  // append the survivors: one atomic per warp that has any (no CTA barrier, so a warp
  // that finished early never waits for the CTA's slowest)
  const unsigned b0 = __ballot_sync(kFull, s0), b1 = __ballot_sync(kFull, s1);
  if (b0 | b1) {
    unsigned base = 0u;
    if (lane == 0) base = atomicAdd(&q->tail, (unsigned)(__popc(b0) + __popc(b1)));
    base = __shfl_sync(kFull, base, 0);
    const unsigned lt = (1u << lane) - 1u;
    if (s0) {
      QItem<T> it;
      it.x = x;
      it.y = y;
      it.cnt = cnt;
      it.idx = i0;
      items[base + (unsigned)__popc(b0 & lt)] = it;
    }
    if (s1) {
      QItem<T> it;
      it.x = x2;
      it.y = y2;
      it.cnt = cnt2;
      it.idx = i1;
      items[base + (unsigned)__popc(b0) + (unsigned)__popc(b1 & lt)] = it;
    }
  }
}

// NT > 1: each CTA renders NT vertically adjacent 32x16 tiles one after the other (fewer,
// longer CTAs; the FRACTAL_P1_TILES experiment of DESIGN.md §5.1c)
template <class T, bool STRICT, bool MANDEL, bool COLOR, int KS = 0, int PRE = 0, int KV = 4,
          int NT = 1>
__global__ void __launch_bounds__(kP1Threads)
escape_budget_kernel(const Geom g, const PalRef pal, const T jcr, const T jci, int budget,
                     ContQueue* q, QItem<T>* items) {
  int tx, ty, grp;
  tile_of(g, tx, ty, grp);
#pragma unroll 1
  for (int h = 0; h < NT; ++h)
    budget_tile<T, STRICT, MANDEL, COLOR, KS, PRE, KV>(g, pal, jcr, jci, budget, q, items, tx,
                                                       ty * NT + h);
}

// AMORT (P2 only, under the escape-monotonicity precondition |C| <= 1.989 checked on the
// host): blocks run the bare Z^2+C core and test |Z|^2 once at the block end; a finished
// lane recovers its exact index by replaying its last block from the saved start state
// with the per-iteration test, when the warp services it (as kernel A).
template <class T, bool STRICT, bool MANDEL, bool COLOR, int K, int TH, bool AMORT = false>
__global__ void __launch_bounds__(kThreads)
escape_cont_kernel(const Geom g, const Palette pal, const T jcr, const T jci, ContQueue* q,
                   const QItem<T>* items) {
  __shared__ uint32_t spal[COLOR ? 256 : 1];
  if (COLOR) {
    spal[threadIdx.x] = pal.e[threadIdx.x];
    __syncthreads();
  }
  using It = Iter<T, STRICT>;
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int max_iter = g.max_iter;
  const unsigned n_items = *reinterpret_cast<volatile unsigned*>(&q->tail);
  unsigned long long* trace = g_refill_trace;
  const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  if (trace && lane == 0) trace[gw * 3] = global_ns();
  bool exhausted = false;
  unsigned need = kFull;
  // Items are staged in registers, one per lane: `cur` holds the current grab of 32
  // positions [cbase, cbase + 32), `nxt` the next one.  The next grab's atomic is issued
  // when a grab becomes current and its items are loaded at the following dispense
  // event, so a refill takes its item by shuffle with no memory latency.
  unsigned cbase = 0u, gpos = 0u, gend = 0u;  // current grab; [gpos, gend) undispensed
  QItem<T> cur{}, nxt{};
  unsigned nbase = 0u;
  bool nxt_loaded = false;  // nxt holds the items of grab nbase
  unsigned pf = 0u;         // lane 0: base of the prefetched grab (valid if pf_issued)
  bool pf_issued = false;
  auto load_grab = [&](unsigned base, QItem<T>& dst) {
    if (base + (unsigned)lane < n_items) dst = items[base + (unsigned)lane];
  };

  T x = T(0), y = T(0), cr = jcr, ci = jci;
  unsigned alive = 0u;
  int cnt = 0;
  int64_t off = -1;

  for (;;) {
    while (need != 0u && !exhausted) {
      if (gpos >= gend) {
        // switch to the next grab: staged if possible, else fetch it now
        if (!nxt_loaded) {
          unsigned base = 0u;
          if (lane == 0) base = pf_issued ? pf : atomicAdd(&q->head, 32u);
          nbase = __shfl_sync(kFull, base, 0);
          pf_issued = false;
          if (nbase < n_items) load_grab(nbase, nxt);
        }
        nxt_loaded = false;
        if (nbase >= n_items) {
          exhausted = true;
          if (trace && lane == 0) trace[gw * 3 + 1] = global_ns();
          break;
        }
        cur = nxt;
        cbase = nbase;
        gpos = nbase;
        gend = min(nbase + 32u, n_items);
        if (gend < n_items) {  // prefetch the following grab
          if (lane == 0) pf = atomicAdd(&q->head, 32u);
          pf_issued = true;
        }
      } else if (pf_issued && !nxt_loaded) {
        // the prefetch atomic has had a block to return: stage its items
        nbase = __shfl_sync(kFull, pf, 0);
        pf_issued = false;
        nxt_loaded = true;
        if (nbase < n_items) load_grab(nbase, nxt);
      }
      const unsigned avail = gend - gpos;
      const unsigned rank = (unsigned)__popc(need & lt_mask);
      const bool mine = (need >> lane) & 1u;
      const int src = (int)(gpos - cbase + (rank < avail ? rank : 0u));
      const T ix = __shfl_sync(kFull, cur.x, src);
      const T iy = __shfl_sync(kFull, cur.y, src);
      const int icnt = __shfl_sync(kFull, cur.cnt, src);
      const unsigned iidx = __shfl_sync(kFull, cur.idx, src);
      bool got = false;
      if (mine && rank < avail) {
        got = true;
        off = iidx;
        x = ix;
        y = iy;
        cnt = icnt;
        alive = 1u;
        if (MANDEL) {
          const int row = (int)(iidx / (unsigned)g.W);
          const int px = (int)(iidx - (unsigned)row * (unsigned)g.W);
          cr = to_state<T, STRICT>(pixel_re(g, px));
          ci = to_state<T, STRICT>(pixel_im(g, global_row(g, row)));
        }
      }
      const unsigned nneed = (unsigned)__popc(need);
      gpos += nneed < avail ? nneed : avail;
      need = __ballot_sync(kFull, mine && !got);
    }
    const int n_held = __popc(__ballot_sync(kFull, off >= 0));
    if (n_held == 0) break;
    const bool held = off >= 0;
    if constexpr (AMORT) {
      // cnt = iterations done; Z_cnt (= (x, y)) not yet tested.  A finished lane freezes
      // (x0, y0, cnt) until it is serviced.  Once the queue is dry the warp runs until
      // every held lane has finished and services them all at once.
      const int thr = exhausted ? n_held : (TH < n_held ? TH : n_held);
      // the block is NS sub-blocks of KS iterations; each sub-block's start state is
      // checkpointed, so the replay covers one sub-block, not the whole block
      constexpr int KS = (K % FR_P2A_KS == 0) ? FR_P2A_KS : K;
      constexpr int NS = K / KS;
      static_assert(KS % 2 == 0, "the replay runs pairs of steps");
      bool done = !held, esc = false;
      T xs[NS], ys[NS];
#pragma unroll
      for (int sb = 0; sb < NS; ++sb) {
        xs[sb] = x;
        ys[sb] = y;
      }
      unsigned fm;
      for (;;) {
#pragma unroll
        for (int sb = 0; sb < NS; ++sb) {
          if (!done) {
            xs[sb] = x;
            ys[sb] = y;
          }
#pragma unroll
          for (int j = 0; j < KS; ++j) It::core(x, y, cr, ci);
        }
        const bool e = !(It::mag(x, y) <= It::kLim);  // unordered: NaN/inf count as escaped
        if (!done && (e || cnt + K >= max_iter)) {
          done = true;
          esc = e;
        }
        if (!done) cnt += K;
        fm = __ballot_sync(kFull, held && done);
        if (__popc(fm) >= thr) break;
      }
      if (held && done) {
        // exact index: the first sub-block whose end state escaped (monotonicity: every
        // later state escaped too), replayed from its checkpoint with the per-iteration
        // test until every replaying lane has escaped
        T rx = xs[NS - 1], ry = ys[NS - 1];
        int sbase = (NS - 1) * KS;
#pragma unroll
        for (int sb = NS - 2; sb >= 0; --sb) {
          if (!(It::mag(xs[sb + 1], ys[sb + 1]) <= It::kLim)) {
            rx = xs[sb];
            ry = ys[sb];
            sbase = sb * KS;
          }
        }
        unsigned ra = 1u;
        int rc = 0;
        for (int j = 0; j < KS; j += 2) {
          It::step(rx, ry, cr, ci, ra, rc);
          It::step(rx, ry, cr, ci, ra, rc);
          if (!__any_sync(fm, ra)) break;
        }
        // rc < KS: escaped at cnt + sbase + rc; rc == KS: at the sub-block's end state if
        // `esc`, else the iteration limit was reached without escape
        const int count0 = esc ? cnt + sbase + rc : max_iter;
        const int count = count0 < max_iter ? count0 : max_iter;
        g.counts[off] = (uint16_t)count;
        if (COLOR) g.rgba[off] = colour_of(spal, pal, count, max_iter);
        off = -1;
      }
      if (exhausted) break;
      need = fm;
      continue;
    }
    if (exhausted) {
      // Queue dry: nothing left to refill, so no per-lane servicing -- run blocks until
      // no held orbit is still alive below max_iter (one vote per block), then store all.
      // A finished lane's count is frozen (sticky alive), and iterating past max_iter
      // is harmless (counts are clamped at the store).
      if (!held) alive = 0u;
      while (__any_sync(kFull, held && alive && cnt < max_iter)) {
#pragma unroll
        for (int j = 0; j < K; ++j) It::step(x, y, cr, ci, alive, cnt);
      }
      if (held) {
        const int count = cnt < max_iter ? cnt : max_iter;
        g.counts[off] = (uint16_t)count;
        if (COLOR) g.rgba[off] = colour_of(spal, pal, count, max_iter);
        off = -1;
      }
      break;
    }
    const int thr = TH < n_held ? TH : n_held;
    const int lim = held ? max_iter : 0x7fffffff;
    if (!held) alive = 0u;
    bool fin;
    unsigned fm;
    for (;;) {
#pragma unroll
      for (int j = 0; j < K; ++j) It::step(x, y, cr, ci, alive, cnt);
      fin = held && (!alive || cnt >= lim);
      fm = __ballot_sync(kFull, fin);
      if (__popc(fm) >= thr) break;
    }
    if (fin) {
      const int count = cnt < max_iter ? cnt : max_iter;
      g.counts[off] = (uint16_t)count;
      if (COLOR) g.rgba[off] = colour_of(spal, pal, count, max_iter);
      off = -1;
      alive = 0u;
    }
    need = fm;
  }
  if (trace && lane == 0) trace[gw * 3 + 2] = global_ns();
  // ---- self-reset of the queue by the last warp to finish
  if (lane == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&q->done_warps, 1u);
    if (prev == gridDim.x * (kThreads / 32) - 1) {
      q->tail = 0u;
      q->head = 0u;
      q->done_warps = 0u;
      __threadfence();
    }
  }
}


// ----------------------------------------------------------------------------------
// "P2S" (experimental, FRACTAL_P2S=1): P2 for FP32_FAST under the
// escape-monotonicity precondition with two orbits ("slots") per lane in packed float2
// registers (FFMA2/FMUL2), blocks of K bare iterations with the sub-block start states
// kept and one |Z|^2 test per slot at the block end.  On cfg3's survivors the 64 slots
// of a warp finish ~8 times per 32-iteration block, so finishing must be cheap and
// mostly non-collective:
//   * a finished slot that escaped appends a replay record (the start of its escaping
//     sub-block and its index) to a per-warp buffer in shared memory; an interior one
//     stores max_iter directly;
//   * it continues with its stash, an item already in registers; emptied stashes are
//     refilled by plain per-lane loads at ranked positions of a warp-private range of
//     queue positions (RG per atomic, the next range reserved ahead), so the load
//     latency hides behind the orbit in front of it -- no shuffles;
//   * once 64 records are pending the warp replays them together, two per lane in the
//     packed loop with the per-iteration test (<= KS steps, vote exit), and stores the
//     exact counts: SIMT-efficient and without a global round trip.
// ----------------------------------------------------------------------------------
template <bool MANDEL, bool COLOR, int K>
__global__ void __launch_bounds__(kThreads)
escape_cont2s_kernel(const Geom g, const PalRef pal, const float jcr2, const float jci2,
                     ContQueue* q, const QItem<float>* items) {
  constexpr int KS = 8, NS = K / KS;
  static_assert(K % KS == 0 && NS >= 1 && NS <= 8, "blocks of sub-blocks of 8");
  constexpr unsigned RG = 32;   // queue positions per range reservation
  constexpr unsigned PB = 128;  // pending replay records per warp (ring; <= 127 live)
  __shared__ QItem<float> pend_buf[kThreads / 32][PB];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int max_iter = g.max_iter;
  const unsigned n_items = *reinterpret_cast<volatile unsigned*>(&q->tail);
  unsigned long long* trace = g_refill_trace;
  const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + warp;
  if (trace && lane == 0) trace[gw * 3] = global_ns();
  QItem<float>* pb = pend_buf[warp];
  unsigned ph = 0u, pn = 0u;  // pending ring: head, count (warp-uniform)
  auto c_of = [&](unsigned idx, float& cr, float& ci) {
    const int row = (int)(idx / (unsigned)g.W);
    const int px = (int)(idx - (unsigned)row * (unsigned)g.W);
    cr = to_state<float, false>(pixel_re(g, px));
    ci = to_state<float, false>(pixel_im(g, global_row(g, row)));
  };
  const float2 HALF = make_float2(0.5f, 0.5f);
  // replay up to 64 pending records (two per lane, packed) and store their counts
  auto replay = [&](unsigned n) {
    const unsigned s0 = (ph + (unsigned)lane) & (PB - 1), s1 = (ph + 32u + (unsigned)lane) & (PB - 1);
    const bool a = (unsigned)lane < n, b = (unsigned)lane + 32u < n;
    QItem<float> r0{}, r1{};
    if (a) r0 = pb[s0];
    if (b) r1 = pb[s1];
    float2 x = make_float2(r0.x, r1.x), y = make_float2(r0.y, r1.y);
    float2 cr = make_float2(jcr2, jcr2), ci = make_float2(jci2, jci2);
    if (MANDEL) {
      if (a) c_of(r0.idx, cr.x, ci.x);
      if (b) c_of(r1.idx, cr.y, ci.y);
    }
    bool pa = a, pb_ = b;
    int na = 0, nb = 0;
#pragma unroll 1
    for (int j = 0; j < KS; ++j) {
      if (!__any_sync(kFull, pa || pb_)) break;
      const float2 m = ffma2(x, x, fmul2(y, y));
      pa = pa && (m.x <= 16.0f);
      pb_ = pb_ && (m.y <= 16.0f);
      if (pa) ++na;
      if (pb_) ++nb;
      const float2 YY = fmul2(y, y);
      const float2 T = ffma2(x, x, fneg2(YY));
      const float2 Yn = ffma2(x, y, ci);
      x = ffma2(T, HALF, cr);
      y = Yn;
    }
    // na == KS: the sub-block's end state escaped
    if (a) {
      const int c0 = r0.cnt + na;
      const int count = c0 < max_iter ? c0 : max_iter;
      g.counts[r0.idx] = (uint16_t)count;
      if (COLOR) g.rgba[r0.idx] = colour_dev(pal, count, max_iter);
    }
    if (b) {
      const int c0 = r1.cnt + nb;
      const int count = c0 < max_iter ? c0 : max_iter;
      g.counts[r1.idx] = (uint16_t)count;
      if (COLOR) g.rgba[r1.idx] = colour_dev(pal, count, max_iter);
    }
    __syncwarp();
    ph = (ph + n) & (PB - 1);
    pn -= n;
  };
  // ---- warp-private queue ranges: current [r0, r1), next [nx, nx + RG) (reserved)
  unsigned r0 = 0u, r1 = 0u, nx = 0u;
  bool exhausted = false;
  {
    unsigned b = 0u;
    if (lane == 0) b = atomicAdd(&q->head, 4u * 32u);  // slots + stashes
    r0 = __shfl_sync(kFull, b, 0);
    if (lane == 0) nx = atomicAdd(&q->head, RG);  // lane 0 only, until shuffled
  }
  float2 X, Y;
  float2 CR = make_float2(jcr2, jcr2), CI = make_float2(jci2, jci2);
  int ca, cb;
  unsigned ia, ib;
  bool ha, hb;
  QItem<float> sa{}, sb{};
  bool va, vb;
  {
    const unsigned pa = r0 + (unsigned)lane, pb2 = pa + 32u, psa = pa + 64u, psb = pa + 96u;
    QItem<float> ta{}, tb{};
    ha = pa < n_items;
    hb = pb2 < n_items;
    va = psa < n_items;
    vb = psb < n_items;
    if (ha) ta = items[pa];
    if (hb) tb = items[pb2];
    if (va) sa = items[psa];
    if (vb) sb = items[psb];
    X = make_float2(ta.x, tb.x);
    Y = make_float2(ta.y, tb.y);
    ca = ta.cnt;
    cb = tb.cnt;
    ia = ta.idx;
    ib = tb.idx;
    if (MANDEL) {
      if (ha) c_of(ia, CR.x, CI.x);
      if (hb) c_of(ib, CR.y, CI.y);
    }
    r0 = r1 = 0u;  // the first block of positions is used up
    exhausted = __shfl_sync(kFull, nx, 0) >= n_items;
  }
  for (;;) {
    if (!__any_sync(kFull, ha || hb)) break;
    float2 CX[NS], CY[NS];
#pragma unroll
    for (int s2 = 0; s2 < NS; ++s2) {
      CX[s2] = X;
      CY[s2] = Y;
#pragma unroll
      for (int j = 0; j < KS; ++j) {
        const float2 YY = fmul2(Y, Y);
        const float2 T = ffma2(X, X, fneg2(YY));
        const float2 Yn = ffma2(X, Y, CI);
        X = ffma2(T, HALF, CR);
        Y = Yn;
      }
    }
    const float2 M = ffma2(X, X, fmul2(Y, Y));
    const bool ea = !(M.x <= 16.0f), eb = !(M.y <= 16.0f);  // unordered: NaN/inf escaped
    const bool fa = ha && (ea || ca + K >= max_iter);
    const bool fb = hb && (eb || cb + K >= max_iter);
    if (ha && !fa) ca += K;
    if (hb && !fb) cb += K;
    if (!__any_sync(kFull, fa || fb)) continue;
    // ---- finished slots: pending replay record (escaped) or the interior count
    {
      float2 sx = CX[NS - 1], sy = CY[NS - 1];
      int oa = (NS - 1) * KS, ob = (NS - 1) * KS;
#pragma unroll
      for (int s2 = NS - 2; s2 >= 0; --s2) {
        const float2 m = ffma2(CX[s2 + 1], CX[s2 + 1], fmul2(CY[s2 + 1], CY[s2 + 1]));
        if (!(m.x <= 16.0f)) { sx.x = CX[s2].x; sy.x = CY[s2].x; oa = s2 * KS; }
        if (!(m.y <= 16.0f)) { sx.y = CX[s2].y; sy.y = CY[s2].y; ob = s2 * KS; }
      }
      const bool ra = fa && ea, rb = fb && eb;
      const unsigned qa_m = __ballot_sync(kFull, ra), qb_m = __ballot_sync(kFull, rb);
      const unsigned ka = (unsigned)__popc(qa_m & lt);
      const unsigned kb = (unsigned)__popc(qa_m) + (unsigned)__popc(qb_m & lt);
      if (ra) {
        QItem<float> r;
        r.x = sx.x; r.y = sy.x; r.cnt = ca + oa; r.idx = ia;
        pb[(ph + pn + ka) & (PB - 1)] = r;
      }
      if (rb) {
        QItem<float> r;
        r.x = sx.y; r.y = sy.y; r.cnt = cb + ob; r.idx = ib;
        pb[(ph + pn + kb) & (PB - 1)] = r;
      }
      pn += (unsigned)(__popc(qa_m) + __popc(qb_m));
      if (fa && !ea) {
        g.counts[ia] = (uint16_t)max_iter;
        if (COLOR) g.rgba[ia] = pal.interior;
      }
      if (fb && !eb) {
        g.counts[ib] = (uint16_t)max_iter;
        if (COLOR) g.rgba[ib] = pal.interior;
      }
      // continue with the stash
      if (fa) {
        X.x = sa.x; Y.x = sa.y; ca = sa.cnt; ia = sa.idx;
        ha = va;
        va = false;
        if (MANDEL && ha) c_of(ia, CR.x, CI.x);
      }
      if (fb) {
        X.y = sb.x; Y.y = sb.y; cb = sb.cnt; ib = sb.idx;
        hb = vb;
        vb = false;
        if (MANDEL && hb) c_of(ib, CR.y, CI.y);
      }
      __syncwarp();
      if (pn >= 64u) replay(64u);
    }
    if (exhausted) continue;
    // ---- refill the emptied stashes from the warp's ranges (per-lane loads)
    const unsigned ma = __ballot_sync(kFull, fa), mb = __ballot_sync(kFull, fb);
    const unsigned m = (unsigned)(__popc(ma) + __popc(mb));
    const unsigned ka = (unsigned)__popc(ma & lt);
    const unsigned kb = (unsigned)__popc(ma) + (unsigned)__popc(mb & lt);
    unsigned cur = r1 - r0;
    unsigned nb = __shfl_sync(kFull, nx, 0);
    // (m <= 64 may need up to two fresh ranges beyond the current one)
    unsigned nb2 = 0u;
    if (m > cur + RG) {
      if (lane == 0) nb2 = atomicAdd(&q->head, RG);
      nb2 = __shfl_sync(kFull, nb2, 0);
    }
    auto pos_of = [&](unsigned k) {
      return k < cur ? r0 + k : (k < cur + RG ? nb + (k - cur) : nb2 + (k - cur - RG));
    };
    if (fa) {
      const unsigned p = pos_of(ka);
      va = p < n_items;
      if (va) sa = items[p];
    }
    if (fb) {
      const unsigned p = pos_of(kb);
      vb = p < n_items;
      if (vb) sb = items[p];
    }
    if (m < cur) {
      r0 += m;
    } else {  // moved into the next range(s): reserve the one after
      if (m < cur + RG) {
        r0 = nb + (m - cur);
        r1 = nb + RG;
      } else {
        r0 = nb2 + (m - cur - RG);
        r1 = nb2 + RG;
        nb = nb2;
      }
      if (lane == 0) nx = atomicAdd(&q->head, RG);
      if (nb >= n_items) {
        exhausted = true;
        if (trace && lane == 0) trace[gw * 3 + 1] = global_ns();
      }
    }
  }
  while (pn > 0u) replay(pn < 64u ? pn : 64u);
  if (trace && lane == 0) trace[gw * 3 + 2] = global_ns();
  // ---- self-reset of the queue by the last warp to finish
  if (lane == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&q->done_warps, 1u);
    if (prev == gridDim.x * (kThreads / 32) - 1) {
      q->tail = 0u;
      q->head = 0u;
      q->left = 0u;
      q->head2 = 0u;
      q->done_warps = 0u;
      __threadfence();
    }
  }
}

// ----------------------------------------------------------------------------------
// Persistent lane-refill kernel (R) for one frame whose counts are heavy-tailed or long
// (SURVEY §7 hard part 1).  Each warp owns a 32x8-pixel chunk at a time, taken from a
// global atomic chunk counter (self-resetting workspace).  Every lane iterates its own
// pixel in unrolled blocks of K; at a block end the lanes whose pixel finished store
// the count (and colour) and, once at least TH lanes are free, take the next pixels of
// the chunk by prefix rank, grabbing a new chunk when it is exhausted.  SIMT lanes
// therefore stay busy whatever their neighbours' counts.
//
// AMORT = false: exact escape test every iteration (sticky predicate + increment).
// AMORT = true : the block runs the bare Z^2+C core (4 FP ops fast, 7 strict) and tests
//   |Z|^2 once at the block end; a lane that escaped inside the block replays the block
//   from its saved start state with the per-iteration test to recover the exact index.
//   Exact given escape monotonicity: with |C| <= 1.99 (checked on the host) an orbit
//   with |Z_n|^2 > 4 satisfies |Z_{n+1}| >= |Z_n|^2 - |C| - err > 2 forever after
//   (DESIGN.md "Escape-monotonicity lemma"), so the block-end test cannot miss an escape.
// ----------------------------------------------------------------------------------
struct Workspace {
  unsigned int next_chunk;
  unsigned int done_warps;
  unsigned int pad[30];
};

template <class T, bool STRICT, bool MANDEL, bool COLOR, bool AMORT, int K, int TH>
__global__ void __launch_bounds__(kThreads)
escape_refill_kernel(const Geom g, const Palette pal, const T jcr, const T jci, Workspace* ws,
                     unsigned n_chunks, unsigned chunks_per_cta) {
  __shared__ uint32_t spal[COLOR ? 256 : 1];
  __shared__ T tre[kThreads / 32][kTileW];
  __shared__ T tim[kThreads / 32][kTileH];
  __shared__ unsigned s_next;  // CTA-local chunk source (chunks_per_cta > 0)
  if (COLOR) spal[threadIdx.x] = pal.e[threadIdx.x];
  if (threadIdx.x == 0) s_next = 0u;
  __syncthreads();
  // chunk source: CTA-local range [c_lo, c_hi) when chunks_per_cta > 0 (the hardware
  // block scheduler balances CTAs and a CTA's drain overlaps its SM neighbours'
  // work), else the global counter of the persistent grid
  const unsigned c_lo = chunks_per_cta ? blockIdx.x * chunks_per_cta : 0u;
  const unsigned c_hi = chunks_per_cta ? min(n_chunks, c_lo + chunks_per_cta) : n_chunks;
  using It = Iter<T, STRICT>;
  constexpr int kChunk = kTileW * kTileH;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int max_iter = g.max_iter;
  unsigned long long* trace = g_refill_trace;
  const int64_t gw = (int64_t)blockIdx.x * (kThreads / 32) + warp;
  if (trace && lane == 0) trace[gw * 3] = global_ns();

  // warp-uniform state
  int chunk_x0 = 0, chunk_y0 = 0;
  int next_idx = kChunk;   // next undispensed pixel of the chunk (kChunk = exhausted)
  bool exhausted = false;  // the global chunk counter ran past the frame
  unsigned need = kFull;   // lanes that need a pixel

  // per-lane pixel state
  T x = T(0), y = T(0), cr = jcr, ci = jci;
  T x0 = T(0), y0 = T(0);  // AMORT: state at the start of the current block
  unsigned alive = 0u;
  int cnt = 0;             // exact: leading iterations with |Z|^2 <= 4; AMORT: iterations done
  int64_t off = -1;        // output offset of the lane's pixel; < 0: no pixel

  for (;;) {
    // ---- hand the next pixels of the chunk to the lanes in `need` (prefix rank)
    while (need != 0u && !exhausted) {
      if (next_idx >= kChunk) {
        unsigned cid = 0;
        if (lane == 0) cid = chunks_per_cta ? c_lo + atomicAdd(&s_next, 1u)
                                            : atomicAdd(&ws->next_chunk, 1u);
        cid = __shfl_sync(kFull, cid, 0);
        if (cid >= c_hi) {
          exhausted = true;
          if (trace && lane == 0) trace[gw * 3 + 1] = global_ns();
          break;
        }
        const int cty = (int)(cid / (unsigned)g.tiles_x);
        chunk_x0 = ((int)cid - cty * g.tiles_x) * kTileW;
        chunk_y0 = cty * kTileH;
        __syncwarp();
        tre[warp][lane] = to_state<T, STRICT>(pixel_re(g, min(chunk_x0 + lane, g.W - 1)));
        if (lane < kTileH)
          tim[warp][lane] = to_state<T, STRICT>(
              pixel_im(g, global_row(g, min(chunk_y0 + lane, g.rows - 1))));
        __syncwarp();
        next_idx = 0;
      }
      const int avail = kChunk - next_idx;
      const int rank = __popc(need & lt_mask);
      const bool mine = (need >> lane) & 1u;
      bool got = false;
      if (mine && rank < avail) {
        const int idx = next_idx + rank;
        const int lx = idx & (kTileW - 1);
        const int lyy = idx >> 5;
        const int px = chunk_x0 + lx;
        const int row = chunk_y0 + lyy;
        if (px < g.W && row < g.rows) {  // else: off-frame pixel of an edge chunk, skipped
          got = true;
          off = (int64_t)row * g.W + px;
          const T a = tre[warp][lx], b = tim[warp][lyy];
          if (MANDEL) {
            x = T(0);
            y = T(0);
            cr = a;
            ci = b;
          } else {
            x = a;
            y = b;
          }
          alive = 1u;
          cnt = 0;
        }
      }
      const int nneed = __popc(need);
      next_idx += nneed < avail ? nneed : avail;
      need = __ballot_sync(kFull, mine && !got);
    }
    const int n_held = __popc(__ballot_sync(kFull, off >= 0));
    if (n_held == 0) break;  // chunks exhausted and every pixel stored
    const bool held = off >= 0;

    // ---- iterate in blocks of K until >= TH lanes finished (or all held lanes, or the end)
    bool fin;
    unsigned fm;
    if (!AMORT) {
      // service the warp once `thr` lanes finished: TH normally, 1 once the chunks are
      // exhausted, and never more than the lanes it holds
      const int thr = exhausted ? 1 : (TH < n_held ? TH : n_held);
      const int lim = held ? max_iter : 0x7fffffff;  // lanes without a pixel never finish
      if (!held) alive = 0u;
      for (;;) {
#pragma unroll
        for (int j = 0; j < K; ++j) It::step(x, y, cr, ci, alive, cnt);
        fin = held && (!alive || cnt >= lim);
        fm = __ballot_sync(kFull, fin);
        if (__popc(fm) >= thr) break;
      }
    } else {
      // a finished lane freezes (x0, y0, cnt) until the warp services it
      bool done = false, esc = false;
      for (;;) {
        if (!done) {
          x0 = x;
          y0 = y;
        }
#pragma unroll
        for (int j = 0; j < K; ++j) It::core(x, y, cr, ci);
        const bool e = !(It::mag(x, y) <= It::kLim);  // unordered: NaN/inf count as escaped
        if (held && !done && (e || cnt + K >= max_iter)) {
          done = true;
          esc = e;
        }
        if (!done) cnt += K;
        fm = __ballot_sync(kFull, held && done);
        if (fm != 0u) {
          const int nf = __popc(fm);
          if (nf >= TH || exhausted || nf == n_held) break;
        }
      }
      fin = held && done;
      if (fin) {
        // exact index: replay the block from its start state with the per-iteration test
        T rx = x0, ry = y0;
        unsigned ra = 1u;
        int rc = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) It::step(rx, ry, cr, ci, ra, rc);
        // rc < K: escaped at cnt + rc; rc == K: escaped at the block-end state (cnt + K)
        // if `esc`, else the iteration limit was reached without escape.
        cnt = esc ? cnt + rc : max_iter;
      }
    }
    if (fin) {
      const int count = cnt < max_iter ? cnt : max_iter;
      g.counts[off] = (uint16_t)count;
      if (COLOR) g.rgba[off] = colour_of(spal, pal, count, max_iter);
      off = -1;
      alive = 0u;
    }
    need = fm;
  }

  if (trace && lane == 0) trace[gw * 3 + 2] = global_ns();
  // ---- self-reset of the workspace by the last warp to finish (persistent grid)
  if (!chunks_per_cta && lane == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(&ws->done_warps, 1u);
    if (prev == gridDim.x * (kThreads / 32) - 1) {
      ws->next_chunk = 0u;
      ws->done_warps = 0u;
      __threadfence();
    }
  }
}

// ----------------------------------------------------------------------------------
// Standalone colour levels (N6): HBM-bound, 8 pixels per thread per step: one 16-byte
// load of counts, two 16-byte stores of RGBA; grid-stride over 8-pixel groups.
// ----------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads)
colorize_kernel(const uint16_t* __restrict__ counts, int64_t n_pixels, int max_iter,
                const Palette pal, uint32_t* __restrict__ rgba) {
  __shared__ uint32_t spal[256];
  spal[threadIdx.x] = pal.e[threadIdx.x];
  __syncthreads();
  const int64_t groups = n_pixels >> 3;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const uint4* __restrict__ c8 = reinterpret_cast<const uint4*>(counts);
  uint4* __restrict__ o8 = reinterpret_cast<uint4*>(rgba);
  auto pack = [&](uint32_t w16) { return colour_of(spal, pal, (int)(w16 & 0xffffu), max_iter); };
  auto emit = [&](int64_t i, const uint4 v) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      o[2 * k] = pack(w[k] & 0xffffu);
      o[2 * k + 1] = pack(w[k] >> 16);
    }
    __stcs(o8 + 2 * i, make_uint4(o[0], o[1], o[2], o[3]));
    __stcs(o8 + 2 * i + 1, make_uint4(o[4], o[5], o[6], o[7]));
  };
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // four 16-byte loads in flight per thread before any store (memory-level parallelism;
  // measured 0.80 of the HBM copy peak vs 0.68 with one and 0.73 with eight)
  constexpr int U = 4;
  for (; i + (U - 1) * stride < groups; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(c8 + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) emit(i + u * stride, v[u]);
  }
  for (; i < groups; i += stride) emit(i, __ldcs(c8 + i));
  // ragged tail (< 8 pixels)
  const int64_t t0 = groups << 3;
  const int64_t t = t0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && t < n_pixels) rgba[t] = colour_of(spal, pal, counts[t], max_iter);
}

// Variant with warp-contiguous stores: a warp handles blocks of 256 pixels, lane l the
// pixels 4l..4l+3 and 128+4l..128+4l+3, so each 16-byte store instruction of the warp
// covers 512 contiguous bytes (whole lines) and each 8-byte load 256 contiguous bytes
// (the kernel above stores 16 bytes per lane at a 32-byte stride).  FR_COLORIZE_V2 picks it.
__global__ void __launch_bounds__(kThreads)
colorize_kernel2(const uint16_t* __restrict__ counts, int64_t n_pixels, int max_iter,
                 const Palette pal, uint32_t* __restrict__ rgba) {
  __shared__ uint32_t spal[256];
  spal[threadIdx.x] = pal.e[threadIdx.x];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nblk = n_pixels >> 8;
  const uint2* __restrict__ c4 = reinterpret_cast<const uint2*>(counts);
  uint4* __restrict__ o4 = reinterpret_cast<uint4*>(rgba);
  auto col4 = [&](const uint2 v) {
    return make_uint4(colour_of(spal, pal, (int)(v.x & 0xffffu), max_iter),
                      colour_of(spal, pal, (int)(v.x >> 16), max_iter),
                      colour_of(spal, pal, (int)(v.y & 0xffffu), max_iter),
                      colour_of(spal, pal, (int)(v.y >> 16), max_iter));
  };
  int64_t b = (((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5);
#ifndef FR_COLORIZE_U
#define FR_COLORIZE_U 4
#endif
  constexpr int U = FR_COLORIZE_U;
  for (; b + (U - 1) * nwarps < nblk; b += U * nwarps) {
    uint2 va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = (b + u * nwarps) * 64 + lane;
      va[u] = __ldcs(c4 + q);
      vb[u] = __ldcs(c4 + q + 32);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = (b + u * nwarps) * 64 + lane;
      __stcs(o4 + q, col4(va[u]));
      __stcs(o4 + q + 32, col4(vb[u]));
    }
  }
  for (; b < nblk; b += nwarps) {
    const int64_t q = b * 64 + lane;
    const uint2 va = __ldcs(c4 + q), vb = __ldcs(c4 + q + 32);
    __stcs(o4 + q, col4(va));
    __stcs(o4 + q + 32, col4(vb));
  }
  // ragged tail (< 256 pixels)
  for (int64_t t = (nblk << 8) + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_pixels;
       t += (int64_t)gridDim.x * blockDim.x)
    rgba[t] = colour_of(spal, pal, counts[t], max_iter);
}

// Unaligned fallback (pointers not 16-byte aligned): one pixel per thread-step.
__global__ void __launch_bounds__(kThreads)
colorize_scalar_kernel(const uint16_t* __restrict__ counts, int64_t n_pixels, int max_iter,
                       const Palette pal, uint32_t* __restrict__ rgba) {
  __shared__ uint32_t spal[256];
  spal[threadIdx.x] = pal.e[threadIdx.x];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_pixels; i += stride)
    rgba[i] = colour_of(spal, pal, counts[i], max_iter);
}

}  // namespace fr
