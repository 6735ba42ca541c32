// Microbenchmark: issue rate of the escape-time inner-loop instruction forms on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define N_IT 4096
__device__ float sink_f; __device__ int sink_i;

// (a) the fast iteration with per-iteration FSETP + predicated IADD (current kernel body)
__global__ void k_iter7(float cr2, float ci2, int n) {
  float X = threadIdx.x * 1e-3f, Y = blockIdx.x * 1e-4f; int cnt = 0; unsigned alive = 1;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      float YY = Y * Y; float M = __fmaf_rn(X, X, YY);
      asm("{\n\t.reg .pred pa, pb;\n\tsetp.ne.u32 pa, %1, 0;\n\tsetp.le.and.f32 pb, %2, 0f41800000, pa;\n\tselp.u32 %1, 1, 0, pb;\n\t@pb add.s32 %0, %0, 1;\n\t}" : "+r"(cnt), "+r"(alive) : "f"(M));
      float T = __fmaf_rn(X, X, -YY); float Yn = __fmaf_rn(X, Y, ci2); X = __fmaf_rn(T, 0.5f, cr2); Y = Yn;
    }
  }
  if (X == 12345.f) { sink_f = Y; sink_i = cnt; }
}
// (b) pure 4-op iteration (amortized test)
__global__ void k_iter4(float cr2, float ci2, int n) {
  float X = threadIdx.x * 1e-3f, Y = blockIdx.x * 1e-4f;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      float YY = Y * Y; float T = __fmaf_rn(X, X, -YY); float Yn = __fmaf_rn(X, Y, ci2); X = __fmaf_rn(T, 0.5f, cr2); Y = Yn;
    }
  }
  if (X == 12345.f) sink_f = Y;
}
// (c) 2 independent pixels per thread, 4-op iteration
__global__ void k_iter4x2(float cr2, float ci2, int n) {
  float X = threadIdx.x * 1e-3f, Y = blockIdx.x * 1e-4f, X2 = X + 0.1f, Y2 = Y - 0.1f;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      float YY = Y * Y; float T = __fmaf_rn(X, X, -YY); float Yn = __fmaf_rn(X, Y, ci2); X = __fmaf_rn(T, 0.5f, cr2); Y = Yn;
      float YY2 = Y2 * Y2; float T2 = __fmaf_rn(X2, X2, -YY2); float Yn2 = __fmaf_rn(X2, Y2, ci2); X2 = __fmaf_rn(T2, 0.5f, cr2); Y2 = Yn2;
    }
  }
  if (X == 12345.f) sink_f = Y + X2 + Y2;
}
// (d) 5-op + FSET/IADD3 pair counting (monotone regime)
__global__ void k_iter65(float cr2, float ci2, int n) {
  float X = threadIdx.x * 1e-3f, Y = blockIdx.x * 1e-4f; int cnt = 0;
  for (int i = 0; i < n; ++i) {
#pragma unroll 4
    for (int j = 0; j < 8; j += 2) {
      float YY = Y * Y; float M = __fmaf_rn(X, X, YY); int e0 = (M <= 16.f) ? -1 : 0;
      float T = __fmaf_rn(X, X, -YY); float Yn = __fmaf_rn(X, Y, ci2); X = __fmaf_rn(T, 0.5f, cr2); Y = Yn;
      YY = Y * Y; M = __fmaf_rn(X, X, YY); int e1 = (M <= 16.f) ? -1 : 0;
      T = __fmaf_rn(X, X, -YY); Yn = __fmaf_rn(X, Y, ci2); X = __fmaf_rn(T, 0.5f, cr2); Y = Yn;
      cnt = cnt - e0 - e1;
    }
  }
  if (X == 12345.f) { sink_f = Y; sink_i = cnt; }
}
// (e) FFMA with 3 distinct registers, independent chains
__global__ void k_ffma3(float a, float b, int n) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, y0 = a, y1 = b, y2 = a + b, y3 = a - b;
  float z0 = 1.f, z1 = 2.f, z2 = 3.f, z3 = 4.f;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      z0 = __fmaf_rn(x0, y0, z0); z1 = __fmaf_rn(x1, y1, z1); z2 = __fmaf_rn(x2, y2, z2); z3 = __fmaf_rn(x3, y3, z3);
    }
  }
  if (z0 == 12345.f) sink_f = z1 + z2 + z3;
}
// (f) FFMA with 1 distinct register pair + immediate
__global__ void k_ffmaimm(float a, float b, int n) {
  float z0 = threadIdx.x, z1 = z0 + 1, z2 = z0 + 2, z3 = z0 + 3;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      z0 = __fmaf_rn(z0, 0.999f, 0.5f); z1 = __fmaf_rn(z1, 0.999f, 0.5f); z2 = __fmaf_rn(z2, 0.999f, 0.5f); z3 = __fmaf_rn(z3, 0.999f, 0.5f);
    }
  }
  if (z0 == 12345.f) sink_f = z1 + z2 + z3;
}
// (g) DFMA chain-ish (fp64 pipe rate)
__global__ void k_dfma(double a, double b, int n) {
  double z0 = threadIdx.x, z1 = z0 + 1, z2 = z0 + 2, z3 = z0 + 3;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      z0 = __fma_rn(z0, a, b); z1 = __fma_rn(z1, a, b); z2 = __fma_rn(z2, a, b); z3 = __fma_rn(z3, a, b);
    }
  }
  if (z0 == 12345.) sink_f = (float)(z1 + z2 + z3);
}
// (h) fp64 4-op iteration
__global__ void k_diter4(double cr2, double ci2, int n) {
  double X = threadIdx.x * 1e-3, Y = blockIdx.x * 1e-4;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      double YY = Y * Y; double T = __fma_rn(X, X, -YY); double Yn = __fma_rn(X, Y, ci2); X = __fma_rn(T, 0.5, cr2); Y = Yn;
    }
  }
  if (X == 12345.) sink_f = (float)Y;
}


// ---- packed FP32 (sm_100: FFMA2 / FMUL2 via __ffma2_rn / __fmul2_rn) ----
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }
// (i) FFMA2 with immediate-like constant operands, 4 independent chains
__global__ void k_ffma2imm(float a, float b, int n) {
  float2 z0 = make_float2(threadIdx.x, threadIdx.x + 0.5f), z1 = make_float2(z0.x + 1, z0.y + 1),
         z2 = make_float2(z0.x + 2, z0.y + 2), z3 = make_float2(z0.x + 3, z0.y + 3);
  const float2 m = f2(0.999f), c = f2(0.5f);
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      z0 = __ffma2_rn(z0, m, c); z1 = __ffma2_rn(z1, m, c); z2 = __ffma2_rn(z2, m, c); z3 = __ffma2_rn(z3, m, c);
    }
  }
  if (z0.x == 12345.f) sink_f = z1.x + z2.y + z3.x + z0.y;
}
// (ii) two orbits packed, bare 4-op iteration: 4 packed instr per 2 pixel-iterations
__global__ void k_iter4p(float cr2, float ci2, int n) {
  float2 X = make_float2(threadIdx.x * 1e-3f, threadIdx.x * 1e-3f + 0.1f);
  float2 Y = make_float2(blockIdx.x * 1e-4f, blockIdx.x * 1e-4f - 0.1f);
  const float2 CR = f2(cr2), CI = f2(ci2), H = f2(0.5f);
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      float2 YY = __fmul2_rn(Y, Y); float2 T = __ffma2_rn(X, X, neg2(YY)); float2 Yn = __ffma2_rn(X, Y, CI);
      X = __ffma2_rn(T, H, CR); Y = Yn;
    }
  }
  if (X.x == 12345.f) sink_f = Y.x + Y.y + X.y;
}
// (iii) two orbits packed + per-iteration exact test (2 FSETP + 2 predicated IADD)
__global__ void k_iter7p(float cr2, float ci2, int n) {
  float2 X = make_float2(threadIdx.x * 1e-3f, threadIdx.x * 1e-3f + 0.1f);
  float2 Y = make_float2(blockIdx.x * 1e-4f, blockIdx.x * 1e-4f - 0.1f);
  const float2 CR = f2(cr2), CI = f2(ci2), H = f2(0.5f);
  int c0 = 0, c1 = 0; unsigned a0 = 1, a1 = 1;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      float2 YY = __fmul2_rn(Y, Y); float2 M = __ffma2_rn(X, X, YY);
      asm("{\n\t.reg .pred pa, pb;\n\tsetp.ne.u32 pa, %1, 0;\n\tsetp.le.and.f32 pb, %2, 0f41800000, pa;\n\tselp.u32 %1, 1, 0, pb;\n\t@pb add.s32 %0, %0, 1;\n\t}" : "+r"(c0), "+r"(a0) : "f"(M.x));
      asm("{\n\t.reg .pred pa, pb;\n\tsetp.ne.u32 pa, %1, 0;\n\tsetp.le.and.f32 pb, %2, 0f41800000, pa;\n\tselp.u32 %1, 1, 0, pb;\n\t@pb add.s32 %0, %0, 1;\n\t}" : "+r"(c1), "+r"(a1) : "f"(M.y));
      float2 T = __ffma2_rn(X, X, neg2(YY)); float2 Yn = __ffma2_rn(X, Y, CI);
      X = __ffma2_rn(T, H, CR); Y = Yn;
    }
  }
  if (X.x == 12345.f) { sink_f = Y.x + Y.y + X.y; sink_i = c0 + c1; }
}
// (iv) four orbits (two packed pairs), bare 4-op iteration
__global__ void k_iter4pp(float cr2, float ci2, int n) {
  float2 X = make_float2(threadIdx.x * 1e-3f, threadIdx.x * 1e-3f + 0.1f);
  float2 Y = make_float2(blockIdx.x * 1e-4f, blockIdx.x * 1e-4f - 0.1f);
  float2 X2 = make_float2(X.x + 0.05f, X.y - 0.05f), Y2 = make_float2(Y.x + 0.01f, Y.y + 0.02f);
  const float2 CR = f2(cr2), CI = f2(ci2), H = f2(0.5f);
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      float2 YY = __fmul2_rn(Y, Y); float2 YY2 = __fmul2_rn(Y2, Y2);
      float2 T = __ffma2_rn(X, X, neg2(YY)); float2 T2 = __ffma2_rn(X2, X2, neg2(YY2));
      float2 Yn = __ffma2_rn(X, Y, CI); float2 Yn2 = __ffma2_rn(X2, Y2, CI);
      X = __ffma2_rn(T, H, CR); X2 = __ffma2_rn(T2, H, CR); Y = Yn; Y2 = Yn2;
    }
  }
  if (X.x == 12345.f) sink_f = Y.x + Y.y + X.y + X2.x + Y2.y + X2.y + Y2.x;
}
// (v) FFMA2 chains interleaved 1:1 with independent integer adds (co-issue check)
__global__ void k_ffma2_int(float a, float b, int n) {
  float2 z0 = make_float2(threadIdx.x, threadIdx.x + 0.5f), z1 = make_float2(z0.x + 1, z0.y + 1),
         z2 = make_float2(z0.x + 2, z0.y + 2), z3 = make_float2(z0.x + 3, z0.y + 3);
  const float2 m = f2(0.999f), c = f2(0.5f);
  int i0 = threadIdx.x, i1 = i0 ^ 5, i2 = i0 ^ 9, i3 = i0 ^ 3;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      z0 = __ffma2_rn(z0, m, c); asm volatile("add.s32 %0, %0, 7;" : "+r"(i0));
      z1 = __ffma2_rn(z1, m, c); asm volatile("add.s32 %0, %0, 7;" : "+r"(i1));
      z2 = __ffma2_rn(z2, m, c); asm volatile("add.s32 %0, %0, 7;" : "+r"(i2));
      z3 = __ffma2_rn(z3, m, c); asm volatile("add.s32 %0, %0, 7;" : "+r"(i3));
    }
  }
  if (z0.x == 12345.f) { sink_f = z1.x + z2.y + z3.x + z0.y; sink_i = i0 + i1 + i2 + i3; }
}
// (vi) scalar FFMA chains interleaved 1:1 with integer adds (the scalar co-issue control)
__global__ void k_ffma_int(float a, float b, int n) {
  float z0 = threadIdx.x, z1 = z0 + 1, z2 = z0 + 2, z3 = z0 + 3;
  int i0 = threadIdx.x, i1 = i0 ^ 5, i2 = i0 ^ 9, i3 = i0 ^ 3;
  for (int i = 0; i < n; ++i) {
#pragma unroll 8
    for (int j = 0; j < 8; ++j) {
      z0 = __fmaf_rn(z0, 0.999f, 0.5f); asm volatile("add.s32 %0, %0, 7;" : "+r"(i0));
      z1 = __fmaf_rn(z1, 0.999f, 0.5f); asm volatile("add.s32 %0, %0, 7;" : "+r"(i1));
      z2 = __fmaf_rn(z2, 0.999f, 0.5f); asm volatile("add.s32 %0, %0, 7;" : "+r"(i2));
      z3 = __fmaf_rn(z3, 0.999f, 0.5f); asm volatile("add.s32 %0, %0, 7;" : "+r"(i3));
    }
  }
  if (z0 == 12345.f) { sink_f = z1 + z2 + z3; sink_i = i0 + i1 + i2 + i3; }
}

template <class F> void run(const char* name, F launch, double ops_per_thread_iter, int n, int blocks, int threads) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); cudaDeviceSynchronize();
  cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double thread_ops = (double)blocks * threads * n * 8 * ops_per_thread_iter;
  double warp_instr = thread_ops / 32;
  double smsp_cycles = ms * 1e-3 * 1965e6 * 148 * 4;
  printf("%-10s %8.3f ms  %.3f warp-instr/clk/SMSP (@1965MHz)  %.3e inner-iter/s\n", name, ms, warp_instr / smsp_cycles,
         (double)blocks * threads * n * 8 / (ms * 1e-3));
}
int main() {
  int n = N_IT, B = 148 * 8, T = 256;
  run("iter7", [&] { k_iter7<<<B, T>>>(0.1f, 0.2f, n); }, 7, n, B, T);
  run("iter4", [&] { k_iter4<<<B, T>>>(0.1f, 0.2f, n); }, 4, n, B, T);
  run("iter4x2", [&] { k_iter4x2<<<B, T>>>(0.1f, 0.2f, n); }, 8, n, B, T);
  run("iter6.5", [&] { k_iter65<<<B, T>>>(0.1f, 0.2f, n); }, 6.5, n, B, T);
  run("ffma3", [&] { k_ffma3<<<B, T>>>(0.1f, 0.2f, n); }, 4, n, B, T);
  run("ffmaimm", [&] { k_ffmaimm<<<B, T>>>(0.1f, 0.2f, n); }, 4, n, B, T);
  run("dfma", [&] { k_dfma<<<B, T>>>(0.1, 0.2, n / 4); }, 4, n / 4, B, T);
  run("diter4", [&] { k_diter4<<<B, T>>>(0.1, 0.2, n / 4); }, 4, n / 4, B, T);
  // packed: "inner-iter" counts thread-loop iterations; pixel-iter = 2x (iter4p/7p), 4x (4pp)
  run("ffma2imm", [&] { k_ffma2imm<<<B, T>>>(0.1f, 0.2f, n); }, 4, n, B, T);
  run("iter4p", [&] { k_iter4p<<<B, T>>>(0.1f, 0.2f, n); }, 4, n, B, T);
  run("iter7p", [&] { k_iter7p<<<B, T>>>(0.1f, 0.2f, n); }, 9, n, B, T);
  run("iter4pp", [&] { k_iter4pp<<<B, T>>>(0.1f, 0.2f, n); }, 8, n, B, T);
  run("ffma2int", [&] { k_ffma2_int<<<B, T>>>(0.1f, 0.2f, n); }, 8, n, B, T);
  run("ffmaint", [&] { k_ffma_int<<<B, T>>>(0.1f, 0.2f, n); }, 8, n, B, T);
  cudaError_t e = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(e));
}
