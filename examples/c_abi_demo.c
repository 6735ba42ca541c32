/*
 * c_abi_demo.c -- libfractal through its C ABI alone: no Python, no torch, no CUDA
 * runtime calls in the caller.  Renders frames of the BASELINE cfg4 C-path (C on the
 * circle |C| = 0.7885, th_k = 2 pi k / n_frames) with julia_render_path_host, which
 * returns once the counts are in HOST memory (include/fractal.h), and writes them as raw
 * little-endian uint16 [n_frames][height][width] to a file.
 *
 *   cc -std=c11 -Iinclude examples/c_abi_demo.c -Lpaper_1611_03079_b200 -lfractal -lm \
 *      -Wl,-rpath,$PWD/paper_1611_03079_b200 -o c_abi_demo
 *   ./c_abi_demo WIDTH HEIGHT N_FRAMES MAX_ITER MODE OUT.bin     (MODE 0..3 = fr_mode)
 *
 * tests/test_gpu_parity.py::test_c_abi_demo_program runs it on the GPU box and compares
 * the file with the oracle; tests/test_abi.py::test_c_abi_demo_builds compiles it here.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "fractal.h"

int main(int argc, char** argv) {
    if (argc != 7) {
        fprintf(stderr, "usage: %s WIDTH HEIGHT N_FRAMES MAX_ITER MODE OUT.bin\n", argv[0]);
        return 2;
    }
    const int32_t w = atoi(argv[1]), h = atoi(argv[2]), n = atoi(argv[3]), mi = atoi(argv[4]);
    const fr_mode mode = (fr_mode)atoi(argv[5]);
    fr_complex* cs = malloc(sizeof(fr_complex) * (size_t)(n > 0 ? n : 1));
    uint16_t* counts = malloc(sizeof(uint16_t) * (size_t)w * (size_t)h * (size_t)(n > 0 ? n : 1));
    if (!cs || !counts) return 3;
    const double pi = 3.14159265358979323846;
    for (int32_t k = 0; k < n; ++k) {  /* DESIGN.md reading c-6 */
        const double th = 2.0 * pi * k / n;
        cs[k].re = 0.7885 * cos(th);
        cs[k].im = 0.7885 * sin(th);
    }
    /* SPEC default Julia viewport (reading c-4): centre 0, real span 4, square pixels */
    const fr_window win = {0.0, 0.0, 2.0, 2.0 * (double)h / (double)w};
    const fr_status st = julia_render_path_host(cs, n, win, w, h, mi, mode, 2, counts, NULL);
    if (st != FR_OK) {
        fprintf(stderr, "julia_render_path_host: %s (cuda error %d)\n", fr_status_str(st),
                fr_last_cuda_error());
        return 1;
    }
    FILE* f = fopen(argv[6], "wb");
    if (!f) return 4;
    const size_t total = (size_t)w * (size_t)h * (size_t)n;
    if (fwrite(counts, sizeof(uint16_t), total, f) != total) return 5;
    fclose(f);
    uint64_t sum = 0;
    for (size_t i = 0; i < total; ++i) sum += counts[i];
    printf("%s: %d frames of %dx%d, max_iter %d, sum of counts %llu\n", fr_version(), n, w, h,
           mi, (unsigned long long)sum);
    free(cs);
    free(counts);
    return 0;
}
