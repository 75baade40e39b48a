/*
 * c_api_demo.c -- the C ABI (include/ldpc_b200.h) driven from plain C, no Python or torch:
 * the paper's (14,7) tutorial code (Table I), priors computed the way serial.py:39-50 does,
 * one batch decoded through the host-buffer decoder, results printed; then the same frames from
 * their observations y (ldpc_decoder_decode_awgn_host: priors formed on the device with numpy's
 * exp algorithm).
 *
 *   make -C examples            # gcc, links paper_1609_01567_b200/_native/libldpc_b200.so
 *   ./examples/c_api_demo       # needs a GPU
 *
 * Output: one line per frame "frame k: success=S iterations=I estimate=<14 bits>", then the same
 * for the observation-input decode, prefixed "obs ".
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "ldpc_b200.h"

#define N 14
#define M 7
#define FRAMES 3

static const int32_t kRows[] = {5, 3, 2, 0, 4, 0, 5, 1, 6, 4, 1, 4, 3, 1, 0, 4, 2, 6, 5, 5, 4, 2, 1, 6, 0, 3, 1, 6, 3, 5, 0};
static const int32_t kCols[] = {0, 0, 0, 0, 1, 1, 2, 2, 3, 3, 3, 4, 4, 5, 5, 6, 6, 7, 7, 8, 8, 9, 9, 10, 10, 11, 11, 12, 12, 13, 13};

static int check(int rc, const char *what) {
    if (rc != LDPC_OK) {
        fprintf(stderr, "%s failed (%d): %s\n", what, rc, ldpc_last_error());
        exit(1);
    }
    return rc;
}

int main(void) {
    const int64_t nnz = (int64_t)(sizeof(kRows) / sizeof(kRows[0]));
    ldpc_graph *g = NULL;
    ldpc_decoder *d = NULL;
    check(ldpc_graph_create(N, M, nnz, kRows, kCols, NULL, &g), "ldpc_graph_create");
    check(ldpc_decoder_create(g, FRAMES, 0, &d), "ldpc_decoder_create");

    /* all-zero codeword sent as -1, a few bits flipped by "noise"; priors as serial.py:49 */
    const double sigma2 = 0.5;
    double y[FRAMES][N], p[FRAMES][N];
    for (int f = 0; f < FRAMES; f++)
        for (int j = 0; j < N; j++) {
            y[f][j] = -1.0 + ((j == f || j == f + 5) ? 1.6 : 0.1 * (double)((j * 7 + f) % 5 - 2));
            p[f][j] = 1.0 / (1.0 + exp((-2.0 * y[f][j]) / sigma2));
        }

    uint32_t est[FRAMES][(N + 31) / 32], syn[FRAMES][(M + 31) / 32];
    uint8_t success[FRAMES];
    int32_t iters[FRAMES];
    check(ldpc_decoder_decode_host(d, &p[0][0], FRAMES, 50, LDPC_FLAG_EARLY_STOP, &est[0][0], success, iters,
                                   &syn[0][0]),
          "ldpc_decoder_decode_host");
    for (int f = 0; f < FRAMES; f++) {
        printf("frame %d: success=%d iterations=%d estimate=", f, success[f], iters[f]);
        for (int j = 0; j < N; j++) putchar('0' + (int)((est[f][j >> 5] >> (j & 31)) & 1u));
        putchar('\n');
    }
    double s2[FRAMES];
    for (int f = 0; f < FRAMES; f++) s2[f] = sigma2;
    check(ldpc_decoder_decode_awgn_host(d, &y[0][0], s2, FRAMES, 50, LDPC_FLAG_EARLY_STOP, &est[0][0], success, iters,
                                        &syn[0][0]),
          "ldpc_decoder_decode_awgn_host");
    for (int f = 0; f < FRAMES; f++) {
        printf("obs frame %d: success=%d iterations=%d estimate=", f, success[f], iters[f]);
        for (int j = 0; j < N; j++) putchar('0' + (int)((est[f][j >> 5] >> (j & 31)) & 1u));
        putchar('\n');
    }
    ldpc_decoder_destroy(d);
    ldpc_graph_destroy(g);
    return 0;
}
