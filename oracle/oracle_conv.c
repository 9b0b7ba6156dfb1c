/*
 * oracle_conv.c -- TEST INFRASTRUCTURE (oracle), not part of the product path.
 *
 * Plain fp64 2-D convolution over one sample in NHWC layout, written out as
 * its definition (no blocking, no im2col, no reordering):
 *
 *   y[ho][wo][o] = b[o] + sum_{r<k} sum_{s<k} sum_{c<C}
 *                  w[o][r][s][c] * x[ho*stride - pad + r][wo*stride - pad + s][c]
 *
 * with out-of-range input positions contributing zero (zero padding).
 * This is the `conv2d` tensor operator of the paper's DAG view of a DNN
 * (Sec. 2.2 "kernel operators (e.g. convolutional operator
 * and dense operator)").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library (through oracle/).
 * Pinned against torch.nn.functional.conv2d (fp64) in tests/test_oracle.py.
 */
#include <stddef.h>

void oracle_conv2d_nhwc(const double* x, int H, int W, int C,
                        const double* w, int Co, int k, int stride, int pad,
                        const double* b, double* y)
{
    const int Ho = (H + 2 * pad - k) / stride + 1;
    const int Wo = (W + 2 * pad - k) / stride + 1;
    for (int ho = 0; ho < Ho; ++ho) {
        for (int wo = 0; wo < Wo; ++wo) {
            for (int o = 0; o < Co; ++o) {
                double acc = b ? b[o] : 0.0;
                for (int r = 0; r < k; ++r) {
                    const int hi = ho * stride - pad + r;
                    if (hi < 0 || hi >= H) continue;
                    for (int s = 0; s < k; ++s) {
                        const int wi = wo * stride - pad + s;
                        if (wi < 0 || wi >= W) continue;
                        const double* xp = x + ((size_t)hi * W + wi) * C;
                        const double* wp = w + (((size_t)o * k + r) * k + s) * C;
                        for (int c = 0; c < C; ++c) acc += wp[c] * xp[c];
                    }
                }
                y[((size_t)ho * Wo + wo) * Co + o] = acc;
            }
        }
    }
}
