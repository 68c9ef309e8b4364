/* oracle/oracle.c — plain, slow, single-threaded CPU oracle of the PNN hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load or call this
 * library.  It shares no code, header, table or generator with the CUDA
 * path (paper_2304_09590_b200/), and neither side imports the other; the
 * only input both sides share is datagen/ (seeded draws, no method math).
 *
 * What it computes (arXiv 2304.09590, "Parallel Neural Networks in Golang"):
 *   forward            PAPER.md:71-97   (§3, Eqs.1-5)        oracle_body.h orc_forward
 *   cost               PAPER.md:100-103 (Eq.6) / R11         oracle_body.h orc_cost
 *   deltas             PAPER.md:104-123 (Eqs.7-11)           oracle_body.h deltas
 *   SGD / mini-batch   PAPER.md:125-134 (Eqs.12-13)          oracle_body.h orc_train
 *   slicing            PAPER.md:166-169, 226 (§4.2-4.3)      orc_shard_bounds
 *   averaging merge    PAPER.md:170-172, 233-238             orc_merge
 *   readout            PAPER.md:97                           oracle_body.h orc_predict
 *   init               PAPER.md:209-213 (+ variants, R15)    orc_init
 * Readings R1-R26 are listed in DESIGN.md §3.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no -ffast-math): every
 * multiply and add is rounded separately, in ascending index order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAX_LAYERS 16
enum { ORC_SIGMOID = 0, ORC_TANH = 1, ORC_RELU = 2, ORC_SOFTMAX = 3, ORC_LEAKY_RELU = 4 };
enum { ORC_INIT_NORMAL = 0, ORC_INIT_UNIFORM = 1, ORC_INIT_XAVIER = 2, ORC_INIT_HE = 3 };

/* ---- fp32 instantiation ------------------------------------------------ */
#define REAL float
#define SUF _f32
#define EXP expf
#define TANH tanhf
#include "oracle_body.h"
#undef REAL
#undef SUF
#undef EXP
#undef TANH

/* ---- fp64 instantiation ------------------------------------------------ */
#define REAL double
#define SUF _f64
#define EXP exp
#define TANH tanh
#include "oracle_body.h"
#undef REAL
#undef SUF
#undef EXP
#undef TANH

/* ---- bf16 mini-batch variant (a10; north_star "bf16 weights and activations
 * with fp32 accumulate and fp32 master weights"; reading R25) ---------------
 * bf16(v): round-to-nearest-even to the 8-bit-mantissa bfloat16, returned as a
 * float.  NaN is kept quiet.                                                 */
float orc_bf16_round(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu)) {
        u |= 0x00400000u;                       /* quiet NaN */
    } else {
        u += 0x7fffu + ((u >> 16) & 1u);        /* RNE on the low 16 bits */
    }
    u &= 0xffff0000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

/* Mini-batch GD (the gradients of the batch are averaged before
 * one update; short last batch averaged over its size, R14) with the rounding
 * points of reading R25, for one network over rows X[0..n):
 *   per step:  Wb^l = bf16(W^l) (fp32 master W), weights fixed over the batch;
 *   forward:   xb^0 = bf16(x); z^l_k = Σ_j Wb^l_kj xb^{l-1}_j (fp32, ascending j) + b^l_k;
 *              x^l = φ(z^l) in fp32 (softmax max-subtracted, R4); hidden layers
 *              pass xb^l = bf16(x^l) on;
 *   deltas:    δ^L = x^L - e (softmax+CE) or (x^L - e)⊙φ'(x^L); δb = bf16(δ);
 *              δ^l_j = (Σ_k Wb^{l+1}_kj δb^{l+1}_k) ⊙ φ'(x^l_j) (pre-update weights, R6);
 *   gradient:  G^l_kj += δb^l_k xb^{l-1}_j (fp32), gb^l_k += δ^l_k (fp32);
 *   update:    W ← W - η·(G / B_actual), b ← b - η·(gb / B_actual)  (fp32).      */
int orc_train_bf16(const int* layers, int L, const int* act, float* params, const float* X,
                   const int* y, long n, float lr, int epochs, int batch) {
    long woff[ORC_MAX_LAYERS + 1], noff[ORC_MAX_LAYERS + 1];
    long w = 0, nn = 0;
    for (int l = 1; l <= L; ++l) {
        woff[l] = w;
        noff[l] = nn;
        w += (long)layers[l] * layers[l - 1] + layers[l];
        nn += layers[l];
    }
    const long P = w, tot = nn;
    const int d0 = layers[0];
    float* Wb = (float*)malloc(sizeof(float) * P);
    float* G = (float*)malloc(sizeof(float) * P);
    float* xs = (float*)malloc(sizeof(float) * tot);   /* x^l (fp32)           */
    float* xb = (float*)malloc(sizeof(float) * tot);   /* bf16(x^l)            */
    float* ds = (float*)malloc(sizeof(float) * tot);   /* δ^l (fp32)           */
    float* db = (float*)malloc(sizeof(float) * tot);   /* bf16(δ^l)            */
    float* x0b = (float*)malloc(sizeof(float) * d0);
    if (!Wb || !G || !xs || !xb || !ds || !db || !x0b) {
        free(Wb); free(G); free(xs); free(xb); free(ds); free(db); free(x0b);
        return -1;
    }
    if (batch < 1) batch = 1;
    for (int e = 0; e < epochs; ++e) {
        for (long t0 = 0; t0 < n; t0 += batch) {
            const long bsz = (n - t0 < batch) ? (n - t0) : batch;
            for (long i = 0; i < P; ++i) { Wb[i] = orc_bf16_round(params[i]); G[i] = 0.f; }
            for (long t = t0; t < t0 + bsz; ++t) {
                for (int j = 0; j < d0; ++j) x0b[j] = orc_bf16_round(X[t * d0 + j]);
                /* forward */
                for (int l = 1; l <= L; ++l) {
                    const int nin = layers[l - 1], nout = layers[l];
                    const float* W = Wb + woff[l];
                    const float* b = params + woff[l] + (long)nout * nin;   /* fp32 bias */
                    const float* xin = (l == 1) ? x0b : xb + noff[l - 1];
                    float* x = xs + noff[l];
                    for (int k = 0; k < nout; ++k) {
                        float acc = 0.f;
                        for (int j = 0; j < nin; ++j) acc += W[(long)k * nin + j] * xin[j];
                        x[k] = acc + b[k];                                  /* z, then φ */
                    }
                    if (act[l - 1] == ORC_SOFTMAX) {
                        float m = x[0];
                        for (int k = 1; k < nout; ++k) if (x[k] > m) m = x[k];
                        float s = 0.f;
                        for (int k = 0; k < nout; ++k) { x[k] = expf(x[k] - m); s += x[k]; }
                        for (int k = 0; k < nout; ++k) x[k] = x[k] / s;
                    } else {
                        for (int k = 0; k < nout; ++k) x[k] = act_scalar_f32(act[l - 1], x[k]);
                    }
                    for (int k = 0; k < nout; ++k) xb[noff[l] + k] = orc_bf16_round(x[k]);
                }
                /* deltas */
                {
                    const int nL = layers[L];
                    const float* xo = xs + noff[L];
                    for (int i = 0; i < nL; ++i) {
                        const float ev = (i == y[t]) ? 1.f : 0.f;
                        float d = (act[L - 1] == ORC_SOFTMAX)
                                      ? xo[i] - ev
                                      : (xo[i] - ev) * act_deriv_from_x_f32(act[L - 1], xo[i]);
                        ds[noff[L] + i] = d;
                        db[noff[L] + i] = orc_bf16_round(d);
                    }
                    for (int l = L - 1; l >= 1; --l) {
                        const int nh = layers[l], nn2 = layers[l + 1];
                        const float* Wn = Wb + woff[l + 1];
                        for (int j = 0; j < nh; ++j) {
                            float acc = 0.f;
                            for (int k = 0; k < nn2; ++k) acc += Wn[(long)k * nh + j] * db[noff[l + 1] + k];
                            const float d = acc * act_deriv_from_x_f32(act[l - 1], xs[noff[l] + j]);
                            ds[noff[l] + j] = d;
                            db[noff[l] + j] = orc_bf16_round(d);
                        }
                    }
                }
                /* gradient sums */
                for (int l = 1; l <= L; ++l) {
                    const int nin = layers[l - 1], nout = layers[l];
                    float* Gl = G + woff[l];
                    float* gb = Gl + (long)nout * nin;
                    const float* xin = (l == 1) ? x0b : xb + noff[l - 1];
                    for (int k = 0; k < nout; ++k) {
                        const float dk = db[noff[l] + k];
                        for (int j = 0; j < nin; ++j) Gl[(long)k * nin + j] += dk * xin[j];
                        gb[k] += ds[noff[l] + k];
                    }
                }
            }
            for (long i = 0; i < P; ++i) params[i] -= lr * (G[i] / (float)bsz);
        }
    }
    free(Wb); free(G); free(xs); free(xb); free(ds); free(db); free(x0b);
    return 0;
}

/* ---- init (reading R15) ------------------------------
 * Counter-based: uniform u(seed, layer, kind, index, s) with
 *   ctr = (layer << 48) ^ (kind << 47) ^ (2*index + s)
 *   h   = mix(seed * 0x9E3779B97F4A7C15 + mix(ctr + 0x632BE59BD9B4E019))
 *   u   = (h >> 11) * 2^-53                     ∈ [0, 1)
 * with mix = the SplitMix64 finaliser.  N(0,1) by Box–Muller in double:
 *   z = sqrt(-2 ln(1 - u(s=0))) * cos(2π u(s=1)).
 * The paper's rand.NormFloat64 seeded by the clock is
 * replaced by this explicit seed so both sides draw the same numbers.     */
static uint64_t orc_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double orc_uniform(uint64_t seed, int layer, int kind, int64_t index, int s) {
    uint64_t ctr = ((uint64_t)layer << 48) ^ ((uint64_t)kind << 47) ^ (uint64_t)(2 * index + s);
    uint64_t h = orc_mix(seed * 0x9E3779B97F4A7C15ULL + orc_mix(ctr + 0x632BE59BD9B4E019ULL));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}

double orc_normal(uint64_t seed, int layer, int kind, int64_t index) {
    double u1 = orc_uniform(seed, layer, kind, index, 0);
    double u2 = orc_uniform(seed, layer, kind, index, 1);
    return sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
}

/* Weights: N(0,1) | U[-0.5,0.5) | N(0, 2/(fan_in+fan_out)) | N(0, 2/fan_in);
 * biases:  N(0,1) | U[-0.5,0.5) | 0 | 0.   (fan_in = n_{l-1}, fan_out = n_l)
 * Returns 0, or -1 for an unknown init code.                               */
int orc_init(const int* layers, int L, int init, uint64_t seed, float* params) {
    float* p = params;
    for (int l = 1; l <= L; ++l) {
        int nin = layers[l - 1], nout = layers[l];
        long nw = (long)nin * nout;
        double sigma = 1.0;
        if (init == ORC_INIT_XAVIER) sigma = sqrt(2.0 / (double)(nin + nout));
        else if (init == ORC_INIT_HE) sigma = sqrt(2.0 / (double)nin);
        else if (init != ORC_INIT_NORMAL && init != ORC_INIT_UNIFORM) return -1;
        for (long i = 0; i < nw; ++i) {
            if (init == ORC_INIT_UNIFORM) p[i] = (float)(orc_uniform(seed, l, 0, i, 0) - 0.5);
            else p[i] = (float)(sigma * orc_normal(seed, l, 0, i));
        }
        float* b = p + nw;
        for (long k = 0; k < nout; ++k) {
            if (init == ORC_INIT_NORMAL) b[k] = (float)orc_normal(seed, l, 1, k);
            else if (init == ORC_INIT_UNIFORM) b[k] = (float)(orc_uniform(seed, l, 1, k, 0) - 0.5);
            else b[k] = 0.0f;
        }
        p = b + nout;
    }
    return 0;
}

long orc_param_count(const int* layers, int L) {
    long P = 0;
    for (int l = 1; l <= L; ++l) P += (long)layers[l] * layers[l - 1] + layers[l];
    return P;
}

/* ---- slicing ("divided into as many slices as there are
 * networks"; :226 "the dataset is split according to the amount of CNs").
 * Reading R17: contiguous; slice i has floor(N/K) + [i < N mod K] rows.    */
void orc_shard_bounds(long N, int K, long* start, long* count) {
    long base = N / K, rem = N % K, s = 0;
    for (int i = 0; i < K; ++i) {
        long m = base + (i < rem ? 1 : 0);
        start[i] = s;
        count[i] = m;
        s += m;
    }
}

/* ---- averaging merge ("the average of all weights …
 * For the biases the same procedure"; :235-238 "weights, and biases are
 * added onto the PNN … scaled by the number of CNs").  Reading R18: sum
 * children in ascending order in double (exact for K identical fp32 clones,
 * K ≤ 2^29), then divide by K, round once to fp32.                          */
void orc_merge(const float* children, int K, long P, float* out) {
    for (long i = 0; i < P; ++i) {
        double s = 0.0;
        for (int c = 0; c < K; ++c) s += (double)children[(long)c * P + i];
        out[i] = (float)(s / (double)K);
    }
}
