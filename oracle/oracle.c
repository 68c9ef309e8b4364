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
enum { ORC_SIGMOID = 0, ORC_TANH = 1, ORC_RELU = 2, ORC_SOFTMAX = 3 };
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
