/* oracle/oracle_body.h — TEST INFRASTRUCTURE ONLY (see oracle/oracle.c header).
 *
 * Included twice by oracle.c, once with REAL=float (SUF=_f32) and once with
 * REAL=double (SUF=_f64): the plain C spelling of "templated on float/double".
 * Every loop runs in ascending index order; there is no blocking, fusion or
 * reordering beyond what the paper's equations state.
 *
 * Parameter layout (one network): for l = 1..L: W^l row-major [n_l][n_{l-1}],
 * then b^l [n_l].  (mirrors SPEC.md:251's dump order.)
 */

#define CAT_(a, b) a##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SUF)

/* φ (Eqs.3-5; sigmoid/tanh named in §5.2).   */
static REAL FN(act_scalar)(int act, REAL z) {
    switch (act) {
    case ORC_SIGMOID: return (REAL)1 / ((REAL)1 + EXP(-z));
    case ORC_TANH:    return TANH(z);
    case ORC_RELU:    return z >= (REAL)0 ? z : (REAL)0;      /* Eq.4: z>=0 → z */
    /* leaky ReLU (§5.2; slope unstated → 0.01, reading R30)   */
    case ORC_LEAKY_RELU: return z >= (REAL)0 ? z : (REAL)0.01 * z;
    default:          return z;
    }
}

/* φ'(z) evaluated from the stored activation x = φ(z) (reading R10; R9: ReLU'(0)=0).
 * Eq.11 needs "the first derivative of the activation".  */
static REAL FN(act_deriv_from_x)(int act, REAL x) {
    switch (act) {
    case ORC_SIGMOID: return x * ((REAL)1 - x);
    case ORC_TANH:    return (REAL)1 - x * x;
    case ORC_RELU:    return x > (REAL)0 ? (REAL)1 : (REAL)0;
    case ORC_LEAKY_RELU: return x > (REAL)0 ? (REAL)1 : (REAL)0.01;   /* R30: left slope at 0 (as R9) */
    default:          return (REAL)1;
    }
}

/* Forward pass of one sample (Eqs.2-5).
 * z[off_l + k] = Σ_j W^l_kj x^{l-1}_j + b^l_k   (bias added once: reading R1)
 * x[off_l + k] = φ_l(z)                         (softmax: max-subtracted, R4)  */
void FN(orc_forward)(const int* layers, int L, const int* act, const REAL* params,
                     const REAL* x0, REAL* zs, REAL* xs) {
    const REAL* p = params;
    const REAL* xin = x0;
    long off = 0;
    for (int l = 1; l <= L; ++l) {
        int nin = layers[l - 1], nout = layers[l];
        const REAL* W = p;
        const REAL* b = p + (long)nout * nin;
        REAL* z = zs + off;
        REAL* x = xs + off;
        for (int k = 0; k < nout; ++k) {
            REAL acc = 0;
            for (int j = 0; j < nin; ++j) acc += W[(long)k * nin + j] * xin[j];
            z[k] = acc + b[k];
        }
        if (act[l - 1] == ORC_SOFTMAX) {
            REAL m = z[0];
            for (int k = 1; k < nout; ++k) if (z[k] > m) m = z[k];
            REAL s = 0;
            for (int k = 0; k < nout; ++k) { x[k] = EXP(z[k] - m); s += x[k]; }
            for (int k = 0; k < nout; ++k) x[k] = x[k] / s;
        } else {
            for (int k = 0; k < nout; ++k) x[k] = FN(act_scalar)(act[l - 1], z[k]);
        }
        p = b + nout;
        xin = x;
        off += nout;
    }
}

/* Cost of one sample.  Softmax output: cross entropy C = -Σ e_i ln x_i
 * (Eq.6; natural log, reading R3).  Otherwise
 * C = ½ Σ (x_i - e_i)^2 (reading R11: the MSE of BASELINE C1/C2).          */
double FN(orc_cost)(const int* layers, int L, const int* act, const REAL* params,
                    const REAL* x0, int label, REAL* scratch) {
    long tot = 0;
    for (int l = 1; l <= L; ++l) tot += layers[l];
    REAL* zs = scratch;
    REAL* xs = scratch + tot;
    FN(orc_forward)(layers, L, act, params, x0, zs, xs);
    const REAL* out = xs + tot - layers[L];
    double c = 0;
    if (act[L - 1] == ORC_SOFTMAX) {
        c = -log((double)out[label]);
    } else {
        for (int i = 0; i < layers[L]; ++i) {
            double e = (i == label) ? 1.0 : 0.0;
            c += 0.5 * ((double)out[i] - e) * ((double)out[i] - e);
        }
    }
    return c;
}

/* Deltas of one sample (Eqs.9-11), after orc_forward.
 * δ^L: softmax+CE → x - e (Eq.10); other output → (x - e) ⊙ φ'(z) (Eq.9 with R11).
 * δ^l = ((W^{l+1})^T δ^{l+1}) ⊙ φ'_l(z^l), l = L-1..1, with the weights as
 * they are before this sample's update (reading R6).                        */
static void FN(deltas)(const int* layers, int L, const int* act, const REAL* params,
                       const REAL* xs, REAL* ds, int label, const long* woff, const long* noff) {
    int nL = layers[L];
    const REAL* xo = xs + noff[L];
    REAL* dL = ds + noff[L];
    for (int i = 0; i < nL; ++i) {
        REAL e = (i == label) ? (REAL)1 : (REAL)0;
        if (act[L - 1] == ORC_SOFTMAX) dL[i] = xo[i] - e;
        else dL[i] = (xo[i] - e) * FN(act_deriv_from_x)(act[L - 1], xo[i]);
    }
    for (int l = L - 1; l >= 1; --l) {
        int n = layers[l], nn = layers[l + 1];
        const REAL* Wn = params + woff[l + 1];
        const REAL* dn = ds + noff[l + 1];
        REAL* d = ds + noff[l];
        const REAL* x = xs + noff[l];
        for (int j = 0; j < n; ++j) {
            REAL acc = 0;
            for (int k = 0; k < nn; ++k) acc += Wn[(long)k * n + j] * dn[k];
            d[j] = acc * FN(act_deriv_from_x)(act[l - 1], x[j]);
        }
    }
}

static void FN(offsets)(const int* layers, int L, long* woff, long* noff) {
    long w = 0, n = 0;
    for (int l = 1; l <= L; ++l) {
        woff[l] = w;               /* W^l at woff[l], b^l at woff[l] + n_l*n_{l-1} */
        noff[l] = n;               /* per-neuron arrays (z, x, δ) of layer l at noff[l] */
        w += (long)layers[l] * layers[l - 1] + layers[l];
        n += layers[l];
    }
}

/* Train ONE network sequentially over rows X[0..n) (one child network on its
 * slice, "Each child-network learns only a slice"), for `epochs`
 * passes in index order (reading R8: no shuffling).
 * batch == 1: stochastic GD, update after every instance;
 *   per sample: forward (Eqs.2-5) → δ (Eqs.9-11) → g_k = η δ_k;
 *   W_kj ← W_kj - g_k x_j ; b_k ← b_k - g_k (Eqs.12-13, "applied by adding", R5).
 * batch  > 1: mini-batch GD; with the weights fixed over the batch, the
 *   per-instance gradients δ x^T, δ are summed, averaged over the batch's
 *   actual size ("the gradients of all instances are averaged before the
 *   updates"; short last batch kept, R14), then W ← W - η·avg.
 * Returns 0, or -1 on allocation failure.                                  */
int FN(orc_train)(const int* layers, int L, const int* act, REAL* params,
                  const REAL* X, const int* y, long n, REAL lr, int epochs, int batch) {
    long woff[ORC_MAX_LAYERS + 1], noff[ORC_MAX_LAYERS + 1];
    FN(offsets)(layers, L, woff, noff);
    long tot = noff[L] + layers[L];
    long P = woff[L] + (long)layers[L] * layers[L - 1] + layers[L];
    REAL* zs = (REAL*)malloc(sizeof(REAL) * tot);
    REAL* xs = (REAL*)malloc(sizeof(REAL) * tot);
    REAL* ds = (REAL*)malloc(sizeof(REAL) * tot);
    REAL* gsum = batch > 1 ? (REAL*)calloc(P, sizeof(REAL)) : NULL;
    if (!zs || !xs || !ds || (batch > 1 && !gsum)) {
        free(zs); free(xs); free(ds); free(gsum);
        return -1;
    }
    int d0 = layers[0];
    for (int e = 0; e < epochs; ++e) {
        if (batch <= 1) {
            for (long t = 0; t < n; ++t) {
                const REAL* x0 = X + t * d0;
                FN(orc_forward)(layers, L, act, params, x0, zs, xs);
                FN(deltas)(layers, L, act, params, xs, ds, y[t], woff, noff);
                for (int l = 1; l <= L; ++l) {
                    int nin = layers[l - 1], nout = layers[l];
                    REAL* W = params + woff[l];
                    REAL* b = W + (long)nout * nin;
                    const REAL* xin = (l == 1) ? x0 : xs + noff[l - 1];
                    const REAL* d = ds + noff[l];
                    for (int k = 0; k < nout; ++k) {
                        REAL g = lr * d[k];
                        for (int j = 0; j < nin; ++j) W[(long)k * nin + j] -= g * xin[j];
                        b[k] -= g;
                    }
                }
            }
        } else {
            for (long t0 = 0; t0 < n; t0 += batch) {
                long bsz = (n - t0 < batch) ? (n - t0) : batch;
                for (long i = 0; i < P; ++i) gsum[i] = 0;
                for (long t = t0; t < t0 + bsz; ++t) {
                    const REAL* x0 = X + t * d0;
                    FN(orc_forward)(layers, L, act, params, x0, zs, xs);
                    FN(deltas)(layers, L, act, params, xs, ds, y[t], woff, noff);
                    for (int l = 1; l <= L; ++l) {
                        int nin = layers[l - 1], nout = layers[l];
                        REAL* G = gsum + woff[l];
                        REAL* gb = G + (long)nout * nin;
                        const REAL* xin = (l == 1) ? x0 : xs + noff[l - 1];
                        const REAL* d = ds + noff[l];
                        for (int k = 0; k < nout; ++k) {
                            for (int j = 0; j < nin; ++j) G[(long)k * nin + j] += d[k] * xin[j];
                            gb[k] += d[k];
                        }
                    }
                }
                for (long i = 0; i < P; ++i) params[i] -= lr * (gsum[i] / (REAL)bsz);
            }
        }
    }
    free(zs); free(xs); free(ds); free(gsum);
    return 0;
}

/* Readout ("each class is represented by one neuron"; reading
 * R19): label = argmax_k z^L_k of the forward pass, ties → lowest index.
 * logits_out (nullable) receives z^L [n][n_L].                               */
int FN(orc_predict)(const int* layers, int L, const int* act, const REAL* params,
                    const REAL* X, long n, int* labels, REAL* logits_out) {
    long woff[ORC_MAX_LAYERS + 1], noff[ORC_MAX_LAYERS + 1];
    FN(offsets)(layers, L, woff, noff);
    long tot = noff[L] + layers[L];
    REAL* zs = (REAL*)malloc(sizeof(REAL) * tot);
    REAL* xs = (REAL*)malloc(sizeof(REAL) * tot);
    if (!zs || !xs) { free(zs); free(xs); return -1; }
    int nL = layers[L];
    for (long t = 0; t < n; ++t) {
        FN(orc_forward)(layers, L, act, params, X + t * layers[0], zs, xs);
        const REAL* z = zs + noff[L];
        int best = 0;
        for (int k = 1; k < nL; ++k) if (z[k] > z[best]) best = k;
        labels[t] = best;
        if (logits_out) for (int k = 0; k < nL; ++k) logits_out[t * nL + k] = z[k];
    }
    free(zs); free(xs);
    return 0;
}

#undef FN
#undef CAT
#undef CAT_
