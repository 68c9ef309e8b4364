/* include/pnn.h — C ABI of the B200-native PNN hot path.
 *
 * The method: arXiv 2304.09590, "Parallel Neural Networks in Golang"
 * (Kalwarowskyj & Schikuta), §3-§4:
 *   - K identical-architecture child networks (CNs) are built by cloning one
 *     random network (reading R16),
 *   - the training set is split into K contiguous slices, one per CN
 *     (R17),
 *   - every CN trains independently by backpropagation with stochastic
 *     (per-instance) gradient descent (Eqs.1-13, 225-231),
 *   - the CNs are fused into one PNN by averaging all weights and biases
 *     (PAPER.md:170-172, 233-238),
 *   - the PNN (or a CN) classifies by the output neuron with the highest
 *     value (R19).
 * SNN and PNN are interchangeable (the TrainableNetwork interface,
 * PAPER.md:187-191): a handle with n_subnets = 1 is the sequential network.
 *
 * Conventions for every entry point
 *   - Returns pnn_status; no C++ exception crosses the ABI.
 *   - Everything is validated before anything is enqueued.  On a validation
 *     error the call returns a code, sets pnn_last_error(), and the handle
 *     stays usable.  A CUDA or NCCL failure poisons the handle: every later
 *     call except pnn_last_error/pnn_destroy returns PNN_ERR_STATE.
 *   - Device pointers are caller-owned, on the handle's device (the current
 *     CUDA device at pnn_create), contiguous, and must stay valid until the
 *     work enqueued on `cuda_stream` has completed.  Host pointers are only
 *     read/written during the call.
 *   - `cuda_stream` is a cudaStream_t (NULL = the legacy default stream).
 *     Calls are stream-ordered and asynchronous unless stated otherwise.
 *   - A handle is driven by one host thread at a time.
 *
 * Parameter layout (pnn_get_params / pnn_set_params, device slabs): for
 * l = 1..L, W^l row-major [n_l][n_{l-1}] (W^l_kj = weight from neuron j of
 * layer l-1 to neuron k of layer l, Eq.2), then b^l [n_l];
 * fp32, little endian.  P_total = Σ_l n_l·n_{l-1} + n_l  (pnn_param_count).
 */
#ifndef PNN_H_
#define PNN_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pnn_net_s* pnn_net;   /* opaque; owns all of its device state */

typedef enum {
    PNN_OK = 0,
    PNN_ERR_INVALID = 1,   /* bad argument (enum, size, pointer, lr, index)      */
    PNN_ERR_SHAPE = 2,     /* n_floats / layer shape mismatch                    */
    PNN_ERR_DATA = 3,      /* too few rows: some CN would get an empty slice     */
    PNN_ERR_STATE = 4,     /* poisoned handle, or call not valid in this state   */
    PNN_ERR_CUDA = 5,      /* CUDA runtime error (poisons the handle)            */
    PNN_ERR_NCCL = 6,      /* NCCL error (poisons the handle)                    */
    PNN_ERR_OOM = 7        /* device allocation failed                           */
} pnn_status;

/* Activation φ per layer (Eqs.4-5; §5.2).
 * The loss follows from the output activation: PNN_SOFTMAX → cross entropy
 * (Eq.6; δ^L = x - e, Eq.10); any other output → C = ½Σ(x - e)² (reading
 * R11; δ^L = (x - e)⊙φ'(z^L), Eq.9).  PNN_SOFTMAX is only valid on the last
 * layer.                                                                    */
enum { PNN_SIGMOID = 0, PNN_TANH = 1, PNN_RELU = 2, PNN_SOFTMAX = 3,
       PNN_LEAKY_RELU = 4   /* φ(z) = z ≥ 0 ? z : 0.01·z (PAPER.md:281 names it, §5.2;
                               slope unstated → 0.01, DESIGN.md §3 R30)          */ };

/* Initialisation (reading R15).  Weights / biases:
 *   NORMAL         N(0,1) / N(0,1)          (the paper's NormFloat64)
 *   UNIFORM        U[-0.5,0.5) / U[-0.5,0.5)
 *   XAVIER_NORMAL  N(0, 2/(n_{l-1}+n_l)) / 0
 *   HE_NORMAL      N(0, 2/n_{l-1}) / 0
 * drawn from a counter-based generator of (seed, layer, weight|bias, index)
 * (DESIGN.md §3 R15), then cloned into every CN (R16).                      */
enum { PNN_INIT_NORMAL = 0, PNN_INIT_UNIFORM = 1, PNN_INIT_XAVIER_NORMAL = 2,
       PNN_INIT_HE_NORMAL = 3 };

/* Precision of the mini-batch variant (pnn_set_minibatch). */
enum { PNN_FP32 = 0, PNN_BF16 = 1 };

/* Training kernel selection (pnn_set_kernel). */
enum { PNN_KERNEL_AUTO = 0,      /* fastest kernel valid for the shape          */
       PNN_KERNEL_REFERENCE = 1, /* one CTA per CN, weights in global memory    */
       PNN_KERNEL_RESIDENT = 2,  /* persistent per-CN kernel, on-chip weights
                                    (2-layer nets, 768 < D <= 784, O = 10,
                                    H <= 256); variants (pnn_set_variant):
                                    TMEM (one SM per CN, W1 in registers +
                                    tensor memory, H <= 128), v8 (W1 in the
                                    registers of a cluster, chain on rotating
                                    warp pairs) and v10 (chain on its own CTA).
                                    AUTO: v10 when every concurrently trained
                                    CN fits with its chain CTA (K_local or
                                    slots x 3 <= 120, H <= 128), else TMEM
                                    (H <= 128), else v8.                       */
       PNN_KERNEL_TC_BF16 = 3,   /* bf16 mini-batch on tcgen05 GEMMs; chosen by
                                    pnn_set_minibatch(.., PNN_BF16), reported
                                    by pnn_kernel_info, not settable         */
       PNN_KERNEL_MB_F32 = 4,    /* fp32 mini-batch step kernels (D-H-O nets,
                                    batch 2..64; AUTO picks it, REFERENCE
                                    opts out), reported, not settable        */
       PNN_KERNEL_MB_RESIDENT = 6, /* fp32 mini-batch as one persistent launch per
                                    epoch: W1 in the registers of a cluster of
                                    ceil(H/32) CTAs (k_mbres.cu; D-H-O nets,
                                    768 < D <= 784, H <= 256, O <= 16, batch
                                    2..64).  AUTO's first choice for fp32
                                    mini-batch; environment PNN_MBRES=0 falls
                                    back to _MB_F32; reported, not settable   */
       PNN_KERNEL_CLUSTER = 5    /* per-sample SGD, any depth, weights resident
                                    in the shared memory of a cluster of <= 8
                                    CTAs (AUTO's choice when the resident
                                    kernel does not cover the shape, e.g. C3).
                                    3-layer nets with 768 < D <= 784, H1 <= 320,
                                    H2 <= 120, O <= 16 run its deep variant
                                    (W1 in registers, k_deep.cu; 2 launches per
                                    epoch in pnn_kernel_info);
                                    PNN_VARIANT_CLUSTER_GENERIC forces the
                                    generic kernel.                           */ };

/* Kernel variant inside a family (pnn_set_variant / pnn_kernel_variant).  All
 * variants of a family compute the same method (§3); they differ in
 * data placement and schedule, so results agree to rounding (DESIGN.md §3 R27). */
enum { PNN_VARIANT_AUTO = 0,             /* the family's AUTO rule              */
       PNN_VARIANT_RESIDENT_V8 = 8,      /* W1 in the registers of a 1-4 CTA
                                            cluster, chain on warp pairs        */
       PNN_VARIANT_RESIDENT_V10 = 10,    /* sweep CTA(s) + a dedicated chain CTA */
       PNN_VARIANT_RESIDENT_TMEM = 11,   /* one SM per CN: W1 in registers and
                                            tensor memory (H <= 128)            */
       PNN_VARIANT_RESIDENT_WS = 12,     /* as TMEM, warp-specialised: sweeps and
                                            the per-sample chain on separate
                                            warpgroups (H <= 128)               */
       PNN_VARIANT_CLUSTER_GENERIC = 20, /* any depth, weights in shared memory  */
       PNN_VARIANT_CLUSTER_DEEP = 21,    /* 3-layer nets, W1 in registers       */
       PNN_VARIANT_MB_STEP = 30,         /* fp32 mini-batch: step kernels       */
       PNN_VARIANT_MB_RESIDENT = 31 };   /* fp32 mini-batch: one launch/epoch   */

/* Build a PNN of n_subnets CNs with layer sizes layers[0..n_layers-1]
 * (layers[0] = inputs, e.g. {784,128,10}; n_layers >= 2, each size >= 1,
 * at most 16 layers), activation[l-1] for layer l = 1..n_layers-1 (per-layer
 * choice), init (enum above), learning rate lr (η in
 * Eqs.12-13; finite, > 0), seed for init.  Allocates on the current CUDA
 * device: n_subnets slabs of P_total fp32 (until pnn_set_comm narrows them to
 * this rank's share), one merged slab (initialised to the init, so predict
 * before any merge sees the untrained network) and scratch.  Synchronous.
 * Errors: PNN_ERR_INVALID (every violation is listed in the message:
 * n_layers < 2 or > 16, size <= 0, softmax on a hidden layer, unknown enum,
 * n_subnets < 1, lr <= 0 or not finite, out == NULL), PNN_ERR_OOM,
 * PNN_ERR_CUDA.  On error *out is NULL (message via pnn_last_error(NULL)).   */
pnn_status pnn_create(const int32_t* layers, int32_t n_layers, const int32_t* activation,
                      int32_t init, int32_t n_subnets, float lr, uint64_t seed, pnn_net* out);

/* Multi-GPU (SPMD over ranks, one process per GPU): this rank owns CNs
 * [floor(rank*K/nranks), floor((rank+1)*K/nranks)) and trains on exactly their
 * slices (pnn_local_rows says which rows of the full set); pnn_merge finishes
 * with one NCCL all-reduce over the nranks ranks.  nccl_unique_id points to the
 * 128-byte ncclUniqueId every rank received (e.g. via torch.distributed
 * broadcast).  nranks == 1 needs no id: with NULL it uses no NCCL (the fused
 * local merge); with an id it makes a one-rank communicator and pnn_merge runs
 * the same partial → ncclAllReduce → finish chain as on N ranks.  With
 * nranks > 1 and id == NULL the rank bookkeeping applies but no communicator
 * is made: the caller reduces itself (pnn_merge_partial → its own all-reduce of
 * the fp64 sums → pnn_merge_finish) and pnn_merge returns PNN_ERR_STATE.  A rank
 * that owns no CN (K < nranks) trains nothing and contributes zeros.
 * Re-initialises the local CN slabs to the init.  Collective over ranks (with an
 * id), synchronous.  Errors: PNN_ERR_INVALID (nranks < 1, rank out of range),
 * PNN_ERR_NCCL (libnccl.so.2 missing or init failed), PNN_ERR_OOM.            */
pnn_status pnn_set_comm(pnn_net net, const void* nccl_unique_id, int32_t nranks, int32_t rank);

/* Update schedule: batch = 1 is stochastic GD (the default:
 * update after every instance); batch > 1 is mini-batch GD (gradients of the
 * batch averaged before one update; the short last batch of a slice is
 * averaged over its actual size, R14).  precision PNN_FP32 or PNN_BF16 (bf16
 * operands, fp32 accumulate + master weights, rounding points of DESIGN.md
 * §3 R25; built for D-H1-H2-O nets with ReLU, ReLU, softmax, batch 64,
 * D % 8 == 0, H1 % 128 == 0, H2 % 256 == 0, O <= 16 — the C5 shape
 * 784-1024-1024-10; it then overrides pnn_set_kernel).
 * Errors: PNN_ERR_INVALID (batch < 1, unknown precision, PNN_BF16 on a shape
 * outside the list above — the message names the violated condition).     */
pnn_status pnn_set_minibatch(pnn_net net, int32_t batch, int32_t precision);

/* Force a training kernel (PNN_KERNEL_AUTO, _REFERENCE, _RESIDENT or _CLUSTER).
 * PNN_KERNEL_RESIDENT / _CLUSTER return PNN_ERR_INVALID when the shape does
 * not fit them; _TC_BF16 and _MB_F32 are not settable.    */
pnn_status pnn_set_kernel(pnn_net net, int32_t kernel);

/* Force a kernel variant (PNN_VARIANT_*; AUTO restores the rule).  A non-AUTO
 * variant also selects its family (as pnn_set_kernel would); pnn_set_kernel
 * resets the variant to AUTO.  The variant must support the shape and the
 * current mini-batch setting (pnn_set_minibatch first).  The choice is fixed
 * here, not read from the environment, and pnn_kernel_variant reports it.
 * Errors: PNN_ERR_INVALID (unknown variant, or the shape / batch does not fit
 * it: the message says why).                                                 */
pnn_status pnn_set_variant(pnn_net net, int32_t variant);

/* The variant (PNN_VARIANT_*) the next pnn_train_epoch launches: the forced one or
 * AUTO's resolution; PNN_VARIANT_AUTO for kernels without variants (reference,
 * bf16).  Errors: PNN_ERR_INVALID.                                             */
pnn_status pnn_kernel_variant(pnn_net net, int32_t* variant);

/* Limit how many local CNs train concurrently (the GPU
 * analogue of the paper's goroutine count, Table 2): each
 * pnn_train_epoch then trains the CNs in consecutive waves of `slots` CNs, one
 * wave after the other on the stream.  0 (the default) = all local CNs in one
 * wave.  Results are identical for every slots value (the CNs are independent).
 * Errors: PNN_ERR_INVALID (slots < 0).                                       */
pnn_status pnn_set_slots(pnn_net net, int32_t slots);

/* One training epoch of every local CN ("Each child-network
 * learns only a slice of the dataset"; :225-231).  On a rank that owns no CN
 * (K < nranks) the call is a no-op that needs n = 0 (x / labels may be NULL).
 * x: device fp32
 * [n][layers[0]] row-major; labels: device int32 [n], each in
 * [0, layers[n_layers-1]) (the one-hot target e of Eqs.6-10 is implicit).
 * n = this rank's rows: the concatenated slices of its CNs, split among them
 * contiguously by R17 (the first n mod K_local CNs get one extra row), each
 * visited in index order (R8).  Asynchronous on cuda_stream.
 * Errors: PNN_ERR_INVALID (NULL pointer), PNN_ERR_DATA (n < local CN count,
 * or a slice shorter than the mini-batch), PNN_ERR_STATE, PNN_ERR_CUDA.
 * Labels out of range are not checked on the device (undefined result).    */
pnn_status pnn_train_epoch(pnn_net net, const float* x, const int32_t* labels, int64_t n,
                           void* cuda_stream);

/* Same, with HOST x / labels (pageable or pinned).  The rows are copied to
 * the device in slices overlapped with training; the call returns when the
 * epoch has been enqueued and the host buffers have been consumed
 * (synchronous w.r.t. the host buffers).  Errors as pnn_train_epoch, plus
 * PNN_ERR_OOM for the staging buffer.                                        */
pnn_status pnn_train_epoch_host(pnn_net net, const float* x_host, const int32_t* labels_host,
                                int64_t n, void* cuda_stream);

/* Fuse: merged := (Σ over ALL K CNs of W, b) / K (
 * R18).  The local sum runs in ascending CN order in fp64, the cross-rank sum
 * is one ncclAllReduce(sum, fp64) (nranks > 1 only), then ÷K and one
 * rounding to fp32.  CNs are left untouched.  Asynchronous.
 * Errors: PNN_ERR_STATE (also: nranks > 1 without a communicator), PNN_ERR_CUDA,
 * PNN_ERR_NCCL.                                                              */
pnn_status pnn_merge(pnn_net net, void* cuda_stream);

/* The two device steps of pnn_merge around its all-reduce, for callers that run
 * the cross-rank reduction themselves (e.g. torch.distributed) and for testing
 * the multi-rank arithmetic on one GPU.  pnn_merge_partial: sum_out (device fp64
 * [P_total], caller-owned) = Σ of this rank's CNs in ascending CN order (zeros on a
 * rank that owns no CN).  pnn_merge_finish: merged := (float)(sum / K) from a
 * device fp64 [P_total] that holds the sum over ALL K CNs (PAPER.md:233-238,
 * R18).  pnn_merge with nranks > 1 is exactly partial → ncclAllReduce(sum, fp64)
 * → finish.  Asynchronous.  Errors: PNN_ERR_INVALID (NULL pointer),
 * PNN_ERR_STATE, PNN_ERR_CUDA.                                               */
pnn_status pnn_merge_partial(pnn_net net, double* sum_out, void* cuda_stream);
pnn_status pnn_merge_finish(pnn_net net, const double* sum, void* cuda_stream);

/* Classify n rows of x (device fp32 [n][layers[0]]) with the merged network
 * (subnet = -1) or local CN `subnet` (global index): labels_out[i] (device
 * int32 [n]) = argmax_k z^L_k, ties to the lowest k (R19).  The
 * forward pass accumulates in fp64 from the fp32 parameters (the argmax
 * decision is taken in fp64; DESIGN.md §3 R26).  Asynchronous.
 * Errors: PNN_ERR_INVALID (NULL pointer, n < 0, subnet not local).          */
pnn_status pnn_predict(pnn_net net, int32_t subnet, const float* x, int64_t n,
                       int32_t* labels_out, void* cuda_stream);

/* Evaluation metrics of the merged network (subnet = -1) or a local CN (global
 * index) on n labelled rows (x: device fp32 [n][layers[0]], labels: device int32
 * [n]), the quantities of the paper's experiments (PAPER.md
 * :333-401, 486-547), computed in fp64 from the fp32 parameters (as pnn_predict):
 *   metrics_out[0] accuracy   = fraction of rows whose readout label (argmax z^L,
 *                               ties → lowest, R19) equals the label;
 *   metrics_out[1] confidence = mean over rows of max_k x^L_k (softmax output: the
 *                               predicted class's probability; the paper never
 *                               defines confidence — reading R29);
 *   metrics_out[2] cost       = mean over rows of −log(max(x^L_y, 1e-12)) (Eq.6,
 *                               PAPER.md:100-103, ε-clamp R29).
 * A label outside [0, n_out) counts as wrong with the ε cost.  Synchronises
 * cuda_stream (metrics_out is host memory).  Errors: PNN_ERR_INVALID (NULL
 * pointer, n <= 0, subnet not local), PNN_ERR_OOM, PNN_ERR_CUDA.             */
pnn_status pnn_evaluate(pnn_net net, int32_t subnet, const float* x, const int32_t* labels, int64_t n,
                        double* metrics_out, void* cuda_stream);

/* Copy parameters to host_out (n_floats must equal P_total).  subnet = -1:
 * the merged network; otherwise a local CN (global index).  Synchronises
 * the device.  Errors: PNN_ERR_INVALID, PNN_ERR_SHAPE, PNN_ERR_CUDA.        */
pnn_status pnn_get_params(pnn_net net, int32_t subnet, float* host_out, int64_t n_floats);

/* Copy host_in (P_total floats) into a local CN (global index), into every
 * local CN (subnet = -1), or into the merged network (subnet = -2).
 * Synchronous.  Errors: PNN_ERR_INVALID, PNN_ERR_SHAPE, PNN_ERR_CUDA.        */
pnn_status pnn_set_params(pnn_net net, int32_t subnet, const float* host_in, int64_t n_floats);

/* Device pointer of a local CN's slab (global index) or of the merged slab
 * (-1), for zero-copy export (e.g. wrapping as a torch tensor).  NULL on
 * error.                                                                      */
float* pnn_device_params(pnn_net net, int32_t subnet);

/* P_total, or -1 for a NULL handle. */
int64_t pnn_param_count(pnn_net net);

/* This rank's CN range [*first, *first + *count).  Errors: PNN_ERR_INVALID. */
pnn_status pnn_local_subnets(pnn_net net, int32_t* first, int32_t* count);

/* The rows of an n_total-row training set this rank trains on (PAPER.md:166-169
 * slicing, R17 over all K CNs): [*first, *first + *count) = the concatenated
 * slices of its CNs, which is what pnn_train_epoch expects as x / labels.  A rank
 * that owns no CN (K < nranks) gets *count = 0.  Errors: PNN_ERR_INVALID (NULL
 * pointer, n_total < K).                                                      */
pnn_status pnn_local_rows(pnn_net net, int64_t n_total, int64_t* first, int64_t* count);

/* Which training kernel the next pnn_train_epoch launches (PNN_KERNEL_*),
 * and how many kernel launches it makes (PNN_KERNEL_TC_BF16: launches per
 * mini-batch step; an epoch makes 1 + that × ceil(longest slice / batch);
 * PNN_KERNEL_MB_F32: per step, an epoch makes that × ceil(longest slice / batch);
 * PNN_KERNEL_MB_RESIDENT: per epoch).
 * Errors: PNN_ERR_INVALID.                                                  */
pnn_status pnn_kernel_info(pnn_net net, int32_t* kernel, int32_t* launches_per_epoch);

/* Measurement hook: enable = 1 starts recording a pair of CUDA events around every
 * training-kernel launch that follows (on the caller's stream; the resident path
 * brackets its SGD kernel, not the Gram pre-pass; the mini-batch paths their epoch
 * graph); enable = 0 stops, waits for the recorded events and returns the mean
 * launch duration in ms and the number of launches (either pointer may be NULL).
 * Errors: PNN_ERR_INVALID (NULL handle), PNN_ERR_CUDA.                           */
pnn_status pnn_kernel_timing(pnn_net net, int32_t enable, double* mean_ms, int32_t* count);

/* Last error message of this handle (or of the last failed pnn_create when
 * net is NULL).  Never NULL; valid until the next call on the handle.        */
const char* pnn_last_error(pnn_net net);

/* Free all device state (synchronises the device).  NULL is a no-op. */
pnn_status pnn_destroy(pnn_net net);

#ifdef __cplusplus
}
#endif
#endif /* PNN_H_ */
