// pnn_internal.h — shared declarations of the CUDA path (host library + kernels).
// Nothing here is visible through the C ABI (include/pnn.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PNN_MAX_LAYERS 16

// Network shape, passed by value to every kernel.
//   n[0..L]   layer sizes (n[0] = inputs)
//   act[l-1]  activation of layer l (PNN_SIGMOID..PNN_SOFTMAX)
//   woff[l]   offset of W^l in a parameter slab; b^l follows at woff[l] + n[l]*n[l-1]
//   noff[l]   offset of layer l's neurons in per-sample scratch (z, x, δ)
struct NetDesc {
    int L;
    int n[PNN_MAX_LAYERS + 1];
    int act[PNN_MAX_LAYERS];
    long long woff[PNN_MAX_LAYERS + 1];
    int noff[PNN_MAX_LAYERS + 1];
    long long P;        // P_total
    int neurons;        // Σ_{l>=1} n[l]
    int max_width;      // max_l n[l], l >= 0
};

// R17: CN s of K gets rows [start, start+count): floor(n/K) + [s < n mod K].
__host__ __device__ inline void shard_of(long long n, int K, int s, long long* start,
                                         long long* count) {
    long long base = n / K, rem = n % K;
    *start = (long long)s * base + (s < rem ? s : rem);
    *count = base + (s < rem ? 1 : 0);
}

// ---- kernels (launchers return cudaGetLastError()) -----------------------
// Reference SGD: one CTA per CN, parameters in global memory.  CNs
// [s_first, s_first+s_count) of the K_local local ones; rows split by R17
// over n_local rows.  batch == 1: per-instance SGD; batch > 1: mini-batch
// (gscratch: [K_local][P] fp32 gradient sums).
cudaError_t launch_sgd_reference(const NetDesc& d, float* children, const float* x,
                                 const int32_t* labels, long long n_local, int K_local,
                                 int s_first, int s_count, float lr, int batch, float* gscratch,
                                 cudaStream_t st);

// Resident (persistent, on-chip weights) SGD kernel; see k_resident.cu.
struct ResidentPlan {
    bool ok;
    int cluster;        // CTAs per cluster (each CN is split over all of them)
    int groups;         // CNs per cluster (warp groups per CTA)
    int threads;        // threads per CTA
    size_t smem;        // dynamic shared memory per CTA
    int variant;        // template instance id
    char why[160];      // reason when !ok
};
// concurrent: CNs trained at once (0 = unknown); variant: PNN_VARIANT_AUTO or a forced
// PNN_VARIANT_RESIDENT_* (see plan_resident's rule)
ResidentPlan plan_resident(const NetDesc& d, int batch, int concurrent = 0, int variant = 0);
// gram: scratch of 2·n_local float4 (32-B records: the lookahead's Gram terms and the
// label of every row, recomputed per call).
cudaError_t launch_sgd_resident(const ResidentPlan& p, const NetDesc& d, float* children,
                                const float* x, const int32_t* labels, float4* gram, long long n_local,
                                int K_local, int s_first, int s_count, float lr,
                                cudaStream_t st, cudaEvent_t ev0 = nullptr, cudaEvent_t ev1 = nullptr);

// TMEM variant (k_tmem.cu, v11): one SM per CN, W¹ rows in registers + tensor memory,
// Gram terms formed in the launch.  nullptr when the shape is supported.
const char* tmem_plan(const NetDesc& d, int batch);
cudaError_t launch_sgd_tmem(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                            int K_local, int s_first, int s_count, float lr, cudaStream_t st);

// Warp-specialised TMEM variant (k_ws.cu, v12): as v11 with the per-sample chain on its own
// warpgroup.  nullptr when the shape is supported.  rec: the Gram records of launch_gram (the
// chain reads the terms and the labels from the x ring).
const char* ws_plan(const NetDesc& d, int batch);
cudaError_t launch_sgd_ws(const NetDesc& d, float* children, const float* x, const int32_t* y, const float4* rec,
                          long long n_local, int K_local, int s_first, int s_count, float lr, cudaStream_t st);

// The lookahead's Gram records (32 B per row: x(u-4..u-1)·x(u) and the label), k_resident.cu.
cudaError_t launch_gram(const float* x, const int32_t* labels, int D, long long n_local, int K_local, int s_first,
                        int s_count, float4* rec, cudaStream_t st);

// Deep kernel (k_deep.cu): 3-layer nets D-H1-H2-O, W¹ rows register-resident across a cluster of
// 8 CTAs with the R27 lookahead, layers 2-3 and the per-sample chain on dedicated warps.
const char* deep_plan(const NetDesc& d, int batch);   // nullptr when supported
int deep_cluster_size(const NetDesc& d);
cudaError_t launch_sgd_deep(const NetDesc& d, float* children, const float* x, const int32_t* labels,
                            float4* rec, long long n_local, int K_local, int s_first, int s_count, float lr,
                            cudaStream_t st);

// Cluster kernel (k_cluster.cu): any depth, weights resident in the shared memory of a
// cluster of C <= 8 CTAs, per-sample SGD.
struct ClusterPlan {
    bool ok;
    int cluster;
    size_t smem;
    char why[160];
};
ClusterPlan plan_cluster(const NetDesc& d, int batch);
cudaError_t launch_sgd_cluster(const ClusterPlan& p, const NetDesc& d, float* children, const float* x,
                               const int32_t* labels, long long n_local, int K_local, int s_first,
                               int s_count, float lr, cudaStream_t st);

// bf16 mini-batch variant on tcgen05 GEMMs (k_minibatch.cu): nullptr when the shape /
// batch is supported, else the reason.
struct MbState;
const char* mb_plan(const NetDesc& d, int batch);
MbState* mb_create(const NetDesc& d, int K_local, int batch, cudaError_t* err);
void mb_destroy(MbState* s);
cudaError_t launch_minibatch_bf16(MbState* s, const NetDesc& d, float* children, const float* x,
                                  const int32_t* y, long long n_local, int K_local, int s_first,
                                  int s_count, float lr, cudaStream_t st);

// fp32 mini-batch kernels for D-H-O nets (k_minibatch_f32.cu; f1): nullptr when supported.
struct Mb32State;
const char* mb32_plan(const NetDesc& d, int batch);
// Resident fp32 mini-batch kernel (k_mbres.cu): one launch per epoch, W¹ in registers.
const char* mbres_plan(const NetDesc& d, int batch);   // nullptr when supported
int mbres_cluster(const NetDesc& d);
cudaError_t launch_mbres(const NetDesc& d, float* children, const float* x, const int32_t* y, long long n_local,
                         int K_local, int s_first, int s_count, int B, float lr, cudaStream_t st);
Mb32State* mb32_create(const NetDesc& d, int K_local, int batch, cudaError_t* err);
void mb32_destroy(Mb32State* s);
cudaError_t launch_minibatch_f32(Mb32State* s, const NetDesc& d, float* children, const float* x,
                                 const int32_t* y, long long n_local, int K_local, int s_first,
                                 int s_count, float lr, cudaStream_t st);

// Merge: sum[i] = Σ_{c<K_local} children[c][i] in fp64, ascending c.
cudaError_t launch_merge_sum(const float* children, int K_local, long long P, double* sum,
                             cudaStream_t st);
// merged[i] = (float)(sum[i] / K).
cudaError_t launch_merge_finish(const double* sum, long long P, int K, float* merged,
                                cudaStream_t st);
// Single-rank fused version: merged[i] = (float)((Σ_c children[c][i]) / K).
cudaError_t launch_merge_local(const float* children, int K_local, long long P, int K,
                               float* merged, cudaStream_t st);

// Predict: labels[i] = argmax z^L (fp64 forward from fp32 params), ties → lowest.
// f2 evaluation: rowstats [n][3] scratch; out3 (device) = mean of (correct, max x^L,
// −log max(x^L_y, 1e-12)) over the n rows.
cudaError_t launch_evaluate(const NetDesc& d, const float* params, const float* x, const int32_t* y,
                            long long n, double* rowstats, double* out3, cudaStream_t st);
cudaError_t launch_predict(const NetDesc& d, const float* params, const float* x, long long n,
                           int32_t* labels, cudaStream_t st);
