/* examples/pnn_example.c — the C ABI (include/pnn.h) driven from plain C: no Python, no
 * torch.  Builds a 784-64-10 ReLU/softmax PNN of 8 child networks, trains 3 epochs from
 * HOST buffers (pnn_train_epoch_host), fuses the children (pnn_merge) and evaluates the
 * merged network on device-resident test rows (pnn_evaluate).
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/pnn_example.c -L paper_2304_09590_b200 -lpnn \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_2304_09590_b200 -o pnn_example
 *
 * Data: a learnable synthetic 10-class task (class c lights pixels with (i·7 + c·31) % 10
 * == 0, plus deterministic noise), generated here.  Exit status 0 iff every call succeeds
 * and the merged network beats chance clearly.                                          */
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>
#include <cuda_runtime_api.h>
#include "pnn.h"

#define CHECK(call)                                                                       \
    do {                                                                                  \
        pnn_status st_ = (call);                                                          \
        if (st_ != PNN_OK) {                                                              \
            fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, pnn_last_error(net)); \
            return 1;                                                                     \
        }                                                                                 \
    } while (0)

static float noise(uint64_t i) {                 /* deterministic value in [0, 0.3) */
    uint64_t z = i * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return (float)((z ^ (z >> 31)) >> 11) * (1.0f / 9007199254740992.0f) * 0.3f;
}

static void make_rows(float* x, int32_t* y, int n, uint64_t base) {
    for (int r = 0; r < n; ++r) {
        const int c = (int)((r * 7 + base) % 10);
        y[r] = c;
        for (int i = 0; i < 784; ++i)
            x[(size_t)r * 784 + i] = (((i * 7 + c * 31) % 10) == 0 ? 0.7f : 0.0f) + noise(base * 1000003ULL + (uint64_t)r * 784 + i);
    }
}

int main(void) {
    pnn_net net = NULL;
    const int32_t layers[3] = {784, 64, 10};
    const int32_t act[2] = {PNN_RELU, PNN_SOFTMAX};
    const int K = 8, n = 8 * 500, nt = 1000;
    if (pnn_create(layers, 3, act, PNN_INIT_HE_NORMAL, K, 0.01f, 42, &net) != PNN_OK) {
        fprintf(stderr, "pnn_create: %s\n", pnn_last_error(NULL));
        return 1;
    }
    float* x = (float*)malloc(sizeof(float) * (size_t)n * 784);
    int32_t* y = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    float* xt = (float*)malloc(sizeof(float) * (size_t)nt * 784);
    int32_t* yt = (int32_t*)malloc(sizeof(int32_t) * (size_t)nt);
    make_rows(x, y, n, 1);
    make_rows(xt, yt, nt, 2);
    int32_t kernel = -1, launches = -1;
    CHECK(pnn_kernel_info(net, &kernel, &launches));
    for (int e = 0; e < 3; ++e) CHECK(pnn_train_epoch_host(net, x, y, n, NULL));
    CHECK(pnn_merge(net, NULL));
    float *dxt = NULL;
    int32_t* dyt = NULL;
    if (cudaMalloc((void**)&dxt, sizeof(float) * (size_t)nt * 784) != cudaSuccess ||
        cudaMalloc((void**)&dyt, sizeof(int32_t) * (size_t)nt) != cudaSuccess) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    cudaMemcpy(dxt, xt, sizeof(float) * (size_t)nt * 784, cudaMemcpyHostToDevice);
    cudaMemcpy(dyt, yt, sizeof(int32_t) * (size_t)nt, cudaMemcpyHostToDevice);
    double m[3];
    CHECK(pnn_evaluate(net, -1, dxt, dyt, nt, m, NULL));
    printf("kernel %d, %d launches/epoch, P_total %lld: merged accuracy %.4f confidence %.4f cost %.4f\n",
           (int)kernel, (int)launches, (long long)pnn_param_count(net), m[0], m[1], m[2]);
    cudaFree(dxt);
    cudaFree(dyt);
    free(x); free(y); free(xt); free(yt);
    CHECK(pnn_destroy(net));
    return m[0] > 0.5 ? 0 : 2;
}
