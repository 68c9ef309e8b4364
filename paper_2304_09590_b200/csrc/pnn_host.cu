// pnn_host.cu — the C ABI of include/pnn.h: handle, validation, init RNG,
// slicing, kernel selection, merge orchestration and the NCCL communicator.
//
// Every step of the hot path runs in this library's kernels (k_*.cu); this
// file only validates, allocates and enqueues.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <dlfcn.h>
#include <nccl.h>
#include <string>
#include <vector>

#include "pnn.h"
#include "pnn_internal.h"

struct pnn_net_s {
    NetDesc d{};
    std::vector<int> layers, act;
    int init = 0, K = 1;
    float lr = 0.f;
    uint64_t seed = 0;
    int device = 0;
    int nranks = 1, rank = 0;
    int k_first = 0, K_local = 1;     // this rank's CNs [k_first, k_first + K_local)
    void* comm = nullptr;             // ncclComm_t
    int batch = 1, precision = PNN_FP32, kernel = PNN_KERNEL_AUTO;
    int variant = PNN_VARIANT_AUTO;   // forced kernel variant (pnn_set_variant)
    int slots = 0;                    // CNs trained concurrently (0 = all local CNs; f4)
    bool timing = false;              // record CUDA events around each training-kernel launch
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
    float* d_children = nullptr;      // [K_local][P]
    float* d_merged = nullptr;        // [P]
    double* d_msum = nullptr;         // [P] fp64 partial sums (multi-rank merge)
    float* d_gscratch = nullptr;      // [K_local][P] mini-batch gradient sums (lazy)
    MbState* mb = nullptr;            // bf16 mini-batch buffers + tensor maps (lazy, a10)
    Mb32State* mb32 = nullptr;        // fp32 mini-batch buffers (lazy, f1)
    float4* d_gram = nullptr;         // [gram_rows] Gram terms of the resident kernel (lazy)
    long long gram_rows = 0;
    double* d_eval = nullptr;         // evaluation row statistics [eval_rows][3] + 3 means (lazy)
    long long eval_rows = 0;
    float* d_xstage = nullptr;        // host-input staging (lazy)
    int32_t* d_ystage = nullptr;
    long long stage_rows = 0;
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t stage_released = nullptr;   // recorded after the last launch that reads the staging
    cudaEvent_t grp_released[8] = {};       // per group of the last host-input call: recorded after
                                            // the launch that reads that group's staging rows
    long long grp_n = -1;                   // that call's (n, first CN of this handle's groups,
    int grp_count = 0, grp_size = 0;        // groups, group size); -1: no per-group record
                                            // buffers (any stream); copy_stream waits on it
    std::vector<float> h_init;        // init parameters (cloned into every CN)
    bool poisoned = false;
    std::string err;
};

namespace {

thread_local std::string g_create_err;

pnn_status fail(pnn_net net, pnn_status st, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (net) {
        net->err = buf;
        if (st == PNN_ERR_CUDA || st == PNN_ERR_NCCL) net->poisoned = true;
    } else {
        g_create_err = buf;
    }
    return st;
}

#define CUDA_TRY(net, expr)                                                                   \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(net, e_ == cudaErrorMemoryAllocation ? PNN_ERR_OOM : PNN_ERR_CUDA,    \
                        "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

pnn_status check_live(pnn_net net) {
    if (!net) return PNN_ERR_INVALID;
    if (net->poisoned) {
        net->err = "handle poisoned by an earlier CUDA/NCCL error: " + net->err;
        return PNN_ERR_STATE;
    }
    return PNN_OK;
}

// ---- init RNG (reading R15) ---------------------------
// Counter-based SplitMix64: this is the host library's own implementation of
// the generator DESIGN.md §3 R15 specifies (the oracle has its own).
uint64_t splitmix_fin(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
double draw_u01(uint64_t seed, int layer, int kind, int64_t idx, int s) {
    uint64_t ctr = ((uint64_t)layer << 48) ^ ((uint64_t)kind << 47) ^ (uint64_t)(2 * idx + s);
    uint64_t h = splitmix_fin(seed * 0x9E3779B97F4A7C15ULL + splitmix_fin(ctr + 0x632BE59BD9B4E019ULL));
    return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}
double draw_n01(uint64_t seed, int layer, int kind, int64_t idx) {
    double u1 = draw_u01(seed, layer, kind, idx, 0), u2 = draw_u01(seed, layer, kind, idx, 1);
    return std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(6.283185307179586 * u2);
}
void init_params_host(const NetDesc& d, int init, uint64_t seed, std::vector<float>& p) {
    p.assign((size_t)d.P, 0.f);
    for (int l = 1; l <= d.L; ++l) {
        const int nin = d.n[l - 1], nout = d.n[l];
        const long long nw = (long long)nin * nout;
        float* W = p.data() + d.woff[l];
        float* b = W + nw;
        double sigma = 1.0;
        if (init == PNN_INIT_XAVIER_NORMAL) sigma = std::sqrt(2.0 / (double)(nin + nout));
        if (init == PNN_INIT_HE_NORMAL) sigma = std::sqrt(2.0 / (double)nin);
        for (long long i = 0; i < nw; ++i)
            W[i] = (init == PNN_INIT_UNIFORM) ? (float)(draw_u01(seed, l, 0, i, 0) - 0.5)
                                              : (float)(sigma * draw_n01(seed, l, 0, i));
        for (int k = 0; k < nout; ++k)
            b[k] = (init == PNN_INIT_NORMAL)    ? (float)draw_n01(seed, l, 1, k)
                   : (init == PNN_INIT_UNIFORM) ? (float)(draw_u01(seed, l, 1, k, 0) - 0.5)
                                                : 0.f;
    }
}

// ---- NCCL, resolved at run time (the process may already hold torch's copy;
// dlopen by soname then returns that one).  Types come from nccl.h.
struct NcclApi {
    void* h = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclAllReduce) AllReduce = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
};
NcclApi g_nccl;

bool load_nccl(std::string& why) {
    if (g_nccl.h) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { why = std::string("dlopen libnccl.so.2: ") + dlerror(); return false; }
    g_nccl.CommInitRank = (decltype(&ncclCommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.AllReduce = (decltype(&ncclAllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.CommDestroy = (decltype(&ncclCommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.GetErrorString = (decltype(&ncclGetErrorString))dlsym(h, "ncclGetErrorString");
    if (!g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy || !g_nccl.GetErrorString) {
        why = "libnccl.so.2 lacks a required symbol";
        return false;
    }
    g_nccl.h = h;
    return true;
}

pnn_status alloc_local(pnn_net net) {
    mb_destroy(net->mb); net->mb = nullptr;
    mb32_destroy(net->mb32); net->mb32 = nullptr;
    cudaFree(net->d_children); net->d_children = nullptr;
    cudaFree(net->d_gscratch); net->d_gscratch = nullptr;
    const size_t bytes = sizeof(float) * (size_t)net->d.P * (size_t)(net->K_local > 0 ? net->K_local : 1);
    CUDA_TRY(net, cudaMalloc(&net->d_children, bytes));
    for (int c = 0; c < net->K_local; ++c)
        CUDA_TRY(net, cudaMemcpy(net->d_children + (size_t)c * net->d.P, net->h_init.data(),
                                 sizeof(float) * net->d.P, cudaMemcpyHostToDevice));
    return PNN_OK;
}

bool is_resident_variant(int v) {
    return v == PNN_VARIANT_RESIDENT_V8 || v == PNN_VARIANT_RESIDENT_V10 || v == PNN_VARIANT_RESIDENT_TMEM ||
           v == PNN_VARIANT_RESIDENT_WS;
}

// The kernel family (PNN_KERNEL_*, -1 when a forced choice does not fit) and, in *var, the
// variant the next epoch launches.  Everything comes from the handle: no environment reads.
int choose_kernel(pnn_net net, ResidentPlan* plan, int* var = nullptr) {
    int vdummy = 0;
    int& v = var ? *var : vdummy;
    v = PNN_VARIANT_AUTO;
    const int fv = net->variant;
    if (net->precision == PNN_BF16) return PNN_KERNEL_TC_BF16;
    if (fv == PNN_VARIANT_MB_STEP || fv == PNN_VARIANT_MB_RESIDENT) {
        if (net->batch < 2) return -1;
        if (fv == PNN_VARIANT_MB_RESIDENT && mbres_plan(net->d, net->batch)) return -1;
        if (fv == PNN_VARIANT_MB_STEP && mb32_plan(net->d, net->batch)) return -1;
    }
    if (net->kernel != PNN_KERNEL_REFERENCE && net->batch > 1) {
        if (fv != PNN_VARIANT_MB_STEP && !mbres_plan(net->d, net->batch)) {
            v = PNN_VARIANT_MB_RESIDENT;
            return PNN_KERNEL_MB_RESIDENT;
        }
        if (!mb32_plan(net->d, net->batch)) {
            v = PNN_VARIANT_MB_STEP;
            return PNN_KERNEL_MB_F32;
        }
    }
    if (net->kernel == PNN_KERNEL_REFERENCE) return PNN_KERNEL_REFERENCE;
    auto cluster = [&]() -> int {
        if (!plan_cluster(net->d, net->batch).ok) return -1;
        const bool deep_ok = deep_plan(net->d, net->batch) == nullptr;
        if (fv == PNN_VARIANT_CLUSTER_DEEP && !deep_ok) return -1;
        v = (deep_ok && fv != PNN_VARIANT_CLUSTER_GENERIC) ? PNN_VARIANT_CLUSTER_DEEP : PNN_VARIANT_CLUSTER_GENERIC;
        return PNN_KERNEL_CLUSTER;
    };
    if (net->kernel == PNN_KERNEL_CLUSTER) return cluster();
    const int conc = (net->slots > 0 && net->slots < net->K_local) ? net->slots : net->K_local;
    *plan = plan_resident(net->d, net->batch, conc, is_resident_variant(fv) ? fv : PNN_VARIANT_AUTO);
    if (plan->ok)
        v = plan->variant == 8 ? PNN_VARIANT_RESIDENT_V8
            : plan->variant == 10 ? PNN_VARIANT_RESIDENT_V10
            : plan->variant == 12 ? PNN_VARIANT_RESIDENT_WS : PNN_VARIANT_RESIDENT_TMEM;
    if (net->kernel == PNN_KERNEL_RESIDENT) return plan->ok ? PNN_KERNEL_RESIDENT : -1;
    if (plan->ok) return PNN_KERNEL_RESIDENT;
    v = PNN_VARIANT_AUTO;
    const int c = cluster();
    return c >= 0 ? c : PNN_KERNEL_REFERENCE;
}

pnn_status launch_train_wave(pnn_net net, const float* x, const int32_t* y, long long n,
                             int s_first, int s_count, cudaStream_t st);

// Train local CNs [s_first, s_first + s_count), in waves of at most `slots` CNs (f4: the
// GPU analogue of the paper's goroutine count) when a limit is set.
pnn_status launch_train(pnn_net net, const float* x, const int32_t* y, long long n,
                        int s_first, int s_count, cudaStream_t st) {
    const int w = (net->slots > 0 && net->slots < s_count) ? net->slots : s_count;
    for (int s0 = s_first; s0 < s_first + s_count; s0 += w) {
        const int c = (s_first + s_count - s0) < w ? (s_first + s_count - s0) : w;
        pnn_status r = launch_train_wave(net, x, y, n, s0, c, st);
        if (r != PNN_OK) return r;
    }
    return PNN_OK;
}

pnn_status launch_train_wave(pnn_net net, const float* x, const int32_t* y, long long n,
                             int s_first, int s_count, cudaStream_t st) {
    ResidentPlan plan{};
    int var = PNN_VARIANT_AUTO;
    int k = choose_kernel(net, &plan, &var);
    if (k < 0) return fail(net, PNN_ERR_INVALID, "forced kernel / variant not valid here: %s", plan.why);
    cudaError_t e;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    if (net->timing && s_count > 0) {
        CUDA_TRY(net, cudaEventCreate(&ev0));
        CUDA_TRY(net, cudaEventCreate(&ev1));
        net->tev.emplace_back(ev0, ev1);
        if (k != PNN_KERNEL_RESIDENT) CUDA_TRY(net, cudaEventRecord(ev0, st));   // the resident path
    }                                                                               // brackets its SGD launch
    const bool deep = var == PNN_VARIANT_CLUSTER_DEEP;
    const bool gram = deep || (k == PNN_KERNEL_RESIDENT && var != PNN_VARIANT_RESIDENT_TMEM);
    if (gram && net->gram_rows < n) {                                // 32-B Gram records (R27)
        cudaFree(net->d_gram);
        net->d_gram = nullptr;
        net->gram_rows = 0;
        CUDA_TRY(net, cudaMalloc(&net->d_gram, 2 * sizeof(float4) * (size_t)n));
        net->gram_rows = n;
    }
    if (k == PNN_KERNEL_TC_BF16) {
        if (!net->mb) {
            net->mb = mb_create(net->d, net->K_local, net->batch, &e);
            if (!net->mb)
                return fail(net, e == cudaErrorMemoryAllocation ? PNN_ERR_OOM : PNN_ERR_CUDA,
                            "bf16 mini-batch buffers / tensor maps: %s", cudaGetErrorString(e));
        }
        e = launch_minibatch_bf16(net->mb, net->d, net->d_children, x, y, n, net->K_local, s_first,
                                  s_count, net->lr, st);
    } else if (k == PNN_KERNEL_MB_F32) {
        if (!net->mb32) {
            net->mb32 = mb32_create(net->d, net->K_local, net->batch, &e);
            if (!net->mb32)
                return fail(net, e == cudaErrorMemoryAllocation ? PNN_ERR_OOM : PNN_ERR_CUDA,
                            "fp32 mini-batch buffers: %s", cudaGetErrorString(e));
        }
        e = launch_minibatch_f32(net->mb32, net->d, net->d_children, x, y, n, net->K_local, s_first, s_count,
                                 net->lr, st);
    } else if (k == PNN_KERNEL_MB_RESIDENT) {
        e = launch_mbres(net->d, net->d_children, x, y, n, net->K_local, s_first, s_count, net->batch, net->lr, st);
    } else if (deep) {                                       // 3-layer shapes: W¹ in registers
        e = launch_sgd_deep(net->d, net->d_children, x, y, net->d_gram, n, net->K_local, s_first, s_count,
                            net->lr, st);
    } else if (k == PNN_KERNEL_CLUSTER) {
        e = launch_sgd_cluster(plan_cluster(net->d, net->batch), net->d, net->d_children, x, y, n, net->K_local,
                               s_first, s_count, net->lr, st);
    } else if (k == PNN_KERNEL_RESIDENT) {
        e = launch_sgd_resident(plan, net->d, net->d_children, x, y, net->d_gram, n, net->K_local,
                                s_first, s_count, net->lr, st, ev0, ev1);
    } else {
        if (net->batch > 1 && !net->d_gscratch)
            CUDA_TRY(net, cudaMalloc(&net->d_gscratch,
                                     sizeof(float) * (size_t)net->d.P * (size_t)net->K_local));
        e = launch_sgd_reference(net->d, net->d_children, x, y, n, net->K_local, s_first, s_count,
                                 net->lr, net->batch, net->d_gscratch, st);
    }
    if (e != cudaSuccess) return fail(net, PNN_ERR_CUDA, "training launch: %s", cudaGetErrorString(e));
    if (ev1 && k != PNN_KERNEL_RESIDENT) CUDA_TRY(net, cudaEventRecord(ev1, st));
    return PNN_OK;
}

pnn_status check_rows(pnn_net net, long long n) {
    if (net->K_local <= 0)
        return n == 0 ? PNN_OK : fail(net, PNN_ERR_DATA, "this rank owns no CN: n must be 0 (got %lld)", n);
    if (n < net->K_local)
        return fail(net, PNN_ERR_DATA, "n = %lld rows < %d local CNs: some CN would get an empty slice",
                    n, net->K_local);
    if (net->batch > 1 && n / net->K_local < net->batch)
        return fail(net, PNN_ERR_DATA, "slice of %lld rows shorter than the mini-batch %d",
                    n / net->K_local, net->batch);
    return PNN_OK;
}

}  // namespace

extern "C" {

pnn_status pnn_create(const int32_t* layers, int32_t n_layers, const int32_t* activation,
                      int32_t init, int32_t n_subnets, float lr, uint64_t seed, pnn_net* out) {
    if (out) *out = nullptr;
    std::string bad;
    auto add = [&](const std::string& s) { bad += (bad.empty() ? "" : "; ") + s; };
    if (!out) add("out is NULL");
    if (!layers || !activation) add("layers/activation is NULL");
    if (n_layers < 2 || n_layers > PNN_MAX_LAYERS + 1)
        add("n_layers = " + std::to_string(n_layers) + " (need 2.." + std::to_string(PNN_MAX_LAYERS + 1) + ")");
    if (layers && activation && n_layers >= 2 && n_layers <= PNN_MAX_LAYERS + 1) {
        for (int i = 0; i < n_layers; ++i)
            if (layers[i] <= 0) add("layers[" + std::to_string(i) + "] = " + std::to_string(layers[i]) + " <= 0");
        for (int i = 0; i < n_layers - 1; ++i) {
            if (activation[i] < PNN_SIGMOID || activation[i] > PNN_LEAKY_RELU)
                add("activation[" + std::to_string(i) + "] = " + std::to_string(activation[i]) + " unknown");
            else if (activation[i] == PNN_SOFTMAX && i != n_layers - 2)
                add("softmax on hidden layer " + std::to_string(i + 1));
        }
    }
    if (init < PNN_INIT_NORMAL || init > PNN_INIT_HE_NORMAL) add("init = " + std::to_string(init) + " unknown");
    if (n_subnets < 1) add("n_subnets = " + std::to_string(n_subnets) + " < 1");
    if (!(lr > 0.f) || !std::isfinite(lr)) add("lr must be finite and > 0");
    if (!bad.empty()) return fail(nullptr, PNN_ERR_INVALID, "pnn_create: %s", bad.c_str());

    pnn_net net = new pnn_net_s();
    NetDesc& d = net->d;
    d.L = n_layers - 1;
    long long w = 0;
    int nn = 0, mw = 0;
    for (int l = 0; l <= d.L; ++l) { d.n[l] = layers[l]; mw = mw > layers[l] ? mw : layers[l]; }
    for (int l = 1; l <= d.L; ++l) {
        d.act[l - 1] = activation[l - 1];
        d.woff[l] = w;
        d.noff[l] = nn;
        w += (long long)d.n[l] * d.n[l - 1] + d.n[l];
        nn += d.n[l];
    }
    d.P = w;
    d.neurons = nn;
    d.max_width = mw;
    net->layers.assign(layers, layers + n_layers);
    net->act.assign(activation, activation + n_layers - 1);
    net->init = init;
    net->K = n_subnets;
    net->K_local = n_subnets;
    net->lr = lr;
    net->seed = seed;
    cudaGetDevice(&net->device);
    init_params_host(d, init, seed, net->h_init);
    pnn_status st = alloc_local(net);
    if (st == PNN_OK) {
        cudaError_t e = cudaMalloc(&net->d_merged, sizeof(float) * d.P);
        if (e == cudaSuccess)
            e = cudaMemcpy(net->d_merged, net->h_init.data(), sizeof(float) * d.P, cudaMemcpyHostToDevice);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&net->copy_stream, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&net->stage_released, cudaEventDisableTiming);
        for (int g = 0; g < 8 && e == cudaSuccess; ++g)
            e = cudaEventCreateWithFlags(&net->grp_released[g], cudaEventDisableTiming);
        if (e != cudaSuccess)
            st = fail(net, e == cudaErrorMemoryAllocation ? PNN_ERR_OOM : PNN_ERR_CUDA, "%s",
                      cudaGetErrorString(e));
    }
    if (st != PNN_OK) {
        g_create_err = net->err;
        pnn_destroy(net);
        return st;
    }
    *out = net;
    return PNN_OK;
}

pnn_status pnn_set_comm(pnn_net net, const void* id, int32_t nranks, int32_t rank) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(net, PNN_ERR_INVALID, "nranks = %d, rank = %d", nranks, rank);
    CUDA_TRY(net, cudaSetDevice(net->device));
    if (net->comm) { g_nccl.CommDestroy((ncclComm_t)net->comm); net->comm = nullptr; }
    net->nranks = nranks;
    net->rank = rank;
    net->k_first = (int)((long long)rank * net->K / nranks);
    net->K_local = (int)((long long)(rank + 1) * net->K / nranks) - net->k_first;
    // nranks == 1 with an id still makes a (one-rank) communicator, so the NCCL merge path —
    // partial sum → ncclAllReduce → finish — runs on a one-GPU box exactly as on eight.
    if ((nranks > 1 || id) && !net->d_msum) CUDA_TRY(net, cudaMalloc(&net->d_msum, sizeof(double) * net->d.P));
    if (id) {                                     // id == NULL: the caller reduces (merge_partial/finish)
        std::string why;
        if (!load_nccl(why)) return fail(net, PNN_ERR_NCCL, "%s", why.c_str());
        ncclUniqueId uid;
        memcpy(&uid, id, sizeof uid);
        ncclComm_t comm = nullptr;
        ncclResult_t r = g_nccl.CommInitRank(&comm, nranks, uid, rank);
        net->comm = comm;
        if (r != ncclSuccess) return fail(net, PNN_ERR_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
    }
    return alloc_local(net);
}

pnn_status pnn_set_minibatch(pnn_net net, int32_t batch, int32_t precision) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (batch < 1) return fail(net, PNN_ERR_INVALID, "batch = %d < 1", batch);
    if (precision != PNN_FP32 && precision != PNN_BF16)
        return fail(net, PNN_ERR_INVALID, "precision = %d unknown", precision);
    if (precision == PNN_BF16) {
        if (const char* why = mb_plan(net->d, batch))
            return fail(net, PNN_ERR_INVALID, "PNN_BF16 mini-batch: %s", why);
    }
    if (precision != net->precision || batch != net->batch) {
        mb_destroy(net->mb); net->mb = nullptr;
        mb32_destroy(net->mb32); net->mb32 = nullptr;
    }
    net->batch = batch;
    net->precision = precision;
    return PNN_OK;
}

pnn_status pnn_set_kernel(pnn_net net, int32_t kernel) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (kernel < PNN_KERNEL_AUTO || kernel > PNN_KERNEL_CLUSTER || kernel == PNN_KERNEL_TC_BF16 ||
        kernel == PNN_KERNEL_MB_F32)                     // (PNN_KERNEL_MB_RESIDENT = 6: reported only)
        return fail(net, PNN_ERR_INVALID, "kernel = %d unknown or not settable", kernel);
    if (kernel == PNN_KERNEL_CLUSTER) {
        ClusterPlan p = plan_cluster(net->d, net->batch);
        if (!p.ok) return fail(net, PNN_ERR_INVALID, "cluster kernel not valid: %s", p.why);
    }
    if (kernel == PNN_KERNEL_RESIDENT) {
        ResidentPlan p = plan_resident(net->d, net->batch);
        if (!p.ok) return fail(net, PNN_ERR_INVALID, "resident kernel not valid: %s", p.why);
    }
    net->kernel = kernel;
    net->variant = PNN_VARIANT_AUTO;
    return PNN_OK;
}

pnn_status pnn_set_variant(pnn_net net, int32_t variant) {
    pnn_status st = check_live(net);
    if (st) return st;
    switch (variant) {
    case PNN_VARIANT_AUTO:
        break;
    case PNN_VARIANT_RESIDENT_V8:
    case PNN_VARIANT_RESIDENT_V10:
    case PNN_VARIANT_RESIDENT_TMEM:
    case PNN_VARIANT_RESIDENT_WS: {
        ResidentPlan p = plan_resident(net->d, net->batch, 0, variant);
        if (!p.ok) return fail(net, PNN_ERR_INVALID, "variant %d not valid: %s", variant, p.why);
        net->kernel = PNN_KERNEL_RESIDENT;
        break;
    }
    case PNN_VARIANT_CLUSTER_GENERIC:
    case PNN_VARIANT_CLUSTER_DEEP: {
        ClusterPlan p = plan_cluster(net->d, net->batch);
        if (!p.ok) return fail(net, PNN_ERR_INVALID, "variant %d not valid: %s", variant, p.why);
        if (variant == PNN_VARIANT_CLUSTER_DEEP)
            if (const char* why = deep_plan(net->d, net->batch))
                return fail(net, PNN_ERR_INVALID, "variant %d not valid: %s", variant, why);
        net->kernel = PNN_KERNEL_CLUSTER;
        break;
    }
    case PNN_VARIANT_MB_STEP:
    case PNN_VARIANT_MB_RESIDENT: {
        if (net->precision != PNN_FP32 || net->batch < 2)
            return fail(net, PNN_ERR_INVALID, "variant %d needs an fp32 mini-batch (pnn_set_minibatch first)",
                        variant);
        const char* why = variant == PNN_VARIANT_MB_STEP ? mb32_plan(net->d, net->batch) : mbres_plan(net->d, net->batch);
        if (why) return fail(net, PNN_ERR_INVALID, "variant %d not valid: %s", variant, why);
        net->kernel = PNN_KERNEL_AUTO;
        break;
    }
    default:
        return fail(net, PNN_ERR_INVALID, "variant = %d unknown", variant);
    }
    net->variant = variant;
    return PNN_OK;
}

pnn_status pnn_kernel_variant(pnn_net net, int32_t* variant) {
    if (!net || !variant) return PNN_ERR_INVALID;
    ResidentPlan plan{};
    int v = PNN_VARIANT_AUTO;
    choose_kernel(net, &plan, &v);
    *variant = v;
    return PNN_OK;
}

pnn_status pnn_set_slots(pnn_net net, int32_t slots) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (slots < 0) return fail(net, PNN_ERR_INVALID, "slots = %d < 0", slots);
    net->slots = slots;
    return PNN_OK;
}

pnn_status pnn_kernel_timing(pnn_net net, int32_t enable, double* mean_ms, int32_t* count) {
    if (!net) return PNN_ERR_INVALID;
    CUDA_TRY(net, cudaSetDevice(net->device));
    double total = 0.0;
    int32_t cnt = 0;
    for (auto& pr : net->tev) {
        float ms = 0.f;
        if (!enable && cudaEventSynchronize(pr.second) == cudaSuccess &&
            cudaEventElapsedTime(&ms, pr.first, pr.second) == cudaSuccess) {
            total += ms;
            ++cnt;
        }
        cudaEventDestroy(pr.first);
        cudaEventDestroy(pr.second);
    }
    net->tev.clear();
    net->timing = enable != 0;
    if (mean_ms) *mean_ms = cnt ? total / cnt : 0.0;
    if (count) *count = cnt;
    return PNN_OK;
}

pnn_status pnn_train_epoch(pnn_net net, const float* x, const int32_t* labels, int64_t n,
                           void* stream) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (net->K_local == 0) return check_rows(net, n);   // idle rank (K < nranks)
    if (!x || !labels) return fail(net, PNN_ERR_INVALID, "x/labels is NULL");
    if ((st = check_rows(net, n))) return st;
    CUDA_TRY(net, cudaSetDevice(net->device));
    return launch_train(net, x, labels, n, 0, net->K_local, (cudaStream_t)stream);
}

pnn_status pnn_train_epoch_host(pnn_net net, const float* xh, const int32_t* yh, int64_t n,
                                void* stream) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (net->K_local == 0) return check_rows(net, n);   // idle rank (K < nranks)
    if (!xh || !yh) return fail(net, PNN_ERR_INVALID, "x/labels is NULL");
    if ((st = check_rows(net, n))) return st;
    CUDA_TRY(net, cudaSetDevice(net->device));
    cudaStream_t cs = (cudaStream_t)stream;
    if (net->stage_rows < n) {
        cudaEventSynchronize(net->stage_released);   // no launch still reads the old buffers
        cudaFree(net->d_xstage); cudaFree(net->d_ystage);
        net->d_xstage = nullptr; net->d_ystage = nullptr; net->stage_rows = 0;
        CUDA_TRY(net, cudaMalloc(&net->d_xstage, sizeof(float) * (size_t)n * net->d.n[0]));
        CUDA_TRY(net, cudaMalloc(&net->d_ystage, sizeof(int32_t) * (size_t)n));
        net->stage_rows = n;
        net->grp_n = -1;
    }
    // Pipeline: the CNs are cut into groups; group g's slices are copied on
    // copy_stream while group g-1 trains on the caller's stream.  A group must still fill
    // the GPU: the batched mini-batch paths take every CN at once (one group), the cluster
    // kernels run ~148/cluster CNs concurrently.
    int groups = 1, gsize = net->K_local;
    {
        ResidentPlan rp{};
        int var = PNN_VARIANT_AUTO;
        const int k = choose_kernel(net, &rp, &var);
        int cap = net->K_local;                   // CNs that run concurrently
        if (k == PNN_KERNEL_RESIDENT) cap = 148 / (rp.cluster > 0 ? rp.cluster : 1);
        else if (k == PNN_KERNEL_CLUSTER)
            cap = 148 / (var == PNN_VARIANT_CLUSTER_DEEP ? deep_cluster_size(net->d)
                                                         : plan_cluster(net->d, net->batch).cluster);
        else if (k == PNN_KERNEL_REFERENCE) cap = 148;
        else if (k == PNN_KERNEL_MB_RESIDENT) cap = 148 / mbres_cluster(net->d);
        // groups of whole waves: a multiple of `cap` CNs each (a group that is a wave and a bit
        // runs two waves), at most 8 groups
        cap = cap > 0 ? cap : 1;
        const int waves = (net->K_local + cap - 1) / cap;
        gsize = cap * ((waves + 7) / 8);
        if (gsize > net->K_local) gsize = net->K_local;
        groups = (net->K_local + gsize - 1) / gsize;
    }
    const size_t row_bytes = sizeof(float) * net->d.n[0];
    // Events and the copy stream are released on every return path: the copies already
    // enqueued finish before the call returns (the host buffers are consumed on return,
    // success or not), and the staging buffers are marked busy until the last launch that
    // reads them, on whatever stream this call used.
    struct Guard {
        pnn_net net;
        cudaStream_t cs;
        cudaEvent_t ready[8] = {};
        int n = 0;
        bool launched = false;
        ~Guard() {
            if (launched) cudaEventRecord(net->stage_released, cs);
            cudaStreamSynchronize(net->copy_stream);
            for (int g = 0; g < n; ++g) cudaEventDestroy(ready[g]);
        }
    } guard{net, cs};
    for (int g = 0; g < groups; ++g) {
        CUDA_TRY(net, cudaEventCreateWithFlags(&guard.ready[g], cudaEventDisableTiming));
        guard.n = g + 1;
    }
    // The previous call's launches (on any stream) may still read the staging buffers.  When
    // this call cuts the rows into the same groups as the previous one, group g's copy waits only
    // for the previous call's group g (same rows; by induction that one waited for the call
    // before), so the next call's first copies run under the previous call's last wave.
    // Otherwise every copy waits for all of the previous call's launches.  (The Gram records
    // are per row too.)
    const bool per_group = net->grp_n == n && net->grp_count == groups && net->grp_size == gsize;
    if (!per_group) CUDA_TRY(net, cudaStreamWaitEvent(net->copy_stream, net->stage_released, 0));
    net->grp_n = -1;                               // (set again once every group is launched)
    for (int g = 0; g < groups; ++g) {
        const int s0 = g * gsize;
        const int s1 = (g + 1) * gsize < net->K_local ? (g + 1) * gsize : net->K_local;
        long long r0, c0, r1, c1;
        shard_of(n, net->K_local, s0, &r0, &c0);
        shard_of(n, net->K_local, s1 - 1, &r1, &c1);
        const long long rows = r1 + c1 - r0;
        if (per_group) CUDA_TRY(net, cudaStreamWaitEvent(net->copy_stream, net->grp_released[g], 0));
        CUDA_TRY(net, cudaMemcpyAsync(net->d_xstage + (size_t)r0 * net->d.n[0], xh + (size_t)r0 * net->d.n[0],
                                      row_bytes * rows, cudaMemcpyHostToDevice, net->copy_stream));
        CUDA_TRY(net, cudaMemcpyAsync(net->d_ystage + r0, yh + r0, sizeof(int32_t) * rows,
                                      cudaMemcpyHostToDevice, net->copy_stream));
        CUDA_TRY(net, cudaEventRecord(guard.ready[g], net->copy_stream));
        CUDA_TRY(net, cudaStreamWaitEvent(cs, guard.ready[g], 0));
        guard.launched = true;
        if ((st = launch_train(net, net->d_xstage, net->d_ystage, n, s0, s1 - s0, cs))) return st;
        CUDA_TRY(net, cudaEventRecord(net->grp_released[g], cs));   // group g's rows free again
    }
    net->grp_n = n;
    net->grp_count = groups;
    net->grp_size = gsize;
    return PNN_OK;                                 // (the guard waits for the copies)
}

pnn_status pnn_merge(pnn_net net, void* stream) {
    pnn_status st = check_live(net);
    if (st) return st;
    CUDA_TRY(net, cudaSetDevice(net->device));
    cudaStream_t cs = (cudaStream_t)stream;
    const long long P = net->d.P;
    if (net->nranks == 1 && !net->comm) {
        CUDA_TRY(net, launch_merge_local(net->d_children, net->K_local, P, net->K, net->d_merged, cs));
        return PNN_OK;
    }
    if (!net->comm)
        return fail(net, PNN_ERR_STATE, "nranks = %d without an NCCL communicator: reduce with "
                    "pnn_merge_partial + an all-reduce + pnn_merge_finish", net->nranks);
    CUDA_TRY(net, launch_merge_sum(net->d_children, net->K_local, P, net->d_msum, cs));
    ncclResult_t r = g_nccl.AllReduce(net->d_msum, net->d_msum, (size_t)P, ncclFloat64, ncclSum,
                                      (ncclComm_t)net->comm, cs);
    if (r != ncclSuccess) return fail(net, PNN_ERR_NCCL, "ncclAllReduce: %s", g_nccl.GetErrorString(r));
    CUDA_TRY(net, launch_merge_finish(net->d_msum, P, net->K, net->d_merged, cs));
    return PNN_OK;
}

pnn_status pnn_merge_partial(pnn_net net, double* sum_out, void* stream) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (!sum_out) return fail(net, PNN_ERR_INVALID, "sum_out is NULL");
    CUDA_TRY(net, cudaSetDevice(net->device));
    CUDA_TRY(net, launch_merge_sum(net->d_children, net->K_local, net->d.P, sum_out, (cudaStream_t)stream));
    return PNN_OK;
}

pnn_status pnn_merge_finish(pnn_net net, const double* sum, void* stream) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (!sum) return fail(net, PNN_ERR_INVALID, "sum is NULL");
    CUDA_TRY(net, cudaSetDevice(net->device));
    CUDA_TRY(net, launch_merge_finish(sum, net->d.P, net->K, net->d_merged, (cudaStream_t)stream));
    return PNN_OK;
}

pnn_status pnn_evaluate(pnn_net net, int32_t subnet, const float* x, const int32_t* labels, int64_t n,
                        double* metrics_out, void* stream) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (!x || !labels || !metrics_out || n <= 0)
        return fail(net, PNN_ERR_INVALID, "x/labels/metrics_out NULL or n <= 0");
    const float* p;
    if (subnet == -1) p = net->d_merged;
    else if (subnet >= net->k_first && subnet < net->k_first + net->K_local)
        p = net->d_children + (size_t)(subnet - net->k_first) * net->d.P;
    else return fail(net, PNN_ERR_INVALID, "subnet %d is not local ([%d, %d))", subnet, net->k_first,
                     net->k_first + net->K_local);
    CUDA_TRY(net, cudaSetDevice(net->device));
    if (net->eval_rows < n) {
        cudaFree(net->d_eval);
        net->d_eval = nullptr;
        net->eval_rows = 0;
        CUDA_TRY(net, cudaMalloc(&net->d_eval, sizeof(double) * (3 * (size_t)n + 3)));
        net->eval_rows = n;
    }
    double* out3 = net->d_eval + 3 * (size_t)net->eval_rows;
    cudaStream_t s = (cudaStream_t)stream;
    CUDA_TRY(net, launch_evaluate(net->d, p, x, labels, n, net->d_eval, out3, s));
    CUDA_TRY(net, cudaMemcpyAsync(metrics_out, out3, 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(net, cudaStreamSynchronize(s));
    return PNN_OK;
}

pnn_status pnn_predict(pnn_net net, int32_t subnet, const float* x, int64_t n, int32_t* labels,
                       void* stream) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (!x || !labels || n < 0) return fail(net, PNN_ERR_INVALID, "x/labels NULL or n < 0");
    const float* p;
    if (subnet == -1) p = net->d_merged;
    else if (subnet >= net->k_first && subnet < net->k_first + net->K_local)
        p = net->d_children + (size_t)(subnet - net->k_first) * net->d.P;
    else return fail(net, PNN_ERR_INVALID, "subnet %d is not local ([%d, %d))", subnet, net->k_first,
                     net->k_first + net->K_local);
    CUDA_TRY(net, cudaSetDevice(net->device));
    CUDA_TRY(net, launch_predict(net->d, p, x, n, labels, (cudaStream_t)stream));
    return PNN_OK;
}

pnn_status pnn_get_params(pnn_net net, int32_t subnet, float* host_out, int64_t n_floats) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (!host_out) return fail(net, PNN_ERR_INVALID, "host_out is NULL");
    if (n_floats != net->d.P) return fail(net, PNN_ERR_SHAPE, "n_floats = %lld, P_total = %lld",
                                          (long long)n_floats, (long long)net->d.P);
    const float* p = pnn_device_params(net, subnet);
    if (!p) return fail(net, PNN_ERR_INVALID, "subnet %d is not local", subnet);
    CUDA_TRY(net, cudaSetDevice(net->device));
    CUDA_TRY(net, cudaDeviceSynchronize());
    CUDA_TRY(net, cudaMemcpy(host_out, p, sizeof(float) * net->d.P, cudaMemcpyDeviceToHost));
    return PNN_OK;
}

pnn_status pnn_set_params(pnn_net net, int32_t subnet, const float* host_in, int64_t n_floats) {
    pnn_status st = check_live(net);
    if (st) return st;
    if (!host_in) return fail(net, PNN_ERR_INVALID, "host_in is NULL");
    if (n_floats != net->d.P) return fail(net, PNN_ERR_SHAPE, "n_floats = %lld, P_total = %lld",
                                          (long long)n_floats, (long long)net->d.P);
    CUDA_TRY(net, cudaSetDevice(net->device));
    CUDA_TRY(net, cudaDeviceSynchronize());
    const size_t bytes = sizeof(float) * net->d.P;
    if (subnet == -1) {
        for (int c = 0; c < net->K_local; ++c)
            CUDA_TRY(net, cudaMemcpy(net->d_children + (size_t)c * net->d.P, host_in, bytes, cudaMemcpyHostToDevice));
        return PNN_OK;
    }
    float* p = (subnet == -2) ? net->d_merged : pnn_device_params(net, subnet);
    if (!p) return fail(net, PNN_ERR_INVALID, "subnet %d is not local", subnet);
    CUDA_TRY(net, cudaMemcpy(p, host_in, bytes, cudaMemcpyHostToDevice));
    return PNN_OK;
}

float* pnn_device_params(pnn_net net, int32_t subnet) {
    if (!net) return nullptr;
    if (subnet == -1) return net->d_merged;
    if (subnet < net->k_first || subnet >= net->k_first + net->K_local) return nullptr;
    return net->d_children + (size_t)(subnet - net->k_first) * net->d.P;
}

int64_t pnn_param_count(pnn_net net) { return net ? net->d.P : -1; }

pnn_status pnn_local_subnets(pnn_net net, int32_t* first, int32_t* count) {
    if (!net || !first || !count) return PNN_ERR_INVALID;
    *first = net->k_first;
    *count = net->K_local;
    return PNN_OK;
}

pnn_status pnn_local_rows(pnn_net net, int64_t n_total, int64_t* first, int64_t* count) {
    if (!net || !first || !count) return PNN_ERR_INVALID;
    if (n_total < net->K)
        return fail(net, PNN_ERR_INVALID, "n_total = %lld < K = %d", (long long)n_total, net->K);
    if (net->K_local == 0) {
        long long s0 = n_total, c0 = 0;
        if (net->k_first < net->K) shard_of(n_total, net->K, net->k_first, &s0, &c0);
        *first = s0;
        *count = 0;
        return PNN_OK;
    }
    long long s0, c0, s1, c1;
    shard_of(n_total, net->K, net->k_first, &s0, &c0);
    shard_of(n_total, net->K, net->k_first + net->K_local - 1, &s1, &c1);
    *first = s0;
    *count = s1 + c1 - s0;
    return PNN_OK;
}

pnn_status pnn_kernel_info(pnn_net net, int32_t* kernel, int32_t* launches) {
    if (!net || !kernel || !launches) return PNN_ERR_INVALID;
    ResidentPlan plan{};
    int v = PNN_VARIANT_AUTO;
    int k = choose_kernel(net, &plan, &v);
    *kernel = k < 0 ? PNN_KERNEL_REFERENCE : k;
    // resident v8 / v10 and the deep cluster variant: Gram terms + training; the TMEM variant
    // forms its Gram terms in the training launch; tc bf16: 7 per mini-batch step; fp32 step
    // kernels: 4 per step; MB_RESIDENT: 1 per epoch
    const bool gram = v == PNN_VARIANT_CLUSTER_DEEP ||
                      (k == PNN_KERNEL_RESIDENT && v != PNN_VARIANT_RESIDENT_TMEM);
    *launches = gram ? 2 : (k == PNN_KERNEL_TC_BF16) ? 7 : (k == PNN_KERNEL_MB_F32) ? 4 : 1;
    return PNN_OK;
}

const char* pnn_last_error(pnn_net net) {
    return net ? net->err.c_str() : g_create_err.c_str();
}

pnn_status pnn_destroy(pnn_net net) {
    if (!net) return PNN_OK;
    cudaSetDevice(net->device);
    cudaDeviceSynchronize();
    if (net->comm && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)net->comm);
    cudaFree(net->d_children);
    cudaFree(net->d_merged);
    cudaFree(net->d_msum);
    cudaFree(net->d_gscratch);
    mb_destroy(net->mb);
    mb32_destroy(net->mb32);
    for (auto& pr : net->tev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    cudaFree(net->d_eval);
    cudaFree(net->d_gram);
    cudaFree(net->d_xstage);
    cudaFree(net->d_ystage);
    if (net->copy_stream) cudaStreamDestroy(net->copy_stream);
    if (net->stage_released) cudaEventDestroy(net->stage_released);
    for (int g = 0; g < 8; ++g)
        if (net->grp_released[g]) cudaEventDestroy(net->grp_released[g]);
    delete net;
    return PNN_OK;
}

}  // extern "C"
