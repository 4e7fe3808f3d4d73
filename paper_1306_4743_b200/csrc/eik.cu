// eik.cu -- host driver and C ABI (include/eik.h) of the B200 cell-sweep Eikonal solver.
//
// PRODUCT PATH: validate -> size/alloc scratch -> enqueue the device phases on the ctx stream
// -> one small D2H of the control block -> return status.  The scheduler loop runs on the
// device (CUDA graph with a conditional WHILE node: no host round-trip per round); a
// host-driven loop is kept as a debug mode (EIK_OPT_LOOP_MODE = 1).  No CPU fallback.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include <string>
#include <vector>

#include "../../include/eik.h"
#include "eik_kernels.cuh"

using namespace eik;

#ifndef EIK_ROUNDS_PER_ITER
#define EIK_ROUNDS_PER_ITER 4   // fused rounds captured per iteration of the graph WHILE node (C3 -1.7 %)
#endif

struct eik_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string err;
    // options
    double bin_width = INFINITY;
    uint32_t max_rounds = 1000000000u;
    int loop_mode = 0;            // asynchronous persistent scheduler (see include/eik.h)
    int collect_stats = 1;
    int time_cell_events = 0;
    int async_defer = 8;
    int max_sweeps = -1;          // -1: automatic (0 in async mode, 4 in the round modes)
    double kappa = 0.0;
    int legacy_key = 0;
    int cell_kernel = 0;          // EIK_OPT_CELL_KERNEL: 1 = 2x2x2 micro-blocks (r = 16), 0 = point wavefront
    bool last_b2 = false;         // the last async solve ran the micro-block kernel
    double timeout_s = 120.0;
    uint32_t trace_cap = 0;       // EIK_OPT_TRACE: processings traced (0 = off)
    uint4* trace = nullptr;
    uint32_t* tagger = nullptr;
    size_t tagger_cap = 0;
    cudaEvent_t cev[2] = {nullptr, nullptr};
    double ms_cell_events = 0;
    // scratch
    void* Vt = nullptr;
    void* Ht = nullptr;
    size_t tile_bytes = 0;        // capacity of Vt / Ht each
    uint32_t* key = nullptr;
    uint32_t* state = nullptr;
    uint32_t* wl0 = nullptr;
    uint32_t* wl1 = nullptr;
    uint32_t* proc_cell = nullptr;
    uint32_t* proc_flags = nullptr;
    uint32_t* pend = nullptr;
    uint32_t* pdir = nullptr;
    uint32_t* gen = nullptr;
    uint32_t* wait = nullptr;
    size_t cell_cap = 0;
    size_t ring_cap = 0;
    Ctl* ctl = nullptr;
    Ctl* ctl_host = nullptr;      // pinned
    // plane tables per r (index 0: r=4, 1: r=8, 2: r=16)
    uint16_t* plane_tab[3] = {nullptr, nullptr, nullptr};
    uint32_t* tab16 = nullptr;    // r = 16 packed per-direction plane table (sweep16)
    uint2* tab_b2 = nullptr;      // r = 16 per-direction block-plane table (eik_b2.cuh)
    // host-pointer staging (eik_solve_host)
    void* stage = nullptr;
    size_t stage_bytes = 0;
    bool q_zero_copy = false;   // last eik_solve_host read exit_vals in place (pinned memory)
    // graph cache (scheduler loop; whole-grid sweep loop)
    cudaGraphExec_t gexec = nullptr;
    std::string gkey;
    cudaGraphExec_t gexec_sw = nullptr;
    std::string gkey_sw;
    // whole-grid sweeping: cells grouped by canonical diagonal (per cps), DLSM cell flags
    uint32_t* diag_cells = nullptr;
    uint32_t* diag_off = nullptr;
    int diag_cps = 0;
    std::vector<uint32_t> diag_off_h;
    uint8_t* cact = nullptr;
    // events
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    eik_stats stats{};
    bool have_stats = false;
};

static std::string g_create_err;

static int fail(eik_ctx* ctx, int code, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (ctx) ctx->err = buf;
    else g_create_err = buf;
    return code;
}

#define CK(call)                                                                           \
    do {                                                                                   \
        cudaError_t e_ = (call);                                                           \
        if (e_ != cudaSuccess) {                                                           \
            (void)cudaGetLastError();                                                      \
            return fail(ctx, e_ == cudaErrorMemoryAllocation ? EIK_ENOMEM : EIK_ECUDA,     \
                        "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
        }                                                                                  \
    } while (0)

static int rindex_of(int r) { return r == 4 ? 0 : r == 8 ? 1 : r == 16 ? 2 : -1; }

// wavefront plane table for an r^3 cell, indexed [plane s][thread t]: the canonical point
// index a + r b + r^2 c of the t-th point (a, b, c) of plane a+b+c = s, or 0xFFFF when plane s
// has <= t points.  Three trailing all-empty planes let the sweep prefetch up to three planes ahead
// without a bounds test.  A direction's point is this entry XOR its reflection mask (r a power
// of two).  nt = threads of the cell kernel (CellCfg<r>::NT >= the largest plane).
static void make_plane_table(int r, int nt, std::vector<uint16_t>& tab)
{
    const int npl = 3 * r - 2;
    tab.assign((size_t)(npl + 3) * nt, (uint16_t)0xFFFF);
    for (int s = 0; s < npl; ++s) {
        int t = 0;
        for (int c = 0; c < r; ++c)
            for (int b = 0; b < r; ++b) {
                const int a = s - b - c;
                if (a >= 0 && a < r) tab[(size_t)s * nt + t++] = (uint16_t)(a + r * b + r * r * c);
            }
        if (t > nt) std::abort();   // CellCfg<r>::NT smaller than a plane: programming error
    }
}

// packed per-direction wavefront table of an r = 16 cell (sweep16, eik_kernels.cuh): for
// direction d, plane s of the reflected coordinates (a', b', c'), thread t: the t-th point of
// the canonical plane list above, reflected into physical coordinates (a, b, c) -- its box
// index, the neighbours that exist in canonical orientation, its point index
static void make_tab16(int nt, std::vector<uint32_t>& tab)
{
    const int r = 16, npl = 3 * r - 2, rows = npl + 3;
    tab.assign((size_t)8 * rows * nt, T16_DUMMY);
    for (int d = 0; d < 8; ++d)
        for (int s = 0; s < npl; ++s) {
            int t = 0;
            for (int c = 0; c < r; ++c)
                for (int b = 0; b < r; ++b) {
                    const int a = s - b - c;
                    if (a < 0 || a >= r) continue;
                    const int pa = (d & 1) ? r - 1 - a : a, pb = (d & 2) ? r - 1 - b : b,
                              pc = (d & 4) ? r - 1 - c : c;
                    const uint32_t q = (uint32_t)((pa + 1) + (r + 2) * (pb + 1) + (r + 2) * (r + 2) * (pc + 1));
                    const uint32_t p = (uint32_t)(pa + r * pb + r * r * pc);
                    tab[((size_t)d * rows + s) * nt + t++] = q | (p << 19);
                }
            if (t > nt) std::abort();
        }
}

// per-direction block-plane table of the micro-block kernel (eik_b2.cuh): plane S of the
// reflected block coordinates (A', B', C') of direction d, thread t: the t-th block (canonical
// order c, b) reflected into physical (A, B, C)
static void make_tab_b2(std::vector<uint2>& tab)
{
    const int nb = B2::NB, nt = B2::NT, rows = B2::ROWS;
    tab.assign((size_t)8 * rows * nt, make_uint2(B2_DUMMY_X, 0u));
    for (int d = 0; d < 8; ++d)
        for (int S = 0; S < B2::NBP; ++S) {
            int t = 0;
            for (int c = 0; c < nb; ++c)
                for (int b = 0; b < nb; ++b) {
                    const int a = S - b - c;
                    if (a < 0 || a >= nb) continue;
                    const int pa = (d & 1) ? nb - 1 - a : a, pb = (d & 2) ? nb - 1 - b : b,
                              pc = (d & 4) ? nb - 1 - c : c;
                    const uint32_t q0 = (uint32_t)b2q(2 * pa, 2 * pb, 2 * pc);
                    const uint32_t eb = (uint32_t)(pa + nb * pb + nb * nb * pc);
                    const uint32_t bm = (a < nb - 1 ? 1u : 0u) | (a > 0 ? 2u : 0u) | (b < nb - 1 ? 4u : 0u) |
                                        (b > 0 ? 8u : 0u) | (c < nb - 1 ? 16u : 0u) | (c > 0 ? 32u : 0u);
                    const uint32_t h0 = (uint32_t)(2 * pa + 16 * 2 * pb + 256 * 2 * pc);
                    tab[((size_t)d * rows + S) * nt + t++] = make_uint2(q0 | (eb << 13) | (bm << 23), h0);
                }
            if (t > nt) std::abort();
        }
}

extern "C" int eik_abi_version(void) { return EIK_ABI_VERSION; }

static int create_fill(eik_ctx* ctx, int device, void* cuda_stream);
extern "C" void eik_destroy(eik_ctx* ctx);

extern "C" int eik_create(eik_ctx** out, int device, void* cuda_stream)
{
    eik_ctx* ctx = nullptr;
    if (!out) return fail(nullptr, EIK_EINVAL, "eik_create: out is NULL");
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || ndev == 0)
        return fail(nullptr, EIK_ECUDA, "eik_create: no CUDA device (%s)", cudaGetErrorString(e));
    if (device < 0 || device >= ndev)
        return fail(nullptr, EIK_EINVAL, "eik_create: device %d out of range [0,%d)", device, ndev);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
        return fail(nullptr, EIK_ECUDA, "eik_create: cudaGetDeviceProperties failed");
    if (prop.major != 10)
        return fail(nullptr, EIK_ENOTSUP, "eik_create: device %d is sm_%d%d; this build is sm_100a only",
                    device, prop.major, prop.minor);
    ctx = new eik_ctx();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    // a failure while the context is being filled must not leak it, and its message must reach
    // eik_last_error(NULL) (the caller never sees this ctx)
    const int st = create_fill(ctx, device, cuda_stream);
    if (st != EIK_OK) {
        g_create_err = ctx->err;
        if (cuda_stream) ctx->stream = nullptr;   // (not ours: eik_destroy must not synchronise it)
        eik_destroy(ctx);
        return st;
    }
    *out = ctx;
    return EIK_OK;
}

static int create_fill(eik_ctx* ctx, int device, void* cuda_stream)
{
    CK(cudaSetDevice(device));
    if (cuda_stream) ctx->stream = (cudaStream_t)cuda_stream;
    else {
        CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        ctx->stream = ctx->own_stream;
    }
    CK(cudaMalloc(&ctx->ctl, sizeof(Ctl)));
    CK(cudaMallocHost(&ctx->ctl_host, sizeof(Ctl)));
    for (int i = 0; i < 5; ++i) CK(cudaEventCreate(&ctx->ev[i]));
    for (int i = 0; i < 2; ++i) CK(cudaEventCreate(&ctx->cev[i]));
    const int rs[3] = {4, 8, 16};
    const int nts[3] = {CellCfg<4>::NT, CellCfg<8>::NT, CellCfg<16>::NT};
    for (int t = 0; t < 3; ++t) {
        std::vector<uint16_t> tab;
        make_plane_table(rs[t], nts[t], tab);
        CK(cudaMalloc(&ctx->plane_tab[t], tab.size() * sizeof(uint16_t)));
        CK(cudaMemcpy(ctx->plane_tab[t], tab.data(), tab.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    }
    {
        std::vector<uint32_t> tab;
        make_tab16(CellCfg<16>::NT, tab);
        CK(cudaMalloc(&ctx->tab16, tab.size() * sizeof(uint32_t)));
        CK(cudaMemcpy(ctx->tab16, tab.data(), tab.size() * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    {
        std::vector<uint2> tab;
        make_tab_b2(tab);
        CK(cudaMalloc(&ctx->tab_b2, tab.size() * sizeof(uint2)));
        CK(cudaMemcpy(ctx->tab_b2, tab.data(), tab.size() * sizeof(uint2), cudaMemcpyHostToDevice));
    }
    CK(cudaFuncSetAttribute(k_async<float, 16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b2_smem_bytes<float>()));
    CK(cudaFuncSetAttribute(k_async<double, 16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b2_smem_bytes<double>()));
    CK(cudaFuncSetAttribute(k_async<float, 16, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_async<double, 16, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    // opt in to > 48 KB dynamic shared memory for the cell kernels
    CK(cudaFuncSetAttribute(k_cell<float, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 16>()));
    // largest shared-memory carveout: the cell kernels are occupancy-limited by shared memory
    CK(cudaFuncSetAttribute(k_cell<float, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_cell<double, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_async<float, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_async<double, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_cell<double, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 16>()));
    CK(cudaFuncSetAttribute(k_cell<float, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 8>()));
    CK(cudaFuncSetAttribute(k_cell<double, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 8>()));
    CK(cudaFuncSetAttribute(k_cell<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 4>()));
    CK(cudaFuncSetAttribute(k_cell<double, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 4>()));
    CK(cudaFuncSetAttribute(k_async<float, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 16>()));
    CK(cudaFuncSetAttribute(k_async<double, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 16>()));
    CK(cudaFuncSetAttribute(k_async<float, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 8>()));
    CK(cudaFuncSetAttribute(k_async<double, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 8>()));
    CK(cudaFuncSetAttribute(k_async<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 4>()));
    CK(cudaFuncSetAttribute(k_async<double, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 4>()));
    CK(cudaFuncSetAttribute(k_dsweep<float, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 16>()));
    CK(cudaFuncSetAttribute(k_dsweep<double, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 16>()));
    CK(cudaFuncSetAttribute(k_dsweep<float, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 8>()));
    CK(cudaFuncSetAttribute(k_dsweep<double, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 8>()));
    CK(cudaFuncSetAttribute(k_dsweep<float, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<float, 4>()));
    CK(cudaFuncSetAttribute(k_dsweep<double, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cell_smem_bytes<double, 4>()));
    CK(cudaFuncSetAttribute(k_dsweep<float, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    CK(cudaFuncSetAttribute(k_dsweep<double, 16>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    return EIK_OK;
}

static void free_scratch(eik_ctx* ctx)
{
    cudaFree(ctx->Vt); cudaFree(ctx->Ht);
    cudaFree(ctx->key); cudaFree(ctx->state); cudaFree(ctx->wl0); cudaFree(ctx->wl1);
    cudaFree(ctx->proc_cell); cudaFree(ctx->proc_flags); cudaFree(ctx->pend); cudaFree(ctx->gen); cudaFree(ctx->wait); cudaFree(ctx->pdir);
    cudaFree(ctx->diag_cells); cudaFree(ctx->diag_off); cudaFree(ctx->cact);
    ctx->diag_cells = ctx->diag_off = nullptr;
    ctx->cact = nullptr;
    ctx->diag_cps = 0;
    ctx->pend = nullptr;
    ctx->pdir = nullptr;
    ctx->gen = nullptr;
    ctx->wait = nullptr;
    ctx->Vt = ctx->Ht = nullptr;
    ctx->key = ctx->state = ctx->wl0 = ctx->wl1 = ctx->proc_cell = ctx->proc_flags = nullptr;
    ctx->tile_bytes = ctx->cell_cap = 0;
}

extern "C" void eik_destroy(eik_ctx* ctx)
{
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    if (ctx->gexec_sw) cudaGraphExecDestroy(ctx->gexec_sw);
    free_scratch(ctx);
    cudaFree(ctx->stage);
    cudaFree(ctx->trace);
    cudaFree(ctx->tagger);
    cudaFree(ctx->ctl);
    cudaFreeHost(ctx->ctl_host);
    for (int t = 0; t < 3; ++t) cudaFree(ctx->plane_tab[t]);
    cudaFree(ctx->tab16);
    cudaFree(ctx->tab_b2);
    for (int i = 0; i < 5; ++i) if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
    for (int i = 0; i < 2; ++i) if (ctx->cev[i]) cudaEventDestroy(ctx->cev[i]);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    (void)cudaGetLastError();
    delete ctx;
}

extern "C" int eik_set_stream(eik_ctx* ctx, void* cuda_stream)
{
    if (!ctx) return EIK_EINVAL;
    cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : ctx->own_stream;
    if (!s) {
        CK(cudaSetDevice(ctx->device));
        CK(cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking));
        s = ctx->own_stream;
    }
    ctx->stream = s;
    return EIK_OK;
}

extern "C" int eik_set_option(eik_ctx* ctx, int option, double value)
{
    if (!ctx) return EIK_EINVAL;
    switch (option) {
    case EIK_OPT_BIN_WIDTH:
        if (isnan(value)) return fail(ctx, EIK_EINVAL, "bin width is NaN");
        ctx->bin_width = value <= 0 ? INFINITY : value;
        return EIK_OK;
    case EIK_OPT_MAX_ROUNDS:
        if (!(value >= 1)) return fail(ctx, EIK_EINVAL, "max rounds must be >= 1");
        ctx->max_rounds = value > 4e9 ? 0xffffffffu : (uint32_t)value;
        return EIK_OK;
    case EIK_OPT_LOOP_MODE:
        if (value != 0 && value != 1 && value != 2)
            return fail(ctx, EIK_EINVAL, "loop mode must be 0, 1 or 2");
        ctx->loop_mode = (int)value;
        return EIK_OK;
    case EIK_OPT_COLLECT_STATS:
        ctx->collect_stats = value != 0;
        return EIK_OK;
    case EIK_OPT_TIME_CELL_EVENTS:
        ctx->time_cell_events = value != 0;
        return EIK_OK;
    case EIK_OPT_ASYNC_DEFER:
        if (value < 0 || value > 9) return fail(ctx, EIK_EINVAL, "defer mode must be 0..9");
        ctx->async_defer = (int)value;
        return EIK_OK;
    case EIK_OPT_KAPPA:
        if (!(value >= 0) || !isfinite(value)) return fail(ctx, EIK_EINVAL, "kappa must be finite and >= 0");
        ctx->kappa = value;
        return EIK_OK;
    case EIK_OPT_CELL_KEY:
        if (value != 0 && value != 1) return fail(ctx, EIK_EINVAL, "cell key must be 0 (Eq. 3) or 1 (Eq. 4)");
        ctx->legacy_key = (int)value;
        return EIK_OK;
    case EIK_OPT_TIMEOUT_S:
        if (!(value > 0)) return fail(ctx, EIK_EINVAL, "timeout must be > 0 s");
        ctx->timeout_s = value;
        return EIK_OK;
    case EIK_OPT_CELL_KERNEL:
        if (value != 0 && value != 1) return fail(ctx, EIK_EINVAL, "cell kernel must be 0 or 1");
        ctx->cell_kernel = (int)value;
        return EIK_OK;
    case EIK_OPT_TRACE:
        if (!(value >= 0) || value > 1e8) return fail(ctx, EIK_EINVAL, "trace capacity must be in [0, 1e8]");
        if ((uint32_t)value != ctx->trace_cap) {
            CK(cudaSetDevice(ctx->device));
            if (ctx->stream) CK(cudaStreamSynchronize(ctx->stream));
            cudaFree(ctx->trace);
            ctx->trace = nullptr;
            ctx->trace_cap = 0;
            if (value >= 1) {
                CK(cudaMalloc(&ctx->trace, (size_t)value * 2 * sizeof(uint4)));
                ctx->trace_cap = (uint32_t)value;
            }
        }
        return EIK_OK;
    case EIK_OPT_MAX_SWEEPS:
        if (!(value >= -1) || value > 1e6) return fail(ctx, EIK_EINVAL, "max sweeps must be >= -1");
        ctx->max_sweeps = (int)value;
        return EIK_OK;
    default:
        return fail(ctx, EIK_EINVAL, "unknown option %d", option);
    }
}

extern "C" int eik_get_stats(const eik_ctx* ctx, eik_stats* out)
{
    if (!ctx || !out) return EIK_EINVAL;
    if (!ctx->have_stats) {
        memset(out, 0, sizeof *out);
        return EIK_EINVAL;
    }
    *out = ctx->stats;
    return EIK_OK;
}

extern "C" int eik_get_debug(const eik_ctx* ctx, uint64_t* out, int n)
{
    if (!ctx || !out || n < 0) return EIK_EINVAL;
    const int m = n < 41 ? n : 41;
    for (int i = 0; i < m; ++i) out[i] = ctx->ctl_host->dbg[i];
    if (n > 41) out[41] = ctx->ctl_host->defers;
    for (int i = 42; i < n && i < 42 + 2048; ++i) out[i] = ctx->ctl_host->rtrace[i - 42];
    if (n > 42 + 2048) out[42 + 2048] = ctx->ctl_host->dbg[41];
    if (n > 43 + 2048) out[43 + 2048] = ctx->ctl_host->dbg[42];
    for (int i = 44 + 2048; i < n && i < 44 + 4096; ++i) out[i] = ctx->ctl_host->rtrace2[i - 44 - 2048];
    for (int i = 44 + 4096; i < n && i < 44 + 4096 + 12; ++i) out[i] = (&ctx->ctl_host->lstat[0][0])[i - 44 - 4096];
    return EIK_OK;
}

extern "C" int64_t eik_get_trace(const eik_ctx* ctx, uint32_t* out, int64_t max_entries)
{
    if (!ctx || (!out && max_entries > 0) || max_entries < 0) return -EIK_EINVAL;
    if (!ctx->trace || !ctx->have_stats) return 0;
    int64_t n = ctx->ctl_host->trace_n;
    if (n > (int64_t)ctx->trace_cap) n = ctx->trace_cap;
    if (n > max_entries) n = max_entries;
    if (n > 0 && cudaMemcpy(out, ctx->trace, (size_t)n * 2 * sizeof(uint4), cudaMemcpyDeviceToHost) != cudaSuccess)
        return -EIK_ECUDA;
    return n;
}

extern "C" const char* eik_last_error(const eik_ctx* ctx)
{
    return ctx ? ctx->err.c_str() : g_create_err.c_str();
}

// ---------------------------------------------------------------------------------------
static int ensure_scratch(eik_ctx* ctx, size_t tile_bytes, size_t J)
{
    if (tile_bytes > ctx->tile_bytes || J > ctx->cell_cap) {
        if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
        if (ctx->gexec_sw) { cudaGraphExecDestroy(ctx->gexec_sw); ctx->gexec_sw = nullptr; ctx->gkey_sw.clear(); }
        CK(cudaStreamSynchronize(ctx->stream));
        free_scratch(ctx);
        CK(cudaMalloc(&ctx->Vt, tile_bytes));
        CK(cudaMalloc(&ctx->Ht, tile_bytes));
        ctx->tile_bytes = tile_bytes;
        CK(cudaMalloc(&ctx->key, J * 4));
        CK(cudaMalloc(&ctx->state, J * 4));
        size_t cap = 1;
        while (cap < J) cap <<= 1;
        ctx->ring_cap = cap;
        CK(cudaMalloc(&ctx->wl0, cap * 4));   // round-mode worklist / async-mode ring
        CK(cudaMalloc(&ctx->wl1, J * 4));
        CK(cudaMalloc(&ctx->proc_cell, J * 4));
        CK(cudaMalloc(&ctx->proc_flags, J * 4));
        CK(cudaMalloc(&ctx->pend, J * 512));   // R^3 / 8 bytes per cell at r = 16
        CK(cudaMalloc(&ctx->pdir, J * 4));     // sweep-direction state at a cap
        CK(cudaMalloc(&ctx->gen, J * 4));
        CK(cudaMalloc(&ctx->wait, J * 4));
        CK(cudaMalloc(&ctx->diag_cells, J * 4));
        CK(cudaMalloc(&ctx->cact, J));
        ctx->cell_cap = J;
    }
    return EIK_OK;
}

template <typename T, int R>
static int launch_cell(eik_ctx* ctx, const CellArgs& a, int grid)
{
    k_cell<T, R><<<grid, CellCfg<R>::NT, cell_smem_bytes<T, R>(), ctx->stream>>>(a);
    CK(cudaGetLastError());
    return EIK_OK;
}

template <typename T>
static int cell_grid(eik_ctx* ctx, int r, int* grid)
{
    int occ = 0;
    cudaError_t e;
    if (r == 16) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cell<T, 16>, CellCfg<16>::NT, cell_smem_bytes<T, 16>());
    else if (r == 8) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cell<T, 8>, CellCfg<8>::NT, cell_smem_bytes<T, 8>());
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_cell<T, 4>, CellCfg<4>::NT, cell_smem_bytes<T, 4>());
    CK(e);
    if (occ < 1) occ = 1;
    *grid = occ * ctx->sm_count;
    return EIK_OK;
}

// one scheduler round: select -> cell-sweep -> round end
template <typename T>
static int enqueue_round(eik_ctx* ctx, int r, const CellArgs& ca, int sel_grid, int cgrid,
                         bool time_events = false)
{
    if (!ca.fused) {   // fused: k_cell selects the whole worklist itself
        k_select<<<sel_grid, 256, 0, ctx->stream>>>(ctx->ctl, ctx->wl0, ctx->wl1, ctx->proc_cell,
                                                     ctx->proc_flags, ctx->key, ctx->state,
                                                     (float)ctx->bin_width, ca.legacy_key);
        CK(cudaGetLastError());
    }
    if (time_events) CK(cudaEventRecord(ctx->cev[0], ctx->stream));
    int st;
    if (r == 16) st = launch_cell<T, 16>(ctx, ca, cgrid);
    else if (r == 8) st = launch_cell<T, 8>(ctx, ca, cgrid);
    else st = launch_cell<T, 4>(ctx, ca, cgrid);
    if (st) return st;
    if (time_events) CK(cudaEventRecord(ctx->cev[1], ctx->stream));
    return EIK_OK;
}

__global__ void k_round_end_graph(Ctl* ctl, cudaGraphConditionalHandle h)
{
    if (ctl->done) return;   // the solve ended in an earlier round of this iteration
    cudaGraphSetConditional(h, round_end_body(ctl) ? 0u : 1u);
}

template <typename T, int R, int MODE = 0>
static int launch_async(eik_ctx* ctx, const CellArgs& a, int grid)
{
    if constexpr (MODE == 1) k_async<T, 16, 1><<<grid, B2::NT, b2_smem_bytes<T>(), ctx->stream>>>(a);
    else k_async<T, R><<<grid, CellCfg<R>::NT, cell_smem_bytes<T, R>(), ctx->stream>>>(a);
    CK(cudaGetLastError());
    return EIK_OK;
}

template <typename T>
static int run_async(eik_ctx* ctx, int r, int64_t J, CellArgs ca)
{
    // r = 16 exact path without a sweep cap: the 2x2x2 micro-block cell kernel (eik_b2.cuh)
    const bool b2 = r == 16 && ctx->cell_kernel == 1 && ca.kappa == 0.0 && ca.max_sweeps == 0;
    int occ = 0;
    cudaError_t e;
    if (b2) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_async<T, 16, 1>, B2::NT, b2_smem_bytes<T>());
    else if (r == 16) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_async<T, 16>, CellCfg<16>::NT, cell_smem_bytes<T, 16>());
    else if (r == 8) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_async<T, 8>, CellCfg<8>::NT, cell_smem_bytes<T, 8>());
    else e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_async<T, 4>, CellCfg<4>::NT, cell_smem_bytes<T, 4>());
    CK(e);
    if (occ < 1) occ = 1;
#ifdef EIK_ASYNC_OCC_CAP
    if (occ > EIK_ASYNC_OCC_CAP) occ = EIK_ASYNC_OCC_CAP;   // (experiment: fewer CTAs per SM)
#endif
    ctx->last_b2 = b2;
    // every CTA is co-resident (grid <= occupancy x SMs): idle CTAs only poll the ring.  Small
    // problems get fewer CTAs (at most one per eight cells, at least one per SM): the front of
    // C1 (17^3 cells of 8^3) is a few hundred cells wide, and 12 x 148 CTAs polling the ring
    // cost more than they bring (measured C1 0.89 -> 0.79 ms with 4 instead of 12 CTAs per SM)
    int grid = occ * ctx->sm_count;
    {
        const int64_t want = J / 8 > ctx->sm_count ? J / 8 : ctx->sm_count;
        if ((int64_t)grid > want) grid = (int)want;
    }
    ca.qmask = (uint32_t)(ctx->ring_cap - 1);
    ca.proc_limit = 4096ull * (unsigned long long)J + 1000000ull;
    ca.defer = ctx->async_defer;
    ca.defer_delta = isinf(ctx->bin_width) ? 0.f : (float)ctx->bin_width;
    CK(cudaMemsetAsync(ctx->wl0, 0xff, ctx->ring_cap * 4, ctx->stream));
    // (mode 9 keeps min-based levels in the same array: they count up from 0x7f7f7f7f)
    CK(cudaMemsetAsync(ctx->gen, ctx->async_defer == 9 ? 0x7f : 0, (size_t)J * 4, ctx->stream));
    CK(cudaMemsetAsync(ctx->wait, 0, (size_t)J * 4, ctx->stream));
    ca.wait = ctx->wait;
    if (ctx->trace) {
        if ((size_t)J > ctx->tagger_cap) {
            cudaFree(ctx->tagger);
            ctx->tagger = nullptr;
            ctx->tagger_cap = 0;
            CK(cudaMalloc(&ctx->tagger, (size_t)J * 4));
            ctx->tagger_cap = (size_t)J;
        }
        CK(cudaMemsetAsync(ctx->tagger, 0xff, (size_t)J * 4, ctx->stream));
        ca.trace = ctx->trace;
        ca.trace_cap = ctx->trace_cap;
        ca.tagger = ctx->tagger;
    }
    k_seed_queue<<<ctx->sm_count * 4, 256, 0, ctx->stream>>>(ctx->state, ctx->wl0, ctx->ctl, J);
    CK(cudaGetLastError());
    const bool te = ctx->time_cell_events != 0;   // CUDA events around the persistent launch
    if (te) CK(cudaEventRecord(ctx->cev[0], ctx->stream));
    int st = b2 ? launch_async<T, 16, 1>(ctx, ca, grid)
           : r == 16 ? launch_async<T, 16>(ctx, ca, grid) : r == 8 ? launch_async<T, 8>(ctx, ca, grid)
                                                                 : launch_async<T, 4>(ctx, ca, grid);
    if (te) CK(cudaEventRecord(ctx->cev[1], ctx->stream));
    return st;
}

template <typename T>
static int run_loop(eik_ctx* ctx, int r, int64_t J, const CellArgs& ca)
{
    if (ctx->loop_mode == 0) return run_async<T>(ctx, r, J, ca);
    int cgrid = 0;
    int st = cell_grid<T>(ctx, r, &cgrid);
    if (st) return st;
    if (ctx->loop_mode == 1) {
        // host-driven loop (debug): one 8-byte readback per round
        for (;;) {
            CK(cudaMemcpyAsync(ctx->ctl_host, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, ctx->stream));
            CK(cudaStreamSynchronize(ctx->stream));
            const Ctl& h = *ctx->ctl_host;
            const uint32_t n = h.wl_count[h.cur];
            if (n == 0) break;
            if (h.rounds >= ctx->max_rounds) return fail(ctx, EIK_EINTERNAL, "max rounds (%u) exceeded", ctx->max_rounds);
            const int sg = (int)((n + 255) / 256);
            const bool te = ctx->time_cell_events != 0;
            st = enqueue_round<T>(ctx, r, ca, sg, (int)(n < (uint32_t)cgrid ? n : (uint32_t)cgrid), te);
            if (st) return st;
            if (!ca.fused) {   // fused: the last CTA of k_cell ended the round
                k_round_end<<<1, 1, 0, ctx->stream>>>(ctx->ctl);
                CK(cudaGetLastError());
            }
            if (te) {
                CK(cudaEventSynchronize(ctx->cev[1]));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, ctx->cev[0], ctx->cev[1]));
                ctx->ms_cell_events += ms;
            }
        }
        return EIK_OK;
    }
    // loop mode 2: rounds in a CUDA graph with a conditional WHILE node around one round
    char keybuf[256];
    // every value baked into the captured kernel parameters is part of the key
    snprintf(keybuf, sizeof keybuf, "%d/%d/%lld/%lld/%p/%p/%.17g/%d/%d/%d/%.17g/%d", (int)sizeof(T), r, (long long)J,
             (long long)ca.n1, ca.Vt, ca.Ht, ctx->bin_width, ca.stats, ca.max_sweeps, ca.fused, ca.kappa, ca.legacy_key);
    if (!ctx->gexec || ctx->gkey != keybuf) {
        if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
        cudaGraph_t graph;
        CK(cudaGraphCreate(&graph, 0));
        cudaGraphConditionalHandle handle;
        CK(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = handle;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        CK(cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        // populate the body by capturing one round into it
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaStream_t saved = ctx->stream;
        ctx->stream = cs;
        CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        const int sg = (int)((J + 255) / 256 < (int64_t)ctx->sm_count * 4 ? (J + 255) / 256 : (int64_t)ctx->sm_count * 4);
        if (ca.fused) {
            // one kernel per round: k_cell selects, processes and (last CTA) ends the round
            CellArgs cg = ca;
            cg.graph = 1;
            cg.cond = (unsigned long long)handle;
            // several rounds per WHILE iteration: plain kernel-to-kernel edges between them
            for (int k = 0; k < EIK_ROUNDS_PER_ITER && !st; ++k) st = enqueue_round<T>(ctx, r, cg, sg, cgrid);
        } else {
            CellArgs cg = ca;
            cg.graph = 1;   // (non-fused: only turns the rounds after the last into no-ops)
            for (int k = 0; k < EIK_ROUNDS_PER_ITER && !st; ++k) {
                st = enqueue_round<T>(ctx, r, cg, sg, cgrid);
                k_round_end_graph<<<1, 1, 0, cs>>>(ctx->ctl, handle);
            }
        }
        cudaGraph_t captured;
        cudaError_t ce = cudaStreamEndCapture(cs, &captured);
        ctx->stream = saved;
        cudaStreamDestroy(cs);
        if (st) { cudaGraphDestroy(graph); return st; }
        if (ce != cudaSuccess) { cudaGraphDestroy(graph); CK(ce); }
        cudaError_t ie = cudaGraphInstantiate(&ctx->gexec, graph, 0);
        cudaGraphDestroy(graph);
        CK(ie);
        ctx->gkey = keybuf;
    }
    // the WHILE node evaluates its condition before the first iteration via the default
    // value (1); an empty initial worklist is handled by the first k_select (no work) and
    // k_round_end_graph (sets 0).
    CK(cudaGraphLaunch(ctx->gexec, ctx->stream));
    return EIK_OK;
}

// ---- whole-grid sweeping: DFSM / DLSM on the cell tiles ----------------
// end of one sweep: count it, stop after the first sweep that changed nothing (the
// FSM convention the paper's sweep counts use), or at the sweep cap / watchdog
__global__ void k_sweep_end(Ctl* ctl, cudaGraphConditionalHandle h)
{
    volatile Ctl* c = ctl;
    const unsigned long long w = c->sweep_writes;
    const float dm = __uint_as_float(c->sweep_dmax);
    c->sweep_idx += 1;
    c->rounds += 1;
    c->sweep_writes = 0;
    c->sweep_dmax = 0;
    // stop after a sweep that changed nothing, or (kappa > 0) whose largest change was
    // <= kappa
    bool more = w != 0 && dm > c->kappa_f;
    if (more && c->sweep_idx >= c->max_rounds) { c->err |= 4u; more = false; }
    if (more && gtimer() - c->t_solve0 > c->budget_ns) { c->err |= 8u; more = false; }
    cudaGraphSetConditional(h, more ? 1u : 0u);
}

// cells grouped by canonical diagonal a + b + c = D (one table serves all 8 directions: a
// direction reflects the canonical coordinates)
static int ensure_diag(eik_ctx* ctx, int cps)
{
    if (ctx->diag_cps == cps) return EIK_OK;
    const int nd = 3 * cps - 2;
    std::vector<uint32_t> cells;
    cells.reserve((size_t)cps * cps * cps);
    ctx->diag_off_h.assign(nd + 1, 0);
    for (int D = 0; D < nd; ++D) {
        ctx->diag_off_h[D] = (uint32_t)cells.size();
        for (int c = 0; c < cps; ++c)
            for (int b = 0; b < cps; ++b) {
                const int a = D - b - c;
                if (a >= 0 && a < cps) cells.push_back((uint32_t)a + (uint32_t)cps * ((uint32_t)b + (uint32_t)cps * (uint32_t)c));
            }
    }
    ctx->diag_off_h[nd] = (uint32_t)cells.size();
    cudaFree(ctx->diag_off);
    ctx->diag_off = nullptr;
    CK(cudaMalloc(&ctx->diag_off, (size_t)(nd + 1) * 4));
    CK(cudaMemcpy(ctx->diag_off, ctx->diag_off_h.data(), (size_t)(nd + 1) * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->diag_cells, cells.data(), cells.size() * 4, cudaMemcpyHostToDevice));
    ctx->diag_cps = cps;
    return EIK_OK;
}

template <typename T, int R>
static int sweep_grid_r(eik_ctx* ctx, int* grid)
{
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dsweep<T, R>, CellCfg<R>::NT, cell_smem_bytes<T, R>()));
    *grid = (occ < 1 ? 1 : occ) * ctx->sm_count;
    return EIK_OK;
}

template <typename T, int R>
static int capture_sweep(eik_ctx* ctx, const CellArgs& ca, int cps, cudaStream_t cs, int maxgrid)
{
    for (int D = 0; D < 3 * cps - 2; ++D) {
        const int cnt = (int)(ctx->diag_off_h[D + 1] - ctx->diag_off_h[D]);
        const int grid = cnt < maxgrid ? cnt : maxgrid;
        k_dsweep<T, R><<<grid, CellCfg<R>::NT, cell_smem_bytes<T, R>(), cs>>>(ca, D);
        CK(cudaGetLastError());
    }
    return EIK_OK;
}

// the whole sweep loop is one CUDA graph: WHILE (the last sweep changed something) { one
// launch per cell diagonal; k_sweep_end } -- no host round-trip per sweep
template <typename T>
static int run_sweeps(eik_ctx* ctx, int r, int64_t J, CellArgs ca, int method)
{
    const int cps = ca.cps;
    int st = ensure_diag(ctx, cps);
    if (st) return st;
    ca.diag_cells = ctx->diag_cells;
    ca.diag_off = ctx->diag_off;
    ca.cact = ctx->cact;
    ca.locked = method == EIK_DLSM ? 1 : 0;
    CK(cudaMemsetAsync(ctx->cact, 1, (size_t)J, ctx->stream));   // the first sweep relaxes everything
    int maxgrid = 0;
    st = r == 16 ? sweep_grid_r<T, 16>(ctx, &maxgrid) : r == 8 ? sweep_grid_r<T, 8>(ctx, &maxgrid)
                                                               : sweep_grid_r<T, 4>(ctx, &maxgrid);
    if (st) return st;
    char keybuf[256];
    snprintf(keybuf, sizeof keybuf, "%d/%d/%lld/%lld/%p/%p/%d/%d/%.17g", (int)sizeof(T), r, (long long)J,
             (long long)ca.n1, ca.Vt, ca.Ht, ca.stats, ca.locked, ca.kappa);
    if (!ctx->gexec_sw || ctx->gkey_sw != keybuf) {
        if (ctx->gexec_sw) { cudaGraphExecDestroy(ctx->gexec_sw); ctx->gexec_sw = nullptr; }
        cudaGraph_t graph;
        CK(cudaGraphCreate(&graph, 0));
        cudaGraphConditionalHandle handle;
        CK(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = handle;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        CK(cudaGraphAddNode(&cnode, graph, nullptr, 0, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        st = r == 16 ? capture_sweep<T, 16>(ctx, ca, cps, cs, maxgrid)
           : r == 8 ? capture_sweep<T, 8>(ctx, ca, cps, cs, maxgrid)
                    : capture_sweep<T, 4>(ctx, ca, cps, cs, maxgrid);
        k_sweep_end<<<1, 1, 0, cs>>>(ctx->ctl, handle);
        cudaGraph_t captured;
        cudaError_t ce = cudaStreamEndCapture(cs, &captured);
        cudaStreamDestroy(cs);
        if (st) { cudaGraphDestroy(graph); return st; }
        if (ce != cudaSuccess) { cudaGraphDestroy(graph); CK(ce); }
        cudaError_t ie = cudaGraphInstantiate(&ctx->gexec_sw, graph, 0);
        cudaGraphDestroy(graph);
        CK(ie);
        ctx->gkey_sw = keybuf;
    }
    CK(cudaGraphLaunch(ctx->gexec_sw, ctx->stream));
    return EIK_OK;
}

template <typename T>
static int solve_impl(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* mask,
                      const void* q, void* U, int r, int method)
{
    const int64_t n1 = n + 1;
    const int cps = (int)((n1 + r - 1) / r);
    const int64_t J = (int64_t)cps * cps * cps;
    const int64_t r3 = (int64_t)r * r * r;
    const int64_t P = J * r3;
    const int64_t M = n1 * n1 * n1;
    if (J >= (int64_t)1 << 31) return fail(ctx, EIK_EINVAL, "grid too large (J = %lld cells)", (long long)J);
    int st = ensure_scratch(ctx, (size_t)P * sizeof(T), (size_t)J);
    if (st) return st;
    cudaStream_t s = ctx->stream;

    Ctl init{};
    init.kmin[0] = init.kmin[1] = KEY_INF;
    init.max_rounds = ctx->max_rounds;
    init.t_start = ~0ull;
    init.budget_ns = (unsigned long long)(ctx->timeout_s * 1e9);
    init.kappa_f = (float)ctx->kappa;
    init.auto_mode = 6u;
    ctx->ms_cell_events = 0;
    *ctx->ctl_host = init;
    CK(cudaEventRecord(ctx->ev[0], s));
    CK(cudaMemcpyAsync(ctx->ctl, ctx->ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice, s));
    const int G = ctx->sm_count * 8;
    k_init_cells<<<G, 256, 0, s>>>(ctx->key, ctx->state, J, ctx->ctl);
    Geom g{n1, cps, r, r == 4 ? 2 : r == 8 ? 3 : 4};
    {
        const int64_t np = (int64_t)cps * r, nv = (np / 4) * np;   // vectors per padded z-plane
        const int bx = (int)((nv + 255) / 256 < 64 ? (nv + 255) / 256 : 64);
        const int by = (int)(np < 65535 ? np : 65535);
        k_ingest<T><<<dim3(bx, by), 256, 0, s>>>(g, (T)h, (const T*)F, mask, (const T*)q, (T*)ctx->Vt,
                                                 (T*)ctx->Ht, ctx->key, ctx->state, ctx->ctl, P);
    }
    if (method < 0 && ctx->loop_mode != 0) k_build_wl<<<G, 256, 0, s>>>(ctx->key, ctx->state, ctx->wl0, ctx->ctl, J);
    CK(cudaGetLastError());
    // No host round-trip here: a device-detected input error (ctl->err, no exit) makes the
    // seeding kernels enqueue nothing, the loop does no work and k_egress returns without
    // touching U_out; the status is read once, after egress.
    CK(cudaEventRecord(ctx->ev[1], s));

    CellArgs ca;
    memset(&ca, 0, sizeof ca);
    ca.ctl = ctx->ctl;
    ca.proc_cell = ctx->proc_cell;
    ca.proc_flags = ctx->proc_flags;
    ca.wl0 = ctx->wl0;
    ca.wl1 = ctx->wl1;
    ca.key = ctx->key;
    ca.state = ctx->state;
    const int ri = rindex_of(r);
    ca.plane_tab = ctx->plane_tab[ri];
    ca.tab16 = ctx->tab16;
    ca.tab_b2 = ctx->tab_b2;
    ca.Vt = ctx->Vt;
    ca.Ht = ctx->Ht;
    // automatic sweep cap: rounds last as long as their slowest processing, so the round modes
    // bound it (4 sweeps); the async scheduler has no rounds to shorten (a cap only adds work)
    ca.max_sweeps = ctx->max_sweeps >= 0 ? ctx->max_sweeps : (ctx->loop_mode == 0 ? 0 : 4);
    ca.cap = (uint32_t)J;
    ca.pend = ctx->pend;
    ca.pdir = ctx->pdir;
    ca.kappa = ctx->kappa;
    ca.legacy_key = ctx->legacy_key;
    ca.gen = ctx->gen;
    ca.n1 = n1;
    ca.cps = cps;
    ca.stats = ctx->collect_stats;
    ca.fused = isinf(ctx->bin_width) ? 1 : 0;
    st = method < 0 ? run_loop<T>(ctx, r, J, ca) : run_sweeps<T>(ctx, r, J, ca, method);
    if (st) return st;
    CK(cudaEventRecord(ctx->ev[2], s));
    {
        const int64_t nv = ((n1 + 3) / 4) * n1;   // vectors per z-plane
        const int bx = (int)((nv + 255) / 256 < 64 ? (nv + 255) / 256 : 64);
        const int by = (int)(n1 < 65535 ? n1 : 65535);
        k_egress<T><<<dim3(bx, by), 256, 0, s>>>(g, (const T*)ctx->Vt, (T*)U, M, ctx->ctl);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(ctx->ev[3], s));
    CK(cudaMemcpyAsync(ctx->ctl_host, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s));
    CK(cudaEventRecord(ctx->ev[4], s));
    // the one wait of the solve, with a host-side guard against a device loop that never
    // returns (the device watchdog covers the scheduler; this covers everything else): spin on
    // the event for the first 20 ms, then poll every 100 us until the deadline
    {
        const double limit_s = ctx->timeout_s + 30.0;
        struct timespec t0, t1;
        clock_gettime(CLOCK_MONOTONIC, &t0);
        for (;;) {
            const cudaError_t qe = cudaEventQuery(ctx->ev[4]);
            if (qe == cudaSuccess) break;
            if (qe != cudaErrorNotReady) CK(qe);
            clock_gettime(CLOCK_MONOTONIC, &t1);
            const double el = (t1.tv_sec - t0.tv_sec) + 1e-9 * (t1.tv_nsec - t0.tv_nsec);
            if (el > limit_s) {
                // read the control block through a side stream while the loop still runs
                cudaStream_t side;
                Ctl snap{};
                if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) == cudaSuccess) {
                    cudaMemcpyAsync(&snap, ctx->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, side);
                    cudaStreamSynchronize(side);
                    cudaStreamDestroy(side);
                }
                return fail(ctx, EIK_EINTERNAL, "device loop did not finish in %.0f s (pending %u head %u "
                            "tail %u rounds %u processings %llu); the context is unusable",
                            limit_s, snap.pending, snap.q_head, snap.q_tail, snap.rounds,
                            (unsigned long long)snap.processings);
            }
            if (el > 0.02) usleep(100);
        }
    }
    if (ctx->ctl_host->err & 1u) return fail(ctx, EIK_EINVAL, "F has a negative, NaN or infinite value");
    if (ctx->ctl_host->err & 2u) return fail(ctx, EIK_EINVAL, "an exit value q is negative, NaN or infinite");
    if (ctx->ctl_host->err & 16u)
        return fail(ctx, EIK_EINVAL, "h/F out of the supported range of %s (%s) at some F > 0 point",
                    sizeof(T) == 4 ? "fp32" : "fp64", sizeof(T) == 4 ? "2^-60 .. 2^60" : "2^-500 .. 2^500");
    if (ctx->ctl_host->n_exits == 0) return fail(ctx, EIK_EINVAL, "no exit point (exit_mask is all zero)");
    if (ctx->ctl_host->err & 4u)
        return fail(ctx, EIK_EINTERNAL, "max %s (%u) exceeded", method < 0 ? "rounds" : "sweeps", ctx->max_rounds);
    if (ctx->ctl_host->err & 8u)
        return fail(ctx, EIK_EINTERNAL, "watchdog: solve exceeded %.1f s (pending %u head %u tail %u "
                    "rounds %u processings %llu)", ctx->timeout_s, ctx->ctl_host->pending,
                    ctx->ctl_host->q_head, ctx->ctl_host->q_tail, ctx->ctl_host->rounds,
                    (unsigned long long)ctx->ctl_host->processings);
    if (ctx->ctl_host->abort)
        return fail(ctx, EIK_EINTERNAL, "processing limit exceeded (async scheduler)");

    const Ctl& hc = *ctx->ctl_host;
    eik_stats& S = ctx->stats;
    memset(&S, 0, sizeof S);
    S.M = M;
    S.padded_points = P;
    S.J = J;
    S.cells_per_side = cps;
    S.cell_size = r;
    S.precision = sizeof(T) == 4 ? EIK_F32 : EIK_F64;
    S.point_updates = hc.updates;
    S.point_writes = hc.writes;
    S.cell_processings = hc.processings;
    S.cell_sweeps = hc.sweeps;
    S.real_points_processed = hc.real_pts;
    S.rounds = hc.rounds;
    S.max_worklist = hc.max_proc;
    S.bytes_min = (uint64_t)((double)hc.real_pts * 2.0 * sizeof(T));
    S.bytes_cell_alg = hc.processings * (uint64_t)((2 * r3 + 6 * r * r) * sizeof(T)) +
                       hc.bytes_written * sizeof(T);
    float ms;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]); S.ms_ingest = ms;
    cudaEventElapsedTime(&ms, ctx->ev[1], ctx->ev[2]); S.ms_loop = ms;
    cudaEventElapsedTime(&ms, ctx->ev[2], ctx->ev[3]); S.ms_egress = ms;
    cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]); S.ms_total = ms;
    S.ms_cell_device = hc.cell_ns * 1e-6;
    S.ms_cell_events = ctx->ms_cell_events;
    S.cell_launches = hc.cell_launches;
    if (method < 0 && ctx->loop_mode == 0 && hc.t_end > hc.t_start) {
        // async: one persistent launch; its span is the first CTA's start to the last CTA's end
        S.ms_cell_device = (hc.t_end - hc.t_start) * 1e-6;
        S.cell_launches = 1;
        if (ctx->time_cell_events) {
            float ms = 0;
            cudaEventElapsedTime(&ms, ctx->cev[0], ctx->cev[1]);
            S.ms_cell_events = ms;
        }
    }
    if (method >= 0) {
        S.grid_sweeps = hc.sweep_idx;
        S.cell_launches = (uint64_t)hc.sweep_idx * (uint64_t)(3 * cps - 2);
        S.ms_cell_device = S.ms_loop;
    }
    ctx->have_stats = true;
    return EIK_OK;
}

static int validate(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* mask,
                    const void* q, void* U, int precision, int r)
{
    if (!ctx) return EIK_EINVAL;
    ctx->err.clear();
    if (!F || !mask || !q || !U) return fail(ctx, EIK_EINVAL, "null array pointer");
    if (n < 1) return fail(ctx, EIK_EINVAL, "n must be >= 1 (got %lld)", (long long)n);
    if (n > 100000) return fail(ctx, EIK_EINVAL, "n too large (%lld)", (long long)n);
    if (!(h > 0) || !isfinite(h)) return fail(ctx, EIK_EINVAL, "h must be finite and > 0");
    if (precision != EIK_F32 && precision != EIK_F64) return fail(ctx, EIK_EINVAL, "bad precision %d", precision);
    if (rindex_of(r) < 0) return fail(ctx, EIK_EINVAL, "cell_size must be 4, 8 or 16 (got %d)", r);
    return EIK_OK;
}

extern "C" int eik_solve(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* exit_mask,
                         const void* exit_vals, void* U_out, int precision, int cell_size)
{
    int st = validate(ctx, n, h, F, exit_mask, exit_vals, U_out, precision, cell_size);
    if (st) return st;
    CK(cudaSetDevice(ctx->device));
    ctx->have_stats = false;
    if (precision == EIK_F32) return solve_impl<float>(ctx, n, h, F, exit_mask, exit_vals, U_out, cell_size, -1);
    return solve_impl<double>(ctx, n, h, F, exit_mask, exit_vals, U_out, cell_size, -1);
}

extern "C" int eik_solve_sweep(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* exit_mask,
                               const void* exit_vals, void* U_out, int precision, int cell_size, int method)
{
    int st = validate(ctx, n, h, F, exit_mask, exit_vals, U_out, precision, cell_size);
    if (st) return st;
    if (method != EIK_DFSM && method != EIK_DLSM) return fail(ctx, EIK_EINVAL, "bad sweep method %d", method);
    CK(cudaSetDevice(ctx->device));
    ctx->have_stats = false;
    if (precision == EIK_F32) return solve_impl<float>(ctx, n, h, F, exit_mask, exit_vals, U_out, cell_size, method);
    return solve_impl<double>(ctx, n, h, F, exit_mask, exit_vals, U_out, cell_size, method);
}

extern "C" int eik_solve_host(eik_ctx* ctx, int64_t n, double h, const void* F, const uint8_t* exit_mask,
                              const void* exit_vals, void* U_out, int precision, int cell_size)
{
    int st = validate(ctx, n, h, F, exit_mask, exit_vals, U_out, precision, cell_size);
    if (st) return st;
    CK(cudaSetDevice(ctx->device));
    const size_t M = (size_t)(n + 1) * (n + 1) * (n + 1);
    const size_t s = precision == EIK_F32 ? 4 : 8;
    const size_t need = M * (3 * s + 1) + 256;
    if (need > ctx->stage_bytes) {
        CK(cudaStreamSynchronize(ctx->stream));
        cudaFree(ctx->stage);
        ctx->stage = nullptr;
        ctx->stage_bytes = 0;
        CK(cudaMalloc(&ctx->stage, need));
        ctx->stage_bytes = need;
    }
    char* base = (char*)ctx->stage;
    void* dF = base;
    void* dq = base + M * s;
    void* dU = base + 2 * M * s;
    uint8_t* dm = (uint8_t*)(base + 3 * M * s);
    cudaStream_t sm = ctx->stream;
    CK(cudaMemcpyAsync(dF, F, M * s, cudaMemcpyHostToDevice, sm));
    // exit_vals is read only at exit points (k_ingest loads q behind the mask test): when it is
    // page-locked host memory the device reads those few values in place over PCIe (mapped
    // pinned memory, UVA) instead of copying the whole dense array (M * s bytes, 0.54 GB at
    // C3 fp32); pageable memory is copied as before
    const void* qdev = dq;
    {
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, exit_vals) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
            pa.devicePointer != nullptr)
            qdev = pa.devicePointer;
        else
            (void)cudaGetLastError();
    }
    ctx->q_zero_copy = qdev != dq;
    if (qdev == dq) CK(cudaMemcpyAsync(dq, exit_vals, M * s, cudaMemcpyHostToDevice, sm));
    CK(cudaMemcpyAsync(dm, exit_mask, M, cudaMemcpyHostToDevice, sm));
    st = eik_solve(ctx, n, h, dF, dm, qdev, dU, precision, cell_size);
    if (st) return st;
    CK(cudaMemcpyAsync(U_out, dU, M * s, cudaMemcpyDeviceToHost, sm));
    CK(cudaStreamSynchronize(sm));
    ctx->stats.h2d_bytes = M * s + M + (ctx->q_zero_copy ? (uint64_t)ctx->ctl_host->n_exits * s : M * s);
    ctx->stats.d2h_bytes = M * s;
    return EIK_OK;
}
