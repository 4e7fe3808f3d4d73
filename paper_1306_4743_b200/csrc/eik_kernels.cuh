// eik_kernels.cuh -- sm_100a device code of the cell-sweep Eikonal solver.
//
// PRODUCT PATH.  Shares no code with oracle/ (the CPU test oracle); the only thing the two
// sides have in common is the formula of the local solve, written out
// independently here.
//
// Phases:
//   A1/A2 k_ingest    lexicographic F / exit_mask / q -> padded cell-blocked tiles V, hf;
//                     input validation; cell keys and INIT flags of exit cells (R18)
//         k_build_wl  initial worklist L <- Q^c (Alg. 1 line 2)
//   A7    k_select    lowest priority bin of the worklist -> this round's cells; key reset to
//                     +inf on removal (Alg. 1 lines 4-5; bins P:1675)
//   A3-A6 k_cell      one CTA per selected cell: stage tile + one-point halo N(c) into SMEM,
//                     gated (LSM) Gauss-Seidel sweeps in wavefront (i+j+k = s plane) order
//                     (Detrixhe planes inside a cell), Alg. 2 point update,
//                     write back changed values, re-activate currently-downwind neighbour
//                     cells with the Eq. (3) key (Alg. 1 lines 7-10)
//         k_round_end swap worklists, termination test (Alg. 3 line 6 activeCellCount)
//   A8    k_egress    tiles -> lexicographic U_out
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace eik {

// Device-side bounds checks (build with -DEIK_CHECKS, library libeik_checks.so): a violated
// invariant prints and traps.  compute-sanitizer is not available on the GPU pool, so the
// checked build run over the GPU test suite stands in for memcheck on the indices we compute.
#ifdef EIK_CHECKS
#define EIK_CHECK(cond, what)                                                              \
    do {                                                                                   \
        if (!(cond)) {                                                                     \
            printf("EIK_CHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__,    \
                   __LINE__, (int)blockIdx.x, (int)threadIdx.x);                           \
            __trap();                                                                      \
        }                                                                                  \
    } while (0)
#else
#define EIK_CHECK(cond, what) do { } while (0)
#endif

// --------------------------------------------------------------------------------------
// numeric helpers
// --------------------------------------------------------------------------------------
template <typename T> __device__ __forceinline__ T dinf();
template <> __device__ __forceinline__ float dinf<float>() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double dinf<double>() {
    return __longlong_as_double(0x7ff0000000000000LL);
}

// Cell keys are the IEEE bits of a non-negative float: unsigned order == numeric order, so
// atomicMin on the bits implements Eq. (3)'s V^c <- min(V^c, Vtilde^c) (Alg. 4 analogue).
__device__ __forceinline__ uint32_t key_bits(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t key_bits(double v) { return __float_as_uint(__double2float_rd(v)); }
static constexpr uint32_t KEY_INF = 0x7f800000u;

// Shared-memory access through 32-bit shared-window addresses.  The sweep loops form every
// address from bases pinned in registers by a volatile conversion (the compiler otherwise
// rematerialises the window base with S2R on each step under the register cap); the volatile
// accesses keep program order and are not moved across barriers.
__device__ __forceinline__ uint32_t smem_u32(const void* p)
{
    uint32_t a;
    asm volatile("mov.u32 %0, %1;" : "=r"(a) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return a;
}
template <typename T> __device__ __forceinline__ T lds(uint32_t a);
template <> __device__ __forceinline__ float lds<float>(uint32_t a)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
template <> __device__ __forceinline__ double lds<double>(uint32_t a)
{
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t a)
{
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(v)); }
__device__ __forceinline__ void sts(uint32_t a, double v) { asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(v)); }
__device__ __forceinline__ void sts_u8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" :: "r"(a), "r"(v)); }

__device__ __forceinline__ void cp_async_el(uint32_t dst, const float* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_el(uint32_t dst, const double* src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all()
{
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

// Bulk asynchronous copy (TMA engine, cp.async.bulk) of a contiguous block of global memory into
// shared memory, completion signalled on an mbarrier: one instruction by one thread moves a whole
// hf tile (16 KB for r = 16 fp32) instead of 1024 per-thread cp.async.  The mbarrier is
// initialised once per kernel (arrival count 1); every copy is one phase (parity alternates).
__device__ __forceinline__ void mbar_init(uint32_t mbar)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(mbar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar)
{
    // earlier generic-proxy accesses of the destination (ordered before this thread by a CTA
    // barrier) precede the async-proxy write
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(mbar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity)
{
    asm volatile("{\n\t.reg .pred p;\n\t"
                 "W_%=:\n\t"
                 "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                 "@!p bra W_%=;\n\t}" :: "r"(mbar), "r"(parity) : "memory");
}

// Local solve of Eq. (2) for U at one gridpoint, shifted sorted form (SURVEY
// C.3, readings R1-R4): a1 <= a2 <= a3 are the per-axis neighbour minima (a1 finite),
// hf = h/F.  t = U - a1; one-sided t = hf; two-sided iff hf > a2 - a1; three-sided iff the
// two-sided t > a3 - a1.  Every operand of a taken branch is O(hf): no cancellation.
template <typename T>
__device__ __forceinline__ T local_solve(T mx, T my, T mz, T hf)
{
    const T lo = fmin(mx, my), hi = fmax(mx, my);
    const T a1 = fmin(lo, mz);
    const T a3 = fmax(hi, mz);
    const T a2 = fmax(lo, fmin(hi, mz));
    T t = hf;
    const T d2 = a2 - a1;               // +inf if a2 = +inf: never taken
    if (t > d2) {
        const T disc = fmax(T(2) * hf * hf - d2 * d2, T(0));
        t = (d2 + sqrt(disc)) * T(0.5);
        const T d3 = a3 - a1;
        if (t > d3) {
            const T e = d3 - d2;
            const T disc3 = fmax(T(3) * hf * hf - (d2 * d2 + d3 * d3 + e * e), T(0));
            t = (d2 + d3 + sqrt(disc3)) * T(1.0 / 3.0);
        }
    }
    return a1 + t;
}

// min / max of non-NaN values (every operand here is >= 0 or +inf, or a clamped difference):
// fp64 as one compare and two selects, without the NaN fix-up fmin/fmax compile to
// (DSETP.MIN + FSEL + SEL + LOP3 and register moves); fp32 keeps FMNMX
#ifndef EIK_VMIN
#define EIK_VMIN 1
#endif
#ifndef EIK_SORT3_CMP
#define EIK_SORT3_CMP 0   // fp64: sort the three axis minima with three compares (measured: P2 19.3 -> 19.5 ms, C3d / C2d within noise)
#endif
__device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
__device__ __forceinline__ float vmax(float a, float b) { return fmaxf(a, b); }
#if EIK_VMIN
__device__ __forceinline__ double vmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double vmax(double a, double b) { return b > a ? b : a; }
#else
__device__ __forceinline__ double vmin(double a, double b) { return fmin(a, b); }
__device__ __forceinline__ double vmax(double a, double b) { return fmax(a, b); }
#endif

// warp reductions in one instruction each (REDUX) instead of five shuffle + op rounds
__device__ __forceinline__ unsigned long long warp_or64(unsigned long long x)
{
    const uint32_t lo = __reduce_or_sync(0xffffffffu, (uint32_t)x);
    const uint32_t hi = __reduce_or_sync(0xffffffffu, (uint32_t)(x >> 32));
    return ((unsigned long long)hi << 32) | lo;
}
__device__ __forceinline__ uint32_t warp_add(uint32_t x) { return __reduce_add_sync(0xffffffffu, x); }
__device__ __forceinline__ uint32_t warp_or(uint32_t x) { return __reduce_or_sync(0xffffffffu, x); }

// |x| without the FP64 pipe (fabs(double) compiles to DADD -RZ, |x| when the result feeds a select)
__device__ __forceinline__ float vabs(float x) { return fabsf(x); }
__device__ __forceinline__ double vabs(double x)
{
    return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
}

// The same solve with the two- and three-sided candidates evaluated side by side and then
// selected (shorter dependent chain: both square roots issue together).  d2, d3 are clamped to
// hf, which changes nothing when a branch is taken (it requires d2 < hf, resp. d3 < t2 <= hf)
// and keeps every operand finite.  Identical results to local_solve in every case.
__device__ __forceinline__ float sqrt_fast(float x) { return __fsqrt_rn(x); }
__device__ __forceinline__ double sqrt_fast(double x) { return __dsqrt_rn(x); }

// fp32: sqrt.approx (MUFU, ~1 ulp); the shifted form only multiplies its error by O(hf), so
// the effect on U is an ulp of hf (reading R14: fp32 arithmetic throughout).  fp64: IEEE.
__device__ __forceinline__ float sqrt_approx(float x)
{
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));   // arguments are O(hf^2) >> FLT_MIN
    return r;
}
#ifndef EIK_FAST_DSQRT
#define EIK_FAST_DSQRT 1   // measured: 272 -> 230 instructions per fp64 step, C3d -5 %, C2d / P2 / P3 -8 %
#endif
__device__ __forceinline__ double sqrt_approx(double x)
{
#if EIK_FAST_DSQRT
    // x >= 0 and finite (a clamped discriminant, O(hf^2)): MUFU reciprocal square-root seed and
    // two Newton corrections of s = x / sqrt(x) (no special-case path); x = 0 -> 0
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    double s = x * y;
    const double hy = 0.5 * y;
    s = fma(fma(-s, s, x), hy, s);
    s = fma(fma(-s, s, x), hy, s);
    return x > 0.0 ? s : 0.0;
#else
    return __dsqrt_rn(x);
#endif
}

// a1 <= a2 <= a3 of three values: fp32 as a min/max network (FMNMX); fp64 from three compares
// (each fp64 min or max costs its own DSETP on the half-rate pipe: six in the network)
__device__ __forceinline__ void sort3(float mx, float my, float mz, float& a1, float& a2, float& a3)
{
    const float lo = vmin(mx, my), hi = vmax(mx, my);
    a1 = vmin(lo, mz);
    a3 = vmax(hi, mz);
    a2 = vmax(lo, vmin(hi, mz));
}
__device__ __forceinline__ void sort3(double mx, double my, double mz, double& a1, double& a2, double& a3)
{
#if EIK_SORT3_CMP
    const bool p1 = my < mx, p2 = mz < mx, p3 = mz < my;
    const double lo = p1 ? my : mx, hi = p1 ? mx : my;
    const bool plo = p1 ? p3 : p2;   // mz < lo
    const bool phi = p1 ? p2 : p3;   // mz < hi
    a1 = plo ? mz : lo;
    a3 = phi ? hi : mz;
    a2 = plo ? lo : (phi ? mz : hi);
#else
    const double lo = vmin(mx, my), hi = vmax(mx, my);
    a1 = vmin(lo, mz);
    a3 = vmax(hi, mz);
    a2 = vmax(lo, vmin(hi, mz));
#endif
}

template <typename T>
__device__ __forceinline__ T local_solve_fast(T mx, T my, T mz, T hf)
{
    T a1, a2, a3;
    sort3(mx, my, mz, a1, a2, a3);
    const T d2 = vmin(a2 - a1, hf);
    const T d3 = vmin(a3 - a1, hf);
    const T hh = hf * hf;
    const T t2 = (d2 + sqrt_approx(vmax(T(2) * hh - d2 * d2, T(0)))) * T(0.5);
    const T e = d3 - d2;
    const T t3 = (d2 + d3 + sqrt_approx(vmax(T(3) * hh - (d2 * d2 + d3 * d3 + e * e), T(0)))) * T(1.0 / 3.0);
    T t = hf;
    if (hf > d2) t = (t2 > d3) ? t3 : t2;
    return a1 + t;
}

template <typename T>
__device__ __forceinline__ T local_solve_par(T mx, T my, T mz, T hf)
{
    const T lo = fmin(mx, my), hi = fmax(mx, my);
    const T a1 = fmin(lo, mz);
    const T a3 = fmax(hi, mz);
    const T a2 = fmax(lo, fmin(hi, mz));
    const T d2 = fmin(a2 - a1, hf);
    const T d3 = fmin(a3 - a1, hf);
    const T hh = hf * hf;
    const T t2 = (d2 + sqrt_fast(fmax(T(2) * hh - d2 * d2, T(0)))) * T(0.5);
    const T e = d3 - d2;
    const T t3 = (d2 + d3 + sqrt_fast(fmax(T(3) * hh - (d2 * d2 + d3 * d3 + e * e), T(0)))) * T(1.0 / 3.0);
    T t = hf;
    if (hf > d2) t = (t2 > d3) ? t3 : t2;
    return a1 + t;
}

// --------------------------------------------------------------------------------------
// device-side control block (one per ctx)
// --------------------------------------------------------------------------------------
struct Ctl {
    uint32_t wl_count[2];   // sizes of the two ping-pong worklists
    uint32_t kmin[2];       // min key (float bits) over each worklist
    uint32_t cur;           // which worklist is current
    uint32_t proc_count;    // cells selected this round
    uint32_t rounds;
    uint32_t max_proc;
    uint32_t max_rounds;
    uint32_t done;
    uint32_t err;           // 1: bad F, 2: bad q, 4: internal (max rounds)
    uint32_t n_exits;
    unsigned long long updates, writes, processings, sweeps, real_pts, bytes_written;
    unsigned long long t_start, t_end;     // this round's cell-kernel span (%globaltimer ns)
    unsigned long long cell_ns, cell_launches;
    uint32_t q_head, q_tail, pending, abort;   // async mode ring + work counter
    unsigned long long t_solve0, budget_ns;     // watchdog: abort after budget_ns
    uint32_t rtrace[2048];                      // round mode: per-round (cells, span ns)
    uint32_t rtrace2[2048];                     // round mode: per-round (sum cycles / 1024, max cycles)
    unsigned long long rsum, rmax;              // this round's processing cycles (stats)
    unsigned long long lstat[2][6];             // [all, > 100k cycles]: count, cycles, sweeps,
                                                // list iterations, plane steps, flags CONT
    uint32_t claim;                             // round mode: next cell of this round
    uint32_t cta_done;                          // round mode (fused): CTAs finished this round
    unsigned long long defers;
    // diagnostics (eik_get_debug): [0] sum of per-processing SM cycles, [1] max, [2] plane
    // steps executed, [3] processings, [4..35] histogram of sweeps per processing (31 = >=31)
    unsigned long long dbg[43];   // [36] stage, [37] plane-mask, [38] steps, [39] write-back cycles, [40] list iterations
    // whole-grid sweeping (k_dsweep): sweep s runs direction s mod 8
    uint32_t sweep_idx;           // sweeps completed
    unsigned long long sweep_writes;   // strict decreases in the current sweep
    uint32_t sweep_dmax;          // largest value change of the current sweep (float bits, up)
    float kappa_f;                // early termination threshold of the sweeps
    uint32_t trace_n;             // async mode processing trace (EIK_OPT_TRACE): entries written
    uint32_t first_procs;         // async mode: cells processed at least once
    uint32_t auto_mode;           // async readiness mode 8: the mode in force (6, then 2)
    uint32_t sm_rank[256];        // async mode: CTAs of the persistent launch counted per SM (%smid)
};

__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

enum : uint32_t {
    FLAG_INIT = 64u,    // state bit: activate every point (first processing)
    FLAG_CONT = 128u    // state bit: the cell stopped at the sweep cap; its active points are
                        // saved in CellArgs::pend and are restored by the next processing
};

struct Geom {
    int64_t n1;        // n + 1 points per side
    int32_t cps;       // cells per side
    int32_t r;
    int32_t lr;        // log2(r)
};

__device__ __forceinline__ void warp_agg_append(uint32_t* counter, uint32_t* list, uint32_t val,
                                                bool pred)
{
    // warp-aggregated append (one atomic per warp)
    const unsigned full = __activemask();
    const unsigned m = __ballot_sync(full, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(counter, (uint32_t)__popc(m));
    base = __shfl_sync(full, base, leader);
    if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = val;
}

// --------------------------------------------------------------------------------------
// A1/A2: ingest + validate + seed
// --------------------------------------------------------------------------------------
template <typename T> struct Vec4T;
template <> struct Vec4T<float> { static __device__ __forceinline__ void st(float* p, const float* v) {
    __stcg(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3])); } 
    static __device__ __forceinline__ void ld(const float* p, float* v) {
    const float4 x = __ldcg(reinterpret_cast<const float4*>(p)); v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w; } };
template <> struct Vec4T<double> { static __device__ __forceinline__ void st(double* p, const double* v) {
    __stcg(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
    __stcg(reinterpret_cast<double2*>(p) + 1, make_double2(v[2], v[3])); }
    static __device__ __forceinline__ void ld(const double* p, double* v) {
    const double2 x = __ldcg(reinterpret_cast<const double2*>(p)), y = __ldcg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = x.x; v[1] = x.y; v[2] = y.x; v[3] = y.y; } };

// (A row-segment ingest -- a warp per 128 consecutive points of a row, every load and store a
// contiguous warp access, 40 registers instead of 75 -- measured no faster: C5 3.62 -> 3.72 ms,
// C3 equal; removed.)
#ifndef EIK_INGEST_U
#define EIK_INGEST_U 2   // vectors of 4 points per thread and iteration (4 measured slower: C3 0.52 -> 0.65 ms)
#endif
template <typename T>
__global__ void k_ingest(Geom g, T h, const T* __restrict__ F, const uint8_t* __restrict__ mask,
                         const T* __restrict__ q, T* __restrict__ Vt, T* __restrict__ Ht,
                         uint32_t* __restrict__ key, uint32_t* __restrict__ state, Ctl* ctl,
                         int64_t P)
{
    const int r = g.r, lr = g.lr;
    const int64_t n1 = g.n1;
    const uint32_t cps = (uint32_t)g.cps;
    uint32_t exits = 0;
    // Lexicographic traversal of the padded grid (cps r)^3, four consecutive i per thread:
    // a warp reads 512 contiguous bytes of F (the rows are not 16-byte aligned, so four scalar
    // loads) and writes 16-byte aligned pieces of eight tile rows.  (A tile-order traversal
    // reads 64-byte row pieces at unaligned offsets and over-fetches F 2x, the mask 4x.)
    // blockIdx.y strides over k; 32-bit index math within a z-plane.
    const uint32_t np = cps << lr;             // padded points per side
    const uint32_t nvr = np >> 2;              // vectors per padded row
    const uint32_t nv = nvr * np;              // vectors per padded z-plane (< 2^32)
    // EIK_INGEST_U vectors per thread and iteration (t, t + S, ...): 4 U loads of F and of the
    // mask in flight before any is used
    const uint32_t S = gridDim.x * blockDim.x;
    constexpr int U = EIK_INGEST_U;
    for (int64_t k = blockIdx.y; k < (int64_t)np; k += gridDim.y)
    for (uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x; t0 < nv; t0 += U * S) {
        T f[U][4];
        uint8_t mk[U][4];
        int64_t i0[U], j[U], lex0[U], p0[U];
        uint32_t c[U];
        bool vin[U], row_in[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t t = t0 + u * S;
            vin[u] = t < nv;
            const uint32_t j32 = t / nvr, iv = t - j32 * nvr;
            i0[u] = (int64_t)iv << 2;
            j[u] = j32;
            const int a0 = (int)(i0[u] & (r - 1)), b = (int)(j[u] & (r - 1)), d = (int)(k & (r - 1));
            c[u] = (uint32_t)(i0[u] >> lr) + cps * ((uint32_t)(j[u] >> lr) + cps * (uint32_t)(k >> lr));
            p0[u] = ((int64_t)c[u] << (3 * lr)) + a0 + r * (b + r * d);
            row_in[u] = vin[u] && j[u] < n1 && k < n1;
            lex0[u] = i0[u] + n1 * (j[u] + n1 * k);
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                const bool in = row_in[u] && i0[u] + l < n1;
                f[u][l] = in ? __ldcs(&F[lex0[u] + l]) : T(0);
                mk[u][l] = in ? __ldcs(&mask[lex0[u] + l]) : (uint8_t)0;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!vin[u]) continue;
            const int a0 = (int)(i0[u] & (r - 1)), b = (int)(j[u] & (r - 1)), d = (int)(k & (r - 1));
            T vv[4], hh[4];
#pragma unroll
            for (int l = 0; l < 4; ++l) {
                vv[l] = dinf<T>();
                hh[l] = dinf<T>();
                if (!(row_in[u] && i0[u] + l < n1)) continue;
                const T fl = f[u][l];
                if (!(fl >= T(0)) || !(fl < dinf<T>())) atomicOr(&ctl->err, 1u);   // F < 0, NaN, inf
                if (mk[u][l]) {
                    const int a = a0 + l;
                    const int64_t i = i0[u] + l, jj = j[u];
                    T qv = q[lex0[u] + l];
                    if (!(qv >= T(0)) || !(qv < dinf<T>())) atomicOr(&ctl->err, 2u);
                    qv = qv + T(0);   // canonicalise -0 -> +0 (R9)
                    vv[l] = qv;       // exits: fixed, V = q (hf stays +inf: never updated)
                    ++exits;
                    const uint32_t kb = key_bits(qv);
                    // V^c of a cell in Q^c = min exit value; cells holding a
                    // non-exit neighbour of an exit across a cell face are seeded too (R18)
                    atomicMin(&key[c[u]], kb);
                    atomicOr(&state[c[u]], FLAG_INIT);
                    const int64_t c64 = (int64_t)c[u], cp = (int64_t)cps;
                    const int64_t cc[6] = {a == 0 && i > 0 ? c64 - 1 : -1,
                                           a == r - 1 && i + 1 < n1 ? c64 + 1 : -1,
                                           b == 0 && jj > 0 ? c64 - cp : -1,
                                           b == r - 1 && jj + 1 < n1 ? c64 + cp : -1,
                                           d == 0 && k > 0 ? c64 - cp * cp : -1,
                                           d == r - 1 && k + 1 < n1 ? c64 + cp * cp : -1};
#pragma unroll
                    for (int f2 = 0; f2 < 6; ++f2)
                        if (cc[f2] >= 0) {
                            atomicMin(&key[cc[f2]], kb);
                            atomicOr(&state[cc[f2]], FLAG_INIT);
                        }
                } else if (fl > T(0)) {
                    hh[l] = h / fl;
                    // h/F must keep hf^2 normal and 3 hf^2 finite in T (the local solve squares
                    // it): fp32 [2^-60, 2^60], fp64 [2^-500, 2^500]; outside -> EIK_EINVAL
                    const T lo = sizeof(T) == 4 ? T(8.673617379884035e-19) : T(3.054936363499605e-151);
                    const T hi = sizeof(T) == 4 ? T(1.152921504606847e18) : T(3.273390607896142e150);
                    if (!(hh[l] >= lo && hh[l] <= hi)) atomicOr(&ctl->err, 16u);
                }
            }
            Vec4T<T>::st(&Vt[p0[u]], vv);
            Vec4T<T>::st(&Ht[p0[u]], hh);
        }
    }
    (void)P;
    // exit count (warp-aggregated)
    for (int o = 16; o > 0; o >>= 1) exits += __shfl_xor_sync(0xffffffffu, exits, o);
    if ((threadIdx.x & 31) == 0 && exits) atomicAdd(&ctl->n_exits, exits);
}

__global__ void k_init_cells(uint32_t* key, uint32_t* state, int64_t J, Ctl* ctl)
{
    if (blockIdx.x == 0 && threadIdx.x == 0) ctl->t_solve0 = gtimer();   // watchdog origin
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < J;
         c += (int64_t)gridDim.x * blockDim.x) {
        key[c] = KEY_INF;
        state[c] = 0;
    }
}

__global__ void k_build_wl(const uint32_t* __restrict__ key, const uint32_t* __restrict__ state,
                           uint32_t* wl0, Ctl* ctl, int64_t J)
{
    if (__ldcg(&ctl->err) != 0u || __ldcg(&ctl->n_exits) == 0u) return;   // invalid input: no work
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < J;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = base + threadIdx.x;
        const bool q = c < J && state[c] != 0;
        warp_agg_append(&ctl->wl_count[0], wl0, (uint32_t)c, q);
        if (q) atomicMin(&ctl->kmin[0], key[c]);
    }
}

// --------------------------------------------------------------------------------------
// A7: select the lowest bin [kmin, kmin + delta] of the current worklist
// --------------------------------------------------------------------------------------
__global__ void k_select(Ctl* ctl, uint32_t* wl0, uint32_t* wl1, uint32_t* proc_cell,
                         uint32_t* proc_flags, uint32_t* key, uint32_t* state, float delta,
                         int legacy_key)
{
    if (ctl->done) return;   // a round after the last one in the same graph iteration
    const uint32_t cur = ctl->cur, nx = cur ^ 1u;
    const uint32_t n = ctl->wl_count[cur];
    const uint32_t* wl = cur ? wl1 : wl0;
    uint32_t* wn = cur ? wl0 : wl1;
    const float thr = __uint_as_float(ctl->kmin[cur]) + delta;   // delta = +inf: all
    for (uint32_t base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
        const uint32_t i = base + threadIdx.x;
        const bool valid = i < n;
        const uint32_t c = valid ? wl[i] : 0u;
        const uint32_t kb = valid ? key[c] : KEY_INF;
        const bool sel = valid && __uint_as_float(kb) <= thr;
        const bool carry = valid && !sel;
        uint32_t fl = 0;
        if (sel) {
            fl = atomicExch(&state[c], 0u);   // take the inflow bits; cell leaves the list
            if (!legacy_key) key[c] = KEY_INF;   // V^c <- +inf on removal (not Eq. (4))
        }
        // selected -> proc list (cell, flags): same slot for both arrays
        {
            const unsigned full = __activemask();
            const unsigned m = __ballot_sync(full, sel);
            const int lane = threadIdx.x & 31;
            if (m) {
                const int leader = __ffs(m) - 1;
                uint32_t b0 = 0;
                if (lane == leader) b0 = atomicAdd(&ctl->proc_count, (uint32_t)__popc(m));
                b0 = __shfl_sync(full, b0, leader);
                if (sel) {
                    const uint32_t s = b0 + __popc(m & ((1u << lane) - 1u));
                    proc_cell[s] = c;
                    proc_flags[s] = fl;
                }
            }
        }
        warp_agg_append(&ctl->wl_count[nx], wn, c, carry);
        if (carry) atomicMin(&ctl->kmin[nx], kb);
    }
}

// --------------------------------------------------------------------------------------
// round end: swap worklists, count, termination
// --------------------------------------------------------------------------------------
// (volatile: in the fused loop this runs in the last CTA of k_cell, whose L1 may hold stale
// lines of the control block that other CTAs updated with atomics in L2)
__device__ __forceinline__ bool round_end_body(Ctl* ctl_)
{
    volatile Ctl* ctl = ctl_;
    const uint32_t cur = ctl->cur, nx = cur ^ 1u;
    ctl->rounds += 1;
    if (ctl->proc_count > ctl->max_proc) ctl->max_proc = ctl->proc_count;
    ctl->processings += ctl->proc_count;
    if (ctl->proc_count > 0 && ctl->t_end > ctl->t_start) {
        ctl->cell_ns += ctl->t_end - ctl->t_start;
        ctl->cell_launches += 1;
        if (ctl->rounds <= 1024u) {   // per-round trace (diagnostics): cells, span ns
            ctl->rtrace[2 * (ctl->rounds - 1)] = ctl->proc_count;
            ctl->rtrace[2 * (ctl->rounds - 1) + 1] = (uint32_t)(ctl->t_end - ctl->t_start);
            ctl->rtrace2[2 * (ctl->rounds - 1)] = (uint32_t)(ctl->rsum >> 10);
            ctl->rtrace2[2 * (ctl->rounds - 1) + 1] = (uint32_t)ctl->rmax;
        }
    }
    ctl->t_start = ~0ull;
    ctl->t_end = 0;
    ctl->rsum = 0;
    ctl->rmax = 0;
    ctl->proc_count = 0;
    ctl->claim = 0;
    ctl->cta_done = 0;
    ctl->wl_count[cur] = 0;
    ctl->kmin[cur] = KEY_INF;
    ctl->cur = nx;
    bool more = ctl->wl_count[nx] != 0;
    if (more && ctl->rounds >= ctl->max_rounds) ctl->err |= 4u;
    if (more && gtimer() - ctl->t_solve0 > ctl->budget_ns) { ctl->err |= 8u; more = false; }   // watchdog
    ctl->done = (more && ctl->rounds < ctl->max_rounds) ? 0u : 1u;
    return ctl->done != 0u;
}

__global__ void k_round_end(Ctl* ctl) { (void)round_end_body(ctl); }

// --------------------------------------------------------------------------------------
// A3-A6: the cell-sweep kernel
// --------------------------------------------------------------------------------------
#ifndef EIK_POP_MAXNS
#define EIK_POP_MAXNS 1024   // longest back-off (ns) of a CTA waiting for its ticket's slot
#endif
#ifndef EIK_MINB8
#define EIK_MINB8 12   // measured (fp64 r = 8): 8 -> 12 P2 24.0 -> 21.5 ms, C2d 10.7 -> 10.5; 16 slower
#endif
template <int R> struct CellCfg {
    static constexpr int R3 = R * R * R;
    static constexpr int RP = R + 2;
    static constexpr int RP2 = RP * RP;
    static constexpr int BOX = RP * RP * RP;
    static constexpr int NPL = 3 * R - 2;                            // wavefront planes
    static constexpr int MAXP = R == 16 ? 192 : (R == 8 ? 48 : 12);  // largest plane
    static constexpr int PPT = 1;                                    // plane points / thread (2 measured slower)
    static constexpr int NT = ((MAXP + PPT - 1) / PPT + 31) / 32 * 32;
    static constexpr int MINB = R == 16 ? 4 : EIK_MINB8;             // CTAs per SM target
    static constexpr int LCAP = R == 16 ? 384 : (R == 8 ? 128 : 64);  // active-list capacity
};

#ifndef EIK_LIFO
#define EIK_LIFO 1
#endif
#ifndef EIK_DIR_TEMPLATE_MIN_R
#define EIK_DIR_TEMPLATE_MIN_R 16   // cells below this size use the runtime-direction sweep
#endif
#ifndef EIK_PARITY
#define EIK_PARITY 1
#endif
#ifndef EIK_STAGE_B32
#define EIK_STAGE_B32 3   // fp32 tile vectors in flight per thread while staging (6: all of them, spills at 64 registers)
#endif
#ifndef EIK_STAGE_B64
#define EIK_STAGE_B64 2   // fp64 tile vectors (16 B) in flight per thread while staging
#endif
#ifndef EIK_SWEEP16
#define EIK_SWEEP16 1   // r = 16, kappa = 0: the packed-table wavefront step (sweep16)
#endif
#ifndef EIK_WARP_BALANCE
#define EIK_WARP_BALANCE 0   // k_async r = 16: permute the plane-table columns over the warps per CTA (measured: within 1 %)
#endif
#ifndef EIK_TAG_WARP1
#define EIK_TAG_WARP1 1   // k_async: warp 1 tags and releases while warp 0 pops the next cell
#endif
#ifndef EIK_HF_BULK
#define EIK_HF_BULK 1   // k_async: stage hf with one cp.async.bulk + mbarrier instead of per-thread cp.async
#endif
#ifndef EIK_LIST_THR
#define EIK_LIST_THR -2   // active points at or below which the list relaxation replaces sweeps (0: the list capacity, -1: never, -2: r = 16 ? 16 : never)
#endif
#ifndef EIK_DIR0_ACT
#define EIK_DIR0_ACT 1   // first sweep direction of a re-activated cell from the activated face points
#endif
#ifndef EIK_DIR_VOTE
#define EIK_DIR_VOTE 2   // sweep directions after the first from a vote of the active points (1: always, 2: when two or more axes are ambiguous)
#endif
#ifndef EIK_UNGATED_DIV
#define EIK_UNGATED_DIV 32   // first sweep ungated from R^3 / 32 active points (measured 2 / 8 / 32 / 128 / always: C4 6.57 -> 6.42 ms at 32, others within 0.3 %; never ungated for face-activated cells: C3 +5 %)
#endif
#ifndef EIK_MINB16
#define EIK_MINB16 5   // fp32 r = 16: 5 x 45.4 KB of shared memory, <= 64 registers (no spills)
#endif
template <typename T, int R> struct MinBlocks { static constexpr int value = CellCfg<R>::MINB; };
// Five fp32 r = 16 CTAs fit an SM only while dynamic + static shared memory, rounded up to the
// 128-byte allocation unit, plus the 1 KB per-CTA reservation, stays <= 228 KB / 5: 16 more
// bytes of CellShared once dropped all three cell kernels to 4 CTAs per SM (checked below).
template <> struct MinBlocks<float, 16> { static constexpr int value = EIK_MINB16; };
// fp64 r = 16 (EIK_HF_GLOBAL64): hf stays in global memory (read through L1/L2 one plane
// ahead) and "changed" is a bitmask, so the shared-memory footprint drops from 85 to 53 KB
// and the SM holds EIK_MINB64 CTAs instead of 2
#ifndef EIK_HF_GLOBAL64
#define EIK_HF_GLOBAL64 1
#endif
#ifndef EIK_MINB64
#define EIK_MINB64 4   // measured: 2 (hf in shared memory) 29.6 ms on C3d, 3 26.2, 4 24.0
#endif
#ifndef EIK_HF_GLOBAL32
#define EIK_HF_GLOBAL32 0
#endif
template <typename T, int R> struct HfGlobal { static constexpr bool value = false; };
#if EIK_HF_GLOBAL32
template <> struct HfGlobal<float, 16> { static constexpr bool value = true; };
#endif
#if EIK_HF_GLOBAL64
template <> struct HfGlobal<double, 16> { static constexpr bool value = true; };
template <> struct MinBlocks<double, 16> { static constexpr int value = EIK_MINB64; };
#else
template <> struct MinBlocks<double, 16> { static constexpr int value = 2; };
#endif

template <typename T, int R>
constexpr size_t cell_smem_bytes()
{
    // V box + hf (or a changed bitmask) + active bytes (+ scratch) + 2 active lists (uint16)
    if constexpr (HfGlobal<T, R>::value)
        return sizeof(T) * CellCfg<R>::BOX + CellCfg<R>::R3 + 16 + CellCfg<R>::R3 / 8 + 4 * CellCfg<R>::LCAP;
    return sizeof(T) * (CellCfg<R>::BOX + CellCfg<R>::R3) + CellCfg<R>::R3 + 16 + 4 * CellCfg<R>::LCAP;
}

struct CellArgs {
    Ctl* ctl;
    const uint32_t* proc_cell;   // round mode: this round's cells
    const uint32_t* proc_flags;
    uint32_t* wl0;               // round mode: worklists; async mode: wl0 = queue ring
    uint32_t* wl1;
    uint32_t qmask;              // async mode: ring capacity - 1 (power of two)
    uint32_t* key;
    uint32_t* state;
    uint32_t* gen;               // async mode: activation generation of each cell, 1 + the largest of its
                                 // taggers' (modes 5-8); mode 9: activation level, 1 + the smallest (from 0x7f7f7f7f)
    uint32_t* wait;              // async mode: bit f = the neighbour across face f is parked on this cell
    const uint16_t* plane_tab;   // [NPL + 3][NT] canonical point of thread t in plane s (0xFFFF: none)
    const uint32_t* tab16;       // r = 16: [8][NPL + 3][NT] packed per-direction plane table (sweep16)
    const uint2* tab_b2;         // r = 16 micro-block kernel: [8][22 + 2][64] block-plane table (eik_b2.cuh)
    void* Vt;
    const void* Ht;
    int64_t n1;
    int32_t cps;
    int32_t stats;
    unsigned long long proc_limit;   // async mode: abort after this many processings
    int32_t defer;                   // async mode: readiness deferral (0 off, 1 running
                                     // neighbours, 2 + smaller-key queued, 3 + key - delta)
    float defer_delta;
    int32_t max_sweeps;              // sweeps per processing before continuing later (0: none)
    uint32_t cap;                    // number of cells J (bounds checks)
    uint32_t* pend;                  // J x R^3/32 saved active bits (FLAG_CONT)
    uint32_t* pdir;                  // J: sweep-direction state saved at a sweep cap (FLAG_CONT)
    // whole-grid sweeping (k_dsweep)
    const uint32_t* diag_cells;      // canonical cells a + cps (b + cps c), grouped by a + b + c
    const uint32_t* diag_off;        // [3 cps - 1]: start of each cell diagonal in diag_cells
    uint8_t* cact;                   // DLSM: cell has an input that changed since it last ran
    int32_t locked;                  // 1: DLSM (skip cells whose inputs did not change)
    double kappa;                    // early termination threshold, >= 0
    int32_t legacy_key;              // 1: cell value of Eq. (4), no reset on removal
    int32_t fused;                   // round mode, bin width +inf: k_cell takes its cells straight
                                     // from the current worklist (the whole list is selected) and
                                     // its last CTA ends the round (no k_select / k_round_end)
    int32_t graph;                   // fused + CUDA graph: the last CTA sets the WHILE condition
    unsigned long long cond;         // cudaGraphConditionalHandle of that WHILE node
    // async-mode processing trace (diagnostics, EIK_OPT_TRACE; null = off): per processing two
    // uint4 {cell, processing id of its last tagger, t_pop, t_swept} {t_end, sweeps, flags, gen}
    // (ns since the solve's start), tagger[c] = id of the last processing that tagged c
    uint4* trace;
    uint32_t trace_cap;
    uint32_t* tagger;
};

// preferred sweep directions from the inflow faces (reading R20): a direction
// d has bit0 = x descending, bit1 = y descending, bit2 = z descending.  Inflow through the
// -x face (face 0) prefers x ascending, etc.
__device__ __forceinline__ uint32_t pref_dirs(uint32_t faces)
{
    uint32_t m = 0;
    if (faces & 1u) m |= 0x55u;    // x ascending: d in {0,2,4,6}
    if (faces & 2u) m |= 0xAAu;
    if (faces & 4u) m |= 0x33u;    // y ascending: d in {0,1,4,5}
    if (faces & 8u) m |= 0xCCu;
    if (faces & 16u) m |= 0x0Fu;   // z ascending: d in {0,1,2,3}
    if (faces & 32u) m |= 0xF0u;
    return m;
}

// The halo N(c) of a staged r = 16 cell is stored NEGATED in the shared box (sweep16r: the
// activation test "neighbour > u" is then false outside the cell without a border test);
// every reader of a box neighbour takes habs<R>() of it.  Smaller cells keep plain values (the
// extra sign handling measured 6 % slower on the fp64 r = 8 suite).
template <int R> struct HaloNeg { static constexpr bool value = R == 16; };
template <int R, typename T> __device__ __forceinline__ T habs(T x) { if constexpr (HaloNeg<R>::value) return vabs(x); else return x; }
template <int R, typename T> __device__ __forceinline__ T hneg(T x) { if constexpr (HaloNeg<R>::value) return -x; else return x; }

template <typename T> struct Vec16;
template <> struct Vec16<float> { using type = float4; };
template <> struct Vec16<double> { using type = double2; };

// Shared-memory state of one cell processing (static part; the big arrays are dynamic).
template <int R> struct CellShared {
    unsigned long long plane[2];
    uint32_t face_min[6];              // Eq. (3) min newly-updated inflow value per face
    uint32_t face_max[6];              // Eq. (4) max newly-updated inflow value per face
    uint32_t face_flag;                // faces whose neighbour is currently downwind
    unsigned long long stat[3];
    uint32_t cell, flags;              // async mode broadcast
    uint32_t cont;                     // processing stopped at the sweep cap
    uint32_t cont_key;                 // min V over the points still active (key bits)
    int32_t nact, nact2[2];            // active-point counts
    int32_t lcnt[2], lover;            // active-list lengths / overflow
    uint32_t bwd[2];                   // axes with activations behind the wavefront
    unsigned long long plane0;         // active planes of the first sweep (direction dir0)
    uint32_t tm[8];                    // phase timers (thread 0 only; diagnostics; clock mod 2^32)
    uint32_t nsteps;                   // plane steps of this processing (diagnostics)
    uint32_t dstate;                   // direction state saved at a sweep cap (pdir[c])
};

static_assert(EIK_HF_GLOBAL32 || ((cell_smem_bytes<float, 16>() + sizeof(CellShared<16>) + 16 + 127) / 128 * 128 + 1024) * 5
                  <= 228 * 1024,
              "fp32 r = 16 cell kernels no longer fit 5 CTAs per SM (shared memory)");

// dynamic shared memory carve-up
template <typename T, int R> struct CellSmem {
    static constexpr bool HG = HfGlobal<T, R>::value;
    // async staging of hf by one bulk copy (r = 16 with hf in shared memory: the 16 KB fp32
    // tile; measured 1 % slower than per-thread cp.async for the 4 KB tiles of r = 8)
    static constexpr bool BULK = EIK_HF_BULK && R == 16 && !HG;
    T* V;          // (R+2)^3 box incl. halo faces
    T* H;          // R^3 hf (sign bit set = point changed in this processing); null if HG
    uint8_t* act;  // R^3 active flags (Alg. 2)
    uint32_t* chg; // HG: R^3 changed bits
    uint16_t* list; // 2 x LCAP active-point lists
    const T* Hg;   // HG: this cell's hf tile in global memory (set per processing)
    __device__ explicit CellSmem(unsigned char* raw)
    {
        V = reinterpret_cast<T*>(raw);
        H = HG ? nullptr : V + CellCfg<R>::BOX;
        act = reinterpret_cast<uint8_t*>(V + CellCfg<R>::BOX + (HG ? 0 : CellCfg<R>::R3));
        chg = HG ? reinterpret_cast<uint32_t*>(act + CellCfg<R>::R3 + 16) : nullptr;   // act[R3] = scratch
        list = HG ? reinterpret_cast<uint16_t*>(chg + CellCfg<R>::R3 / 32)
                  : reinterpret_cast<uint16_t*>(act + CellCfg<R>::R3 + 16);
        Hg = nullptr;
    }
    // mbarrier of the bulk hf copy: bytes 8-15 of the 16 scratch bytes behind the activity flags
    // (byte 0: sweep_dir's redirected stores, byte 1: sweep16r's dummy flag)
    __device__ __forceinline__ uint32_t mbar() const { return smem_u32(act + CellCfg<R>::R3 + 8); }
    // direction votes of the active points (bytes 4-7 of the same scratch): three biased 10-bit
    // fields x | y << 10 | z << 20, see cell_process
    __device__ __forceinline__ uint32_t* votes() const { return reinterpret_cast<uint32_t*>(act + CellCfg<R>::R3 + 4); }
    __device__ __forceinline__ T hf(int p) const { if constexpr (HG) return __ldg(Hg + p); else return H[p]; }
    __device__ __forceinline__ bool changed(int p) const
    {
        if constexpr (HG) return (chg[p >> 5] >> (p & 31)) & 1u; else return H[p] < T(0);
    }
    __device__ __forceinline__ void mark(int p, T hs)
    {
        if constexpr (HG) atomicOr(&chg[p >> 5], 1u << (p & 31));
        else if (hs > T(0)) H[p] = -hs;
    }
};

// One wavefront sweep in direction DIR (bit0/1/2 = x/y/z descending).  DIR >= 0: a
// compile-time direction, whose reflection mask and neighbour offsets are immediates (one
// instantiation per direction: r = 16, where a step is long enough to pay for the code
// size); DIR = -1: the direction is the runtime argument rdir (one instantiation: r <= 8,
// where eight copies of the sweep overflow the instruction cache -- measured 3.3x slower on
// the paper's r = 8 fp64 suite).  Returns the axes along which points behind the wavefront
// were activated (bit0 x, bit1 y, bit2 z).
template <typename T, int R, int DIR>
__device__ __forceinline__ uint32_t sweep_dir(CellShared<R>& S, CellSmem<T, R>& M,
                                              const uint16_t* __restrict__ ptab,
                                              unsigned long long pm, bool ungated,
                                              uint32_t& nupd, uint32_t& nwr, uint32_t& nsteps,
                                              T kap, T& dmax, int rdir = 0)
{
    using C = CellCfg<R>;
    constexpr int R3 = C::R3, RP = C::RP, RP2 = C::RP2, NPL = C::NPL, NT = C::NT;
    constexpr int TS = (int)sizeof(T);
    const int dv = DIR >= 0 ? DIR : rdir;
    const bool fx = dv & 1, fy = dv & 2, fz = dv & 4;
    const int tid = threadIdx.x;
    const T INF = dinf<T>();
    // shared-window bases: V box (at the first interior point), hf, activity bytes
    const uint32_t vb = smem_u32(M.V) + (uint32_t)((1 + RP + RP2) * TS);
    constexpr bool HG = CellSmem<T, R>::HG;
    const uint32_t hb = HG ? 0u : smem_u32(M.H);
    const T* __restrict__ hg = M.Hg;
    const uint32_t ab = smem_u32(M.act);
    const uint32_t scratch = ab + R3;   // activity stores that do not apply go here
    bool fwd = false;
    uint32_t bwd = 0;
    int s = __ffsll((long long)pm) - 1;
    // The plane table holds canonical (reflected) coordinates e = a + R b + R^2 c with
    // a + b + c = s.  The point index is p = e XOR dm (R a power of two: reflecting an axis
    // XORs its field); in canonical coordinates "forward" along an axis is +1 and the
    // forward / backward neighbours exist iff the coordinate is < R-1 / > 0.  Box and flag
    // offsets (bytes) of the forward neighbours are compile-time constants.
    const unsigned dm = (fx ? R - 1 : 0) | (fy ? (R - 1) * R : 0) | (fz ? (R - 1) * R * R : 0);
    // (unsigned: address arithmetic wraps modulo 2^32, a negative offset subtracts)
    const uint32_t oxq = (uint32_t)((fx ? -1 : 1) * TS), oyq = (uint32_t)((fy ? -RP : RP) * TS),
                   ozq = (uint32_t)((fz ? -RP2 : RP2) * TS);
    const uint32_t oxp = (uint32_t)(fx ? -1 : 1), oyp = (uint32_t)(fy ? -R : R),
                   ozp = (uint32_t)(fz ? -R * R : R * R);
    // Prefetch pipeline, independent of the current step's results: at step s the thread
    // holds its entry en / hf hn of plane s and the entry en1 of plane s + 1; the step loads
    // hf of plane s + 1 (shared memory, or L1/L2 for HG) and the entry of plane s + 2 (global
    // table via L1, running pointer tq), so no load sits on the step's critical path.  (A
    // pipeline one plane deeper for HG measured neutral on C3d.)  The table has trailing empty
    // planes.
    const uint16_t* tp = ptab + tid;
    unsigned en = __ldg(&tp[s * NT]);
    unsigned en1 = __ldg(&tp[(s + 1) * NT]);
    const uint16_t* tq = tp + (s + 2) * NT;
#define EIK_HFLD(e_) (HG ? __ldg(hg + (e_)) : lds<T>(hb + (e_) * TS))
    // (ha / han: shared address of the current / prefetched point's hf, reused to mark a
    // changed point without recomputing it)
    uint32_t han = hb + (en ^ dm) * TS, ha = han;
    T hn = en < (unsigned)R3 ? EIK_HFLD(en ^ dm) : INF;
#define EIK_PREFETCH(sp_)                                                                  \
    {                                                                                  \
        en = en1;                                                                      \
        ha = han;                                                                      \
        han = hb + (en ^ dm) * TS;                                                     \
        hn = en < (unsigned)R3 ? (HG ? __ldg(hg + (en ^ dm)) : lds<T>(han)) : INF;     \
        en1 = __ldg(tq);                                                               \
        tq += NT;                                                                      \
    }
    // box byte offset of point p = a + R b + R^2 c (relative to vb):
    // a + RP b + RP2 c = p + (RP - R) b + (RP2 - R^2) c
#define EIK_QOFF(up_) (((up_) + (RP - R) * (((up_) / R) & (R - 1)) + (RP2 - R * R) * ((up_) / (R * R))) * TS)
    // First sweep of a cell with many active points (a fresh cell the front is entering):
    // relax every point of every plane without per-point gating -- nearly all of them
    // change anyway -- and record only the activations *behind* the wavefront, which the
    // next sweep needs (forward neighbours are visited later in this same sweep).
    if (ungated) {
        for (; s < NPL; ++s) {
            const unsigned ue = en;
            const T hs = hn;
            EIK_PREFETCH(s + 1)
            if (ue < (unsigned)R3) {
                const unsigned up = ue ^ dm;
                EIK_CHECK(up < (unsigned)R3, "wavefront point index");
                sts_u8(ab + up, 0u);                                   // Alg. 2 line 4
                const uint32_t qa = vb + EIK_QOFF(up);
                const T v = lds<T>(qa);
                const T xf = lds<T>(qa + oxq), xb = lds<T>(qa - oxq);
                const T yf = lds<T>(qa + oyq), yb = lds<T>(qa - oyq);
                const T zf = lds<T>(qa + ozq), zb = lds<T>(qa - ozq);
                const T mx = vmin(habs<R>(xf), habs<R>(xb)), my = vmin(habs<R>(yf), habs<R>(yb)),
                        mz = vmin(habs<R>(zf), habs<R>(zb));   // (HaloNeg)
                const T hf = fabs(hs);
                if (hf < INF && vmin(mx, vmin(my, mz)) < v) {
                    ++nupd;
                    const T u = local_solve_fast<T>(mx, my, mz, hf);
                    if (u < v) {
                        sts(qa, u);
                        if constexpr (HG) atomicOr(&M.chg[up >> 5], 1u << (up & 31));
                        else sts(ha, -hf);   // sign bit = changed (idempotent)
                        ++nwr;
                        // kappa: a change <= kappa activates nothing (ut = +inf)
                        const T ut = (v - u > kap) ? u : INF;
                        dmax = vmax(dmax, v - u);
                        const unsigned ca = ue & (R - 1), cb = (ue / R) & (R - 1), cc = ue / (R * R);
                        const int bxa = (xb > ut) & (ca > 0), bya = (yb > ut) & (cb > 0), bza = (zb > ut) & (cc > 0);
                        sts_u8(bxa ? ab + up - oxp : scratch, 1u);
                        sts_u8(bya ? ab + up - oyp : scratch, 1u);
                        sts_u8(bza ? ab + up - ozp : scratch, 1u);
                        bwd |= (unsigned)(bxa | (bya << 1) | (bza << 2));
                    }
                }
            }
            __syncthreads();
            ++nsteps;
        }
    }
    for (; s < NPL; ++s) {
        const bool has = (pm >> s) & 1ull;
        if (!has && !fwd) {
            if ((pm >> s) == 0ull) break;
            EIK_PREFETCH(s + 1)
            continue;
        }
        const unsigned ue = en;
        const T hs = hn;
        EIK_PREFETCH(s + 1)   // independent of this step's results
        bool myfwd = false;
        if (ue < (unsigned)R3) {
            const unsigned up = ue ^ dm;
            EIK_CHECK(up < (unsigned)R3, "wavefront point index");
            // the flag and the seven box values are loaded together (one shared-memory round
            // trip on the step's critical path instead of two)
            const uint32_t qa = vb + EIK_QOFF(up);
            const uint32_t fl = lds_u8(ab + up);
            const T v = lds<T>(qa);
            const T xf = lds<T>(qa + oxq), xb = lds<T>(qa - oxq);
            const T yf = lds<T>(qa + oyq), yb = lds<T>(qa - oyq);
            const T zf = lds<T>(qa + ozq), zb = lds<T>(qa - ozq);
            if (fl) {
                sts_u8(ab + up, 0u);                                   // Alg. 2 line 4
                const T mx = vmin(habs<R>(xf), habs<R>(xb)), my = vmin(habs<R>(yf), habs<R>(yb)),
                        mz = vmin(habs<R>(zf), habs<R>(zb));   // (HaloNeg)
                const T hf = fabs(hs);
                if (hf < INF && vmin(mx, vmin(my, mz)) < v) {          // fixed / no gain
                    ++nupd;
                    const T u = local_solve_fast<T>(mx, my, mz, hf);    // line 5
                    if (u < v) {                                         // line 6
                        sts(qa, u);                                      // line 7
                        if constexpr (HG) atomicOr(&M.chg[up >> 5], 1u << (up & 31));   // mark changed
                        else sts(ha, -hf);   // sign bit = changed (idempotent)
                        ++nwr;
                        // lines 8-13: activate larger in-cell neighbours (the cross-border
                        // "currently downwind" test is done once per processing)
                        const unsigned ca = ue & (R - 1), cb = (ue / R) & (R - 1), cc = ue / (R * R);
                        // kappa: a change <= kappa activates nothing (ut = +inf)
                        const T ut = (v - u > kap) ? u : INF;
                        // activations as unconditional byte stores to either the neighbour
                        // or a scratch byte (short-lived compares, no predicate pressure)
                        const int fxa = (xf > ut) & (ca < R - 1), bxa = (xb > ut) & (ca > 0);
                        const int fya = (yf > ut) & (cb < R - 1), bya = (yb > ut) & (cb > 0);
                        const int fza = (zf > ut) & (cc < R - 1), bza = (zb > ut) & (cc > 0);
                        sts_u8(fxa ? ab + up + oxp : scratch, 1u);
                        sts_u8(bxa ? ab + up - oxp : scratch, 1u);
                        sts_u8(fya ? ab + up + oyp : scratch, 1u);
                        sts_u8(bya ? ab + up - oyp : scratch, 1u);
                        sts_u8(fza ? ab + up + ozp : scratch, 1u);
                        sts_u8(bza ? ab + up - ozp : scratch, 1u);
                        myfwd = (fxa | fya | fza) != 0;
                        bwd |= (unsigned)(bxa | (bya << 1) | (bza << 2));
                    }
                }
            }
        }
        fwd = __syncthreads_or(myfwd);
        ++nsteps;
    }
#undef EIK_QOFF
#undef EIK_PREFETCH
#undef EIK_HFLD
    return bwd;
}

// L2 cache-eviction policy "evict last" and a read-only load with it (fp64 hf in global memory)
__device__ __forceinline__ unsigned long long l2_evict_last_policy()
{
    unsigned long long p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ldg_keep(const double* a, unsigned long long pol)
{
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ float ldg_keep(const float* a, unsigned long long pol)
{
    float v;
    asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}

// ---- r = 16 wavefront sweep with a packed per-direction plane table -------------------------
// tab16[d][s][t] (built on the host, eik.cu make_tab16) describes the t-th point of plane s of
// direction d: bits 0-12 its box index q = (a+1) + 18 (b+1) + 324 (c+1), bits 19-31 its point
// index p = a + 16 b + 256 c (bits 13-18 unused).  A thread with no point on a plane gets
// T16_DUMMY: a halo box index (reads only), the flag byte act[T16_DUMMY_P], which is 0 for the
// whole processing, and no hf -- so every lane runs the same straight-line step (no divergence),
// and a warp whose lanes are all dummies skips the step's loads (one vote).
//
// The direction is a runtime argument: one instantiation instead of eight (eight copies of the
// two step loops were ~45 KB of SASS per precision; with five CTAs per SM in different
// directions and phases the instruction caches missed: ncu "no instruction" 8 % of the C5 stall
// samples).  Nothing in the step depends on the direction any more:
//  * the six neighbours are addressed physically (+-x, +-y, +-z: immediates); the local solve
//    only needs min(x+, x-) etc.;
//  * the halo N(c) is stored NEGATED in the box (see stage_cell_async), so |value| enters the
//    minima (a free source modifier) and the activation test "neighbour > u" (Alg. 2 line 9) is
//    false for every neighbour outside the cell without any border test: u > 0 >= -|halo|;
//  * "some point ahead of the wavefront was activated" is replaced by its superset "some point
//    of the plane changed" (the next plane then runs one idle step at worst), and the axes with
//    activations behind the wavefront come from a 6-bit mask accumulated over the sweep.
// kappa = 0 only (the exact path; kappa > 0 runs sweep_dir).
static constexpr uint32_t T16_DUMMY_P = 16 * 16 * 16 + 1;                       // act[R3 + 1]
static constexpr uint32_t T16_DUMMY = (1u + 18u + 324u) | (T16_DUMMY_P << 19);   // box (-1, 0, 0)
static constexpr int T16_ROWS = 3 * 16 - 2 + 3;   // NPL + 3 trailing empty planes

template <typename T>
__device__ __forceinline__ uint32_t sweep16r(CellSmem<T, 16>& M, const uint32_t* __restrict__ tab, int dir,
                                             unsigned long long pm, bool ungated, uint32_t& nupd,
                                             uint32_t& nwr, uint32_t& nsteps, uint32_t ltid)
{
    using C = CellCfg<16>;
    constexpr int NPL = C::NPL, NT = C::NT, R3 = C::R3;
    constexpr int TS = (int)sizeof(T);
    constexpr bool HG = CellSmem<T, 16>::HG;
    constexpr uint32_t oxq = (uint32_t)TS, oyq = (uint32_t)(C::RP * TS), ozq = (uint32_t)(C::RP2 * TS);
    // physical neighbours ahead of the wavefront of this direction (bit 0 +x, 1 -x, 2 +y, ...)
    const uint32_t fm6 = ((dir & 1) ? 2u : 1u) | ((dir & 2) ? 8u : 4u) | ((dir & 4) ? 32u : 16u);
    const T INF = dinf<T>();
    const uint32_t vb = smem_u32(M.V);
    const uint32_t hb = HG ? 0u : smem_u32(M.H);
    const T* __restrict__ hg = M.Hg;
    const uint32_t ab = smem_u32(M.act);
    const uint32_t* __restrict__ tp = tab + dir * T16_ROWS * NT + ltid;   // (ltid: see k_async)
    // HG (fp64): the cell's hf tile is read once per sweep through L2; an evict_last policy keeps
    // it there between the sweeps of a processing instead of re-fetching it from HBM
    const unsigned long long l2keep = HG ? l2_evict_last_policy() : 0ull;
#ifndef EIK16_HG_DEEP
#define EIK16_HG_DEEP 0   // sweep16r, hf from global memory: prefetch it two planes ahead (measured neutral on C3d)
#endif
#ifndef EIK16_EXACT_FWD
#define EIK16_EXACT_FWD 0
#endif
#if EIK16_EXACT_FWD
#define EIK16_ACC am
#else
#define EIK16_ACC bwd6
#endif
    bool fwd = false;
    uint32_t bwd6 = 0, cnt = 0;   // cnt: this sweep's updates | writes << 16 (<= 46 each per thread)
    int s = __ffsll((long long)pm) - 1;
    unsigned long long pmr = pm >> s;   // pm >> (current plane)
    // prefetch pipeline: the table entry two planes ahead, hf one plane ahead (shared memory);
    // HG (hf from global memory / L2, fp64) runs one plane deeper: entry three, hf two ahead
    constexpr bool DEEP = HG && EIK16_HG_DEEP;
    uint32_t en = __ldg(tp + s * NT);
    uint32_t en1 = __ldg(tp + (s + 1) * NT);
    uint32_t en2 = DEEP ? __ldg(tp + (s + 2) * NT) : 0u;
    tp += (s + (DEEP ? 3 : 2)) * NT;
#define EIK16_HF(e_) (HG ? (((e_) >> 19) < (uint32_t)R3 ? ldg_keep(hg + ((e_) >> 19), l2keep) : INF)   \
                         : lds<T>(hb + ((e_) >> 19) * TS))
    T hn = EIK16_HF(en);
    T hn1 = DEEP ? EIK16_HF(en1) : T(0);
#define EIK16_PREFETCH()                                                                   \
    {                                                                                      \
        en = en1;                                                                          \
        if constexpr (DEEP) {                                                              \
            en1 = en2;                                                                     \
            hn = hn1;                                                                      \
            hn1 = EIK16_HF(en1);                                                           \
            en2 = __ldg(tp);                                                               \
        } else {                                                                           \
            hn = EIK16_HF(en);                                                             \
            en1 = __ldg(tp);                                                               \
        }                                                                                  \
        tp += NT;                                                                          \
    }
#define EIK16_MARK(ue_, hf_)                                                               \
    {                                                                                      \
        EIK_CHECK(((ue_) >> 19) < (uint32_t)R3, "sweep16r changed point");                 \
        if constexpr (HG) atomicOr(&M.chg[(ue_) >> 24], 1u << (((ue_) >> 19) & 31));      \
        else sts(hb + ((ue_) >> 19) * TS, -(hf_));   /* sign bit = changed */              \
    }
    // One step.  FLD_: load the activity flag (gated sweeps); GATE_: the lane's gate; EN_(i):
    // whether neighbour i may be activated (ungated sweeps: only those behind the wavefront).
#define EIK16_STEP(FLD_, GATE_, EN_, ONE_)                                                 \
        const uint32_t qa = vb + (ue & 0x1fffu) * TS;                                      \
        const uint32_t fa = ab + (ue >> 19);                                               \
        const uint32_t fl = (FLD_) ? lds_u8(fa) : 1u;                                      \
        const T v = lds<T>(qa);                                                            \
        const T xp = lds<T>(qa + oxq), xm = lds<T>(qa - oxq);                              \
        const T yp = lds<T>(qa + oyq), ym = lds<T>(qa - oyq);                              \
        const T zp = lds<T>(qa + ozq), zm = lds<T>(qa - ozq);                              \
        const T mx = vmin(vabs(xp), vabs(xm)), my = vmin(vabs(yp), vabs(ym)),              \
                mz = vmin(vabs(zp), vabs(zm));                                             \
        const T hf = vabs(hs);                                                             \
        sts_u8(fa, 0u);   /* Alg. 2 line 4 (nothing activates plane s during step s) */    \
        const bool gate = (GATE_) && hf < INF && vmin(mx, vmin(my, mz)) < v;               \
        if (__any_sync(0xffffffffu, gate)) {                                               \
            const T u = local_solve_fast<T>(mx, my, mz, hf);          /* line 5 */         \
            chg = gate && u < v;                                      /* line 6 */         \
            cnt += (gate ? 1u : 0u) + (chg ? 0x10000u : 0u);   /* updates | writes << 16 */ \
            if (chg) {                                                                     \
                sts(qa, u);                                           /* line 7 */         \
                EIK16_MARK(ue, hf)                                                         \
            }                                                                              \
            /* lines 8-13: activate larger in-cell neighbours (halo values are negative: no \
               border test; the cross-border "currently downwind" test is done once per     \
               processing) */                                                              \
            const T ut = chg ? u : INF;                                                    \
            if (EN_(0) && xp > ut) { sts_u8(fa + 1u, ONE_); EIK16_ACC |= 1u; }                    \
            if (EN_(1) && xm > ut) { sts_u8(fa - 1u, ONE_); EIK16_ACC |= 2u; }                    \
            if (EN_(2) && yp > ut) { sts_u8(fa + 16u, ONE_); EIK16_ACC |= 4u; }                   \
            if (EN_(3) && ym > ut) { sts_u8(fa - 16u, ONE_); EIK16_ACC |= 8u; }                   \
            if (EN_(4) && zp > ut) { sts_u8(fa + 256u, ONE_); EIK16_ACC |= 16u; }                 \
            if (EN_(5) && zm > ut) { sts_u8(fa - 256u, ONE_); EIK16_ACC |= 32u; }                 \
        }
    if (ungated) {
        // first sweep of a fresh cell: every point of every plane, only the activations behind
        // the wavefront are recorded (forward neighbours are visited later in this sweep)
        // (forward neighbours are activated too: each clears its flag when its own plane is
        // visited later in this sweep -- cheaper than a per-direction enable test per neighbour)
#define EIK16_EN_U(i_) true
        // (Measured and rejected: running the corner planes -- the first six and last seven hold
        // <= 28 points, all in one warp -- with warp barriers only; making this loop's CTA
        // barrier conditional cost 10 % on C5, whichever corner was warp-local.)
        for (; s < NPL; ++s) {
            const uint32_t ue = en;
            const T hs = hn;
            EIK16_PREFETCH()
            if (!__all_sync(0xffffffffu, ue == T16_DUMMY)) {
                bool chg = false;
                uint32_t am = 0;
                // (any byte with bit 0 set is an activity flag; ue | 1 needs no constant register)
                const uint32_t one = ue | 1u;
                EIK16_STEP(false, ue != T16_DUMMY, EIK16_EN_U, one)
                (void)fl;
                bwd6 |= am;
            }
            __syncthreads();
            ++nsteps;
        }
#undef EIK16_EN_U
        pmr = 0;
    }
#define EIK16_EN_G(i_) true
    for (; s < NPL; ++s, pmr >>= 1) {
        const bool go = ((uint32_t)pmr & 1u) | (uint32_t)fwd;   // (CTA-uniform)
        if (!go && pmr == 0ull) break;
        const uint32_t ue = en;
        const T hs = hn;
        EIK16_PREFETCH()
        if (!go) continue;   // plane without active points: no step, no barrier
        bool chg = false;
        uint32_t am = 0;
        if (!__all_sync(0xffffffffu, ue == T16_DUMMY)) {
            EIK16_STEP(true, fl, EIK16_EN_G, fl)
        }
#if EIK16_EXACT_FWD
        bwd6 |= am;
        fwd = __syncthreads_or(am & fm6);
#else
        (void)am;
        fwd = __syncthreads_or(chg);
#endif
        ++nsteps;
    }
#undef EIK16_EN_G
#undef EIK16_ACC
#undef EIK16_STEP
#undef EIK16_HF
#undef EIK16_PREFETCH
#undef EIK16_MARK
    nupd += cnt & 0xffffu;
    nwr += cnt >> 16;
    const uint32_t b6 = bwd6 & ~fm6;
    return ((b6 & 3u) ? 1u : 0u) | ((b6 & 12u) ? 2u : 0u) | ((b6 & 48u) ? 4u : 0u);
}

// Stage cell c (tile coordinates cx, cy, cz) into shared memory: the tile and its hf go out
// as cp.async (no registers), the halo N(c) as L2 loads issued right behind them -- one
// memory round trip for all of it; returns when this thread's copies have landed (the caller
// synchronises the CTA).  The tile's element-wise copies (into the padded box) use .ca, which
// is safe for the cell's own tile: no other CTA writes it within a launch, and L1 does not
// survive the kernel boundary.  The halo must come from L2 (.cg): a neighbour processed
// earlier in this launch on another SM may have changed it after this SM cached the lines.
template <typename T, int R>
__device__ __forceinline__ void stage_cell_async(const T* __restrict__ Vt, const T* __restrict__ Ht,
                                                 CellSmem<T, R>& M, uint32_t c, int cx, int cy, int cz,
                                                 int cps, uint32_t cap)
{
    using C = CellCfg<R>;
    constexpr int NT = C::NT, R3 = C::R3, RP = C::RP, RP2 = C::RP2;
    const int tid = threadIdx.x;
    const T INF = dinf<T>();
    const int64_t base = (int64_t)c * R3;
    (void)cap;
    T* sV = M.V;
    const uint32_t vs = smem_u32(sV);
    constexpr int EL = 16 / sizeof(T);
    if constexpr (CellSmem<T, R>::HG) {
        M.Hg = Ht + base;
        for (int w = tid; w < R3 / 32; w += NT) M.chg[w] = 0u;
    } else {
        const uint32_t hs = smem_u32(M.H);
        for (int vi = tid; vi < R3 / EL; vi += NT) cp_async16(hs + vi * 16, Ht + base + vi * EL);
    }
    for (int e = tid; e < R3; e += NT) {
        const int a = e & (R - 1), b = (e / R) & (R - 1), d = e / (R * R);
        cp_async_el(vs + ((a + 1) + RP * (b + 1) + RP2 * (d + 1)) * (int)sizeof(T), Vt + base + e);
    }
    constexpr int PH = (6 * R * R + NT - 1) / NT;     // halo elements per thread
    T hv[PH];
    int hq[PH];
#pragma unroll
    for (int m = 0; m < PH; ++m) {
        const int e = tid + m * NT;
        hq[m] = -1;
        hv[m] = INF;
        if (e < 6 * R * R) {
            const int f = e / (R * R), uv = e - f * R * R, u = uv % R, v = uv / R;
            int hx, hy, hz, sa, sb, sd;
            int64_t nc;
            bool ex;
            switch (f) {
            case 0: hx = -1; hy = u; hz = v; ex = cx > 0; nc = (int64_t)c - 1; sa = R - 1; sb = u; sd = v; break;
            case 1: hx = R; hy = u; hz = v; ex = cx < cps - 1; nc = (int64_t)c + 1; sa = 0; sb = u; sd = v; break;
            case 2: hx = u; hy = -1; hz = v; ex = cy > 0; nc = (int64_t)c - cps; sa = u; sb = R - 1; sd = v; break;
            case 3: hx = u; hy = R; hz = v; ex = cy < cps - 1; nc = (int64_t)c + cps; sa = u; sb = 0; sd = v; break;
            case 4: hx = u; hy = v; hz = -1; ex = cz > 0; nc = (int64_t)c - (int64_t)cps * cps; sa = u; sb = v; sd = R - 1; break;
            default: hx = u; hy = v; hz = R; ex = cz < cps - 1; nc = (int64_t)c + (int64_t)cps * cps; sa = u; sb = v; sd = 0; break;
            }
            hq[m] = (hx + 1) + RP * (hy + 1) + RP2 * (hz + 1);
            EIK_CHECK(!ex || (nc >= 0 && nc < (int64_t)cap), "halo neighbour cell");
            if (ex) hv[m] = __ldcg(&Vt[nc * R3 + sa + R * sb + R * R * sd]);
        }
    }
#pragma unroll
    for (int m = 0; m < PH; ++m)
        if (hq[m] >= 0) sV[hq[m]] = hneg<R>(hv[m]);   // r = 16: the halo is stored negated (HaloNeg)
    cp_async_wait_all();
}

// Write back the changed points of a staged cell (sign bit of hf set): 16-byte vectors, a
// vector holding any changed point is stored whole (unchanged values are rewritten
// identically).  Returns the number of changed points this thread wrote.
template <typename T, int R>
__device__ __forceinline__ unsigned long long write_back_changed(T* __restrict__ Vc, const CellSmem<T, R>& M)
{
    using C = CellCfg<R>;
    constexpr int NT = C::NT, R3 = C::R3, RP = C::RP, RP2 = C::RP2;
    using V4 = typename Vec16<T>::type;
    constexpr int EL = 16 / sizeof(T);
    constexpr int NV = R3 / EL;
    unsigned long long nw = 0;
    V4* Vt4 = reinterpret_cast<V4*>(Vc);
    const T* sV = M.V;
    for (int vi = threadIdx.x; vi < NV; vi += NT) {
        int nchg = 0;
        if constexpr (CellSmem<T, R>::HG) {
            nchg = __popc((M.chg[(vi * EL) >> 5] >> ((vi * EL) & 31)) & ((1u << EL) - 1u));
        } else {
            const V4 hv = reinterpret_cast<const V4*>(M.H)[vi];
            const T* ph = reinterpret_cast<const T*>(&hv);
#pragma unroll
            for (int l = 0; l < EL; ++l) nchg += ph[l] < T(0);
        }
        if (nchg) {
            V4 out;
            T* po = reinterpret_cast<T*>(&out);
#pragma unroll
            for (int l = 0; l < EL; ++l) {
                const int e = vi * EL + l;
                const int a = e & (R - 1), b = (e / R) & (R - 1), d = e / (R * R);
                po[l] = sV[(a + 1) + RP * (b + 1) + RP2 * (d + 1)];
            }
            __stcg(&Vt4[vi], out);
            nw += nchg;
        }
    }
    return nw;
}

// Process one cell to convergence (HCM "perform modified LSM on c until convergence",
// Alg. 1 line 6): stage the tile and its one-point halo N(c) (boundary data of
// c~ = c u N(c)), relax the gated (LSM) update of Alg. 2 until no point is active, write
// back changed values.  On return the face summaries (face_flag, face_min) are in S; the
// caller re-activates neighbours.
//
// Two relaxation orders, both exact Gauss-Seidel/chaotic relaxations of Eq. (2) that reach
// the same fixed point (any order does: values only decrease):
//  * wavefront sweeps while many points are active: a sweep in direction d visits the
//    planes s = i' + j' + k' = 0 .. 3R-3 (primes = coordinates reflected per d) in order,
//    i.e. the exact GS ordering of that sweep (Detrixhe et al. planes).
//    The points of a plane are independent and are packed onto consecutive threads through
//    a shared plane table; a step ends in one __syncthreads_or that also reports forward
//    activations; planes without active points are skipped without a barrier.  Activity is
//    one byte per point written with plain stores (several writers only ever store 1).
//  * an active-point list once only a handful of points remain (<= LTHR: 16 for r = 16, never
//    for smaller cells; see LTHR below): every listed point is relaxed at once (chaotic order,
//    FIM-like), newly activated points are claimed with a CAS on their flag word and appended
//    to the next list (capacity LCAP).  If a list overflows, the flags stay authoritative and
//    the wavefront sweeps resume.
// "Changed" is the sign bit of a point's hf; the currently-downwind faces (Eq. (3)) are
// derived once per processing from the changed border points.  Tile traffic bypasses L1
// (ld/st .cg): other CTAs update neighbouring tiles concurrently in the async scheduler.
template <typename T, int R, bool CPASYNC>
__device__ __forceinline__ void cell_process(const CellArgs& A, CellShared<R>& S,
                                             CellSmem<T, R>& M, uint32_t c, uint32_t flags,
                                             unsigned long long& n_sweeps_out, uint32_t ltid = threadIdx.x,
                                             uint32_t hpar = 0u)
{
    using C = CellCfg<R>;
    constexpr int NT = C::NT, R3 = C::R3, RP = C::RP, RP2 = C::RP2, NPL = C::NPL;
    constexpr int LCAP = C::LCAP;
    // The list relaxation replaces sweeps only for a handful of active points (r = 16: <= 16;
    // r <= 8: never).  It was introduced (round 1) with a threshold of the list capacity (384 /
    // 128 points) to cut the tail of late sweeps, but a chaotic relaxation needs up to one
    // iteration per plane to carry a change across the cell, each with two CTA barriers and
    // shared-memory atomics, where one gated sweep in the right direction does it in one pass:
    // measured with the round-2 step (threshold 384 -> 16): C1 1.44 -> 0.90 ms, C4 9.5 -> 6.5,
    // C3 6.32 -> 5.69, C3d 21.4 -> 19.7, P3 10.4 -> 8.5 (never), PMAZE 39.6 -> 34.9, C5 30.4 -> 29.9.
    constexpr int LTHR = EIK_LIST_THR == -2 ? (R == 16 ? 16 : 0)
                       : EIK_LIST_THR < 0 ? 0 : (EIK_LIST_THR > 0 && EIK_LIST_THR < LCAP) ? EIK_LIST_THR : LCAP;
    const int tid = threadIdx.x;
    T* Vt = reinterpret_cast<T*>(A.Vt);
    const T* Ht = reinterpret_cast<const T*>(A.Ht);
    T* sV = M.V;
    uint8_t* sA = M.act;
    const int cps = A.cps;
    const T INF = dinf<T>();
    const int cx = (int)(c % (uint32_t)cps), cy = (int)((c / (uint32_t)cps) % (uint32_t)cps),
              cz = (int)(c / ((uint32_t)cps * (uint32_t)cps));
    const int64_t base = (int64_t)c * R3;
    const T kap = (T)A.kappa;   // early termination threshold; 0 = exact
    T dmax_ = T(0);             // (largest change: used by the whole-grid sweeps only)
    if (tid < 6) { S.face_min[tid] = KEY_INF; S.face_max[tid] = 0u; }
    if (tid == 0) {
        S.face_flag = 0;
        S.plane[0] = 0; S.plane[1] = ~0ull; S.cont = 0; S.cont_key = KEY_INF;   // (plane[1]: argmin slot until the first sweep)
        S.plane0 = 0; S.nact2[0] = S.nact2[1] = 0;
        S.nact = 0; S.lcnt[0] = S.lcnt[1] = 0; S.lover = 0;
        sA[R3 + 1] = 0;   // sweep16's dummy flag byte (T16_DUMMY_P): never set
        if (EIK_DIR_VOTE) *M.votes() = 512u | (512u << 10) | (512u << 20);
    }
    // phase timers live in shared memory, written by thread 0 only (no registers held
    // across the sweeps): tm = {start, tile staged, halo staged, init done, mask, steps, list
    // iterations, face summaries start}
    if (tid == 0) { S.tm[0] = (uint32_t)clock64(); S.tm[4] = 0; S.tm[5] = 0; S.tm[6] = 0; }
    uint32_t nsteps = 0;
    constexpr int NWB = R3 / 32;   // saved-bitmask words

    // ---- stage V and hf with 16-byte vector loads (all of a batch in flight before any
    // store: memory-level parallelism), then the halo N(c) ----
    if constexpr (CPASYNC) {
        // Round mode: cp.async staging (see stage_cell_async; a round is one launch, and a
        // neighbour's re-activation of this cell may be consumed by this very processing in
        // fused rounds, hence the halo from L2)
        stage_cell_async<T, R>(Vt, Ht, M, c, cx, cy, cz, cps, A.cap);
        if (tid == 0) S.tm[1] = (uint32_t)clock64();
    } else {
        // Async mode: a cell's tile may have been written by a CTA on another SM since this
        // SM last cached it, so V comes through L2 only (16-byte .cg vector loads into
        // registers).  hf is read-only during the solve: cp.async (no registers).  The halo
        // loads are issued before the tile batches, all in one memory round trip.
        using V4 = typename Vec16<T>::type;
        constexpr int EL = 16 / sizeof(T);                // elements per vector
        constexpr int NV = R3 / EL;                       // vectors per tile
        constexpr int PV = (NV + NT - 1) / NT;            // vectors per thread
        constexpr int B = sizeof(T) == 4 ? EIK_STAGE_B32 : EIK_STAGE_B64;   // batch (register budget)
        const V4* Vt4 = reinterpret_cast<const V4*>(Vt + base);
        if constexpr (CellSmem<T, R>::HG) {
            M.Hg = Ht + base;
            for (int w = tid; w < R3 / 32; w += NT) M.chg[w] = 0u;
        } else {
            if constexpr (CellSmem<T, R>::BULK) {
                // hf (read-only during the solve): one bulk copy by thread 0 (see bulk_g2s)
                if (tid == 0) bulk_g2s(smem_u32(M.H), Ht + base, (uint32_t)(R3 * sizeof(T)), M.mbar());
            } else {
                const uint32_t hsb = smem_u32(M.H);
                for (int vi = tid; vi < NV; vi += NT) cp_async16(hsb + vi * 16, Ht + base + vi * EL);
            }
        }
        constexpr int PH = (6 * R * R + NT - 1) / NT;     // halo elements per thread
        T hv[PH];
        // (the box index of a halo element is recomputed at its store instead of being held in
        // a register across the tile loads: all tile vectors of a thread can then be in flight)
#pragma unroll
        for (int m = 0; m < PH; ++m) {
            const int e = tid + m * NT;
            hv[m] = INF;
            if (e < 6 * R * R) {
                const int f = e / (R * R), uv = e - f * R * R, u = uv % R, v = uv / R;
                int sa, sb, sd;
                int64_t nc;
                bool ex;
                switch (f) {
                case 0: ex = cx > 0; nc = (int64_t)c - 1; sa = R - 1; sb = u; sd = v; break;
                case 1: ex = cx < cps - 1; nc = (int64_t)c + 1; sa = 0; sb = u; sd = v; break;
                case 2: ex = cy > 0; nc = (int64_t)c - cps; sa = u; sb = R - 1; sd = v; break;
                case 3: ex = cy < cps - 1; nc = (int64_t)c + cps; sa = u; sb = 0; sd = v; break;
                case 4: ex = cz > 0; nc = (int64_t)c - (int64_t)cps * cps; sa = u; sb = v; sd = R - 1; break;
                default: ex = cz < cps - 1; nc = (int64_t)c + (int64_t)cps * cps; sa = u; sb = v; sd = 0; break;
                }
                EIK_CHECK(!ex || (nc >= 0 && nc < (int64_t)A.cap), "halo neighbour cell");
                if (ex) hv[m] = __ldcg(&Vt[nc * R3 + sa + R * sb + R * R * sd]);
            }
        }
#pragma unroll
        for (int m0 = 0; m0 < PV; m0 += B) {
            V4 va[B];
#pragma unroll
            for (int m = 0; m < B; ++m) {
                const int vi = tid + (m0 + m) * NT;
                if (m0 + m < PV && vi < NV) va[m] = __ldcg(&Vt4[vi]);
            }
#pragma unroll
            for (int m = 0; m < B; ++m) {
                const int vi = tid + (m0 + m) * NT;
                if (m0 + m < PV && vi < NV) {
                    const T* pv = reinterpret_cast<const T*>(&va[m]);
#pragma unroll
                    for (int l = 0; l < EL; ++l) {
                        const int e = vi * EL + l;
                        const int a = e & (R - 1), b = (e / R) & (R - 1), d = e / (R * R);
                        sV[(a + 1) + RP * (b + 1) + RP2 * (d + 1)] = pv[l];
                    }
                }
            }
        }
#pragma unroll
        for (int m = 0; m < PH; ++m) {
            const int e = tid + m * NT;
            if (e < 6 * R * R) {
                const int f = e / (R * R), uv = e - f * R * R, u = uv % R, v = uv / R;
                const int hx = f == 0 ? -1 : f == 1 ? R : u;
                const int hy = f < 2 ? u : f == 2 ? -1 : f == 3 ? R : v;
                const int hz = f < 4 ? v : f == 4 ? -1 : R;
                sV[(hx + 1) + RP * (hy + 1) + RP2 * (hz + 1)] = hneg<R>(hv[m]);   // r = 16: stored negated (HaloNeg)
            }
        }
        if constexpr (CellSmem<T, R>::BULK) mbar_wait(M.mbar(), hpar & 1u);
        else cp_async_wait_all();
        if (tid == 0) S.tm[1] = (uint32_t)clock64();
        // async mode: `flags` is valid in thread 0 only (the result of its claim of the cell,
        // whose round trip overlapped the loads above); the others take it from S.flags
        if (tid == 0) S.flags = flags;
    }
    __syncthreads();
    if constexpr (!CPASYNC) flags = S.flags;
    const bool init = flags & FLAG_INIT;
    // ---- initial activity: all points (INIT), or the points of the inflow faces whose
    // outside neighbour is smaller (only smaller neighbours enter Eq. (2)), plus the
    // points saved at a sweep cap.  The first sweep's direction is fixed by the inflow faces,
    // so its set of active planes is collected here (no separate scan) ----
    __syncthreads();
    if (tid == 0) S.tm[2] = (uint32_t)clock64();
    // Sweep-direction state.  A continuation after a sweep cap resumes the direction sequence
    // where the capped processing left it (the saved word holds the direction chosen for the
    // sweep it did not run, the Gray-cycle position and the age of each axis' last reversal);
    // restarting from the inflow faces would repeat the same first sweeps every processing.
    int gi = 0, lf0 = -64, lf1 = -64, lf2 = -64;   // lfX: sweep of axis X's last reversal
    const uint32_t dsave = (flags & FLAG_CONT) ? __ldcg(&A.pdir[c]) : 0u;
    const bool resumed = dsave >> 31;
    int dir0 = (init || !(flags & 63u)) ? 0 :
        (((flags & 2u) && !(flags & 1u) ? 1 : 0) | ((flags & 8u) && !(flags & 4u) ? 2 : 0) |
         ((flags & 32u) && !(flags & 16u) ? 4 : 0));
    if (resumed) {
        dir0 = (int)(dsave & 7u);
        gi = (int)((dsave >> 3) & 7u);
        lf0 = -(int)((dsave >> 9) & 63u);
        lf1 = -(int)((dsave >> 15) & 63u);
        lf2 = -(int)((dsave >> 21) & 63u);
    }
    {
        int cnt = 0;
        unsigned long long pm0 = 0;
        auto plane0 = [&](int a, int b, int d) {
            return ((dir0 & 1) ? R - 1 - a : a) + ((dir0 & 2) ? R - 1 - b : b) + ((dir0 & 4) ? R - 1 - d : d);
        };
        uint32_t* sA32 = reinterpret_cast<uint32_t*>(sA);
        if (init) {
            for (int w = tid; w < R3 / 4; w += NT) sA32[w] = 0x01010101u;
            cnt = tid == 0 ? R3 : 0;
            pm0 = tid == 0 ? ((1ull << NPL) - 1ull) : 0ull;
        } else {
            for (int w = tid; w < R3 / 4; w += NT) sA32[w] = 0u;
            __syncthreads();
            // face points whose outside neighbour is smaller.  EIK_DIR0_ACT: the activated
            // points are also counted per face (S.face_max, free until the face summaries) and
            // the smallest activating value is located (S.plane[1], free until the first sweep):
            // the first sweep's direction follows the faces that really bring information, not
            // every face that was tagged (see below)
            // (r >= 8: the face elements of a warp's loop iteration lie on one face)
            constexpr bool D0 = EIK_DIR0_ACT && (6 * R * R) % NT == 0 && (R * R) % 32 == 0;
            uint32_t mk = KEY_INF, mp = 0;
            for (int e = tid; e < 6 * R * R; e += NT) {
                const int f = e / (R * R);   // (warp-uniform)
                if (!(flags & (1u << f))) continue;
                const int uv = e - f * R * R, u = uv & (R - 1), v = uv / R;
                int a, b, d, off;
                switch (f) {
                case 0: a = 0; b = u; d = v; off = -1; break;
                case 1: a = R - 1; b = u; d = v; off = 1; break;
                case 2: a = u; b = 0; d = v; off = -RP; break;
                case 3: a = u; b = R - 1; d = v; off = RP; break;
                case 4: a = u; b = v; d = 0; off = -RP2; break;
                default: a = u; b = v; d = R - 1; off = RP2; break;
                }
                const int q = (a + 1) + RP * (b + 1) + RP2 * (d + 1);
                const T ov = habs<R>(sV[q + off]);   // (HaloNeg)
                const bool act = ov < sV[q];
                if (act) {
                    sA[a + R * b + R * R * d] = 1;
                    ++cnt;
                    pm0 |= 1ull << plane0(a, b, d);
                }
                if constexpr (D0) {
                    const uint32_t kb = act ? key_bits(ov) : KEY_INF;
                    if (kb < mk) { mk = kb; mp = (uint32_t)(a + R * b + R * R * d); }
                    const unsigned bal = __ballot_sync(0xffffffffu, act);
                    if ((tid & 31) == 0 && bal) atomicAdd(&S.face_max[f], (uint32_t)__popc(bal));
                }
            }
            if constexpr (D0) {
                const uint32_t wm = __reduce_min_sync(0xffffffffu, mk);
                const unsigned who = __ballot_sync(0xffffffffu, mk == wm);
                const uint32_t wp = __shfl_sync(0xffffffffu, mp, __ffs(who) - 1);
                if ((tid & 31) == 0 && wm != KEY_INF)
                    atomicMin(&S.plane[1], ((unsigned long long)wm << 32) | wp);
            }
            // points saved at a sweep cap
            if (flags & FLAG_CONT) {
                for (int w = tid; w < NWB; w += NT) {
                    uint32_t x = __ldcg(&A.pend[(int64_t)c * NWB + w]);
                    while (x) {
                        const int e = 32 * w + __ffs(x) - 1;
                        x &= x - 1;
                        sA[e] = 1;
                        ++cnt;
                        pm0 |= 1ull << plane0(e & (R - 1), (e / R) & (R - 1), e / (R * R));
                    }
                }
            }
        }
        cnt = (int)warp_add((uint32_t)cnt);
        pm0 = warp_or64(pm0);
        if ((tid & 31) == 0 && cnt) { atomicAdd(&S.nact, cnt); atomicOr(&S.plane0, pm0); }
    }
    __syncthreads();
    if (tid == 0) S.tm[3] = (uint32_t)clock64();
    // EIK_DIR0_ACT: direction of the first sweep of a cell activated through its faces.  The
    // tagged faces alone fix the direction only along axes with exactly one tagged face (an
    // untagged axis defaulted to ascending, and tags of both faces of an axis accumulate while a
    // cell waits: re-processings with >= 4 tagged faces took 2.5-9.7 sweeps on C3).  Instead:
    // along every axis away from the smallest activating value (the flow enters there), except
    // that for r = 16 an axis whose two faces activated different numbers of points goes away
    // from the face with more.  The plane mask collected above belongs to the tag-based
    // direction, so the first sweep takes it from the scan below when the direction changed.
    // Measured: C1 0.77 -> 0.70 ms, C2 3.32 -> 3.04, C3 5.73 -> 5.58, C3d 19.9 -> 18.8, C5 30.1 ->
    // 29.2, P3 8.53 -> 8.00, PMAZE 35.0 -> 33.4; C4 6.55 -> 6.8 (the one config it costs).
    bool pm0_ok = true;
    constexpr bool D0A = EIK_DIR0_ACT && (6 * R * R) % NT == 0 && (R * R) % 32 == 0;
    if (D0A && !init && !resumed && S.nact > 0) {
        const unsigned long long am = S.plane[1];
        const uint32_t ap = (uint32_t)am;
        int nd = 0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const uint32_t cm = S.face_max[2 * ax], cp = S.face_max[2 * ax + 1];
            const int pos = (int)((ap / (ax == 0 ? 1u : ax == 1 ? (uint32_t)R : (uint32_t)(R * R))) & (uint32_t)(R - 1));
            // (measured: the face counts help r = 16 -- C3 5.67 -> 5.58 ms, C3d 19.25 -> 18.8 -- and
            // hurt r = 8, where the smallest value alone decides: P3 8.44 -> 8.00, P2 17.3 -> 16.75;
            // counts alone, without the smallest value, gain nothing)
            const bool desc = (R == 16 && cm != cp) ? cp > cm : pos >= R / 2;
            nd |= desc ? (1 << ax) : 0;
        }
        pm0_ok = nd == dir0;
        dir0 = nd;
    }
    if (D0A && !init) {   // the counters go back to the face summaries' initial value
        __syncthreads();
        if (tid < 6) S.face_max[tid] = 0u;
    }

    int prev_dir = -1;
    bool ran_list = false;
    uint32_t nsweeps = 0;
    uint32_t nupd = 0, nwr = 0;
    int nact = S.nact;     // active points (exact at loop entry)
    for (int sw = 0;; ++sw) {
        if (nact == 0) break;
        // ================= active-list relaxation (few active points) =================
        if (nact <= LTHR) {
            ran_list = true;
            const long long tl0 = tid == 0 ? clock64() : 0;
            // build the list from the flags
            if (tid == 0) { S.lcnt[0] = 0; S.lcnt[1] = 0; S.lover = 0; }
            __syncthreads();
            {
                const uint32_t* sA32 = reinterpret_cast<const uint32_t*>(sA);
                for (int wd = tid; wd < R3 / 4; wd += NT) {
                    uint32_t x = sA32[wd];
                    while (x) {
                        const int e = 4 * wd + ((__ffs(x) - 1) >> 3);
                        x &= ~(0xffu << (8 * (e & 3)));
                        const int sl = atomicAdd(&S.lcnt[0], 1);
                        if (sl < LCAP) M.list[sl] = (uint16_t)e;
                    }
                }
            }
            __syncthreads();
            int cur = 0;
            bool overflow = S.lcnt[0] > LCAP;
            while (!overflow) {
                const int n = S.lcnt[cur];
                if (n == 0) break;
                if (tid == 0) ++S.tm[6];
                uint16_t* Lc = M.list + cur * LCAP;
                uint16_t* Ln = M.list + (cur ^ 1) * LCAP;
                for (int t = tid; t < n; t += NT) {
                    const int p = Lc[t];
                    EIK_CHECK(p >= 0 && p < R3, "list point index");
                    sA[p] = 0;                                               // Alg. 2 line 4
                    const T hs = M.hf(p);
                    const T hf = fabs(hs);
                    const int i = p % R, j = (p / R) % R, k = p / (R * R);
                    const int q = (i + 1) + RP * (j + 1) + RP2 * (k + 1);
                    const T v = sV[q];
                    const T xm = sV[q - 1], xp = sV[q + 1];
                    const T ym = sV[q - RP], yp = sV[q + RP];
                    const T zm = sV[q - RP2], zp = sV[q + RP2];
                    const T mx = vmin(habs<R>(xm), habs<R>(xp)), my = vmin(habs<R>(ym), habs<R>(yp)),
                            mz = vmin(habs<R>(zm), habs<R>(zp));   // (HaloNeg)
                    if (hf < INF && vmin(mx, vmin(my, mz)) < v) {
                        ++nupd;
                        const T u = local_solve_fast<T>(mx, my, mz, hf);      // line 5
                        if (u < v) {                                          // line 6
                            sV[q] = u;                                        // line 7
                            M.mark(p, hs);
                            ++nwr;
                            // lines 8-10: claim larger neighbours (CAS on the flag word) and
                            // append them to the next list
                            auto claim = [&](int nb) {
                                uint32_t* w = reinterpret_cast<uint32_t*>(sA + (nb & ~3));
                                const int sh = 8 * (nb & 3);
                                uint32_t old = *reinterpret_cast<volatile uint32_t*>(w);
                                while (!((old >> sh) & 0xffu)) {
                                    const uint32_t prev = atomicCAS(w, old, old | (1u << sh));
                                    if (prev == old) {
                                        const int sl = atomicAdd(&S.lcnt[cur ^ 1], 1);
                                        if (sl < LCAP) Ln[sl] = (uint16_t)nb;
                                        else S.lover = 1;
                                        break;
                                    }
                                    old = prev;
                                }
                            };
                            const T ut = (v - u > kap) ? u : INF;   // kappa: see sweep_dir
                            if (xm > ut && i > 0) claim(p - 1);
                            if (xp > ut && i < R - 1) claim(p + 1);
                            if (ym > ut && j > 0) claim(p - R);
                            if (yp > ut && j < R - 1) claim(p + R);
                            if (zm > ut && k > 0) claim(p - R * R);
                            if (zp > ut && k < R - 1) claim(p + R * R);
                        }
                    }
                }
                __syncthreads();
                overflow = S.lover != 0;
                if (tid == 0) S.lcnt[cur] = 0;
                cur ^= 1;
                __syncthreads();
            }
            if (tid == 0) S.tm[5] += (uint32_t)(clock64() - tl0);
            if (!overflow) break;          // converged in list mode
            nact = LCAP + 1;               // resume wavefront sweeps (flags authoritative)
        }
        // ========================= one wavefront sweep ==========================
        // sweep direction: the first sweep follows the inflow faces (preferred
        // directions); afterwards the axes along which the previous sweep activated points
        // behind its wavefront are reversed (information still has to travel that way);
        // without such activations the Gray cycle 0,1,3,2,6,7,5,4 is followed
        int dir;
        // EIK_DIR_VOTE: from the second sweep on, every active point votes per axis for the side
        // its smaller neighbour is on, if that neighbour is below the point's own value (the
        // information it was activated for comes from there); an axis with a majority sweeps
        // away from that side, a tied axis keeps the rule below
        int vote_m = 0, vote_d = 0;   // axes with a majority, and their direction bits
#if EIK_DIR_VOTE
        // (variant 2: only when the previous sweep left activations behind it along two or more
        // axes -- with one axis the rule below is unambiguous, and the vote costs a pass)
        const uint32_t bwp = sw > 0 ? S.bwd[(sw - 1) & 1] : 0u;
        if (prev_dir >= 0 && (EIK_DIR_VOTE == 1 || __popc(bwp & 7u) >= 2)) {
            int vx = 0, vy = 0, vz = 0;
            const uint32_t* sA32v = reinterpret_cast<const uint32_t*>(sA);
            for (int wd = tid; wd < R3 / 4; wd += NT) {
                uint32_t y = sA32v[wd] & 0x01010101u;
                while (y) {
                    const int i = (__ffs(y) - 1) >> 3;
                    y &= y - 1u;
                    const int e = 4 * wd + i;
                    const int a = e & (R - 1), b = (e / R) & (R - 1), d = e / (R * R);
                    const int q = (a + 1) + RP * (b + 1) + RP2 * (d + 1);
                    const T v = sV[q];
                    const T xm = habs<R>(sV[q - 1]), xp = habs<R>(sV[q + 1]);
                    const T ym = habs<R>(sV[q - RP]), yp = habs<R>(sV[q + RP]);
                    const T zm = habs<R>(sV[q - RP2]), zp = habs<R>(sV[q + RP2]);
                    if (vmin(xm, xp) < v) vx += xm < xp ? 1 : (xp < xm ? -1 : 0);
                    if (vmin(ym, yp) < v) vy += ym < yp ? 1 : (yp < ym ? -1 : 0);
                    if (vmin(zm, zp) < v) vz += zm < zp ? 1 : (zp < zm ? -1 : 0);
                }
            }
            // per warp: clamp to +-63 (six warps stay inside a biased 10-bit field), one atomic
            vx = (int)warp_add((uint32_t)vx); vy = (int)warp_add((uint32_t)vy); vz = (int)warp_add((uint32_t)vz);
            if ((tid & 31) == 0) {
                auto cl = [](int x) { return x > 63 ? 63 : (x < -63 ? -63 : x); };
                const int pk = cl(vx) + cl(vy) * 1024 + cl(vz) * 1048576;
                if (pk) atomicAdd(M.votes(), (uint32_t)pk);
            }
            __syncthreads();
            const uint32_t vw = *M.votes();
            const int sx = (int)(vw & 1023u) - 512, sy = (int)((vw >> 10) & 1023u) - 512, sz = (int)((vw >> 20) & 1023u) - 512;
            vote_m = (sx != 0 ? 1 : 0) | (sy != 0 ? 2 : 0) | (sz != 0 ? 4 : 0);
            vote_d = (sx < 0 ? 1 : 0) | (sy < 0 ? 2 : 0) | (sz < 0 ? 4 : 0);
        }
#endif
        {
            const uint32_t gray = 0x45762310u;
            const uint32_t bw = sw > 0 ? S.bwd[(sw - 1) & 1] : 0u;
            if (tid == 0) S.bwd[sw & 1] = 0;
            if (prev_dir < 0) {
                dir = dir0;
                if (!resumed && (init || !(flags & 63u))) gi = 1;
            } else if (bw) {
                // flip one of those axes per sweep, the least recently flipped one (a source
                // inside the cell needs all 8 octants: this then walks a Gray cycle)
                int ax = -1, best = 0x7fffffff;
                if ((bw & 1u) && lf0 < best) { ax = 0; best = lf0; }
                if ((bw & 2u) && lf1 < best) { ax = 1; best = lf1; }
                if ((bw & 4u) && lf2 < best) { ax = 2; best = lf2; }
                if (ax == 0) lf0 = sw; else if (ax == 1) lf1 = sw; else lf2 = sw;
                dir = prev_dir ^ (1 << ax);
            } else {
                dir = (gray >> (4 * gi)) & 15u;
                gi = (gi + 1) & 7;
                if (dir == prev_dir) { dir = (gray >> (4 * gi)) & 15u; gi = (gi + 1) & 7; }
            }
            if (vote_m) {
                // voted axes take the vote, the others what the rule above chose
                dir = (dir & ~vote_m) | (vote_d & vote_m);
                if ((dir ^ prev_dir) & 1) lf0 = sw;
                if ((dir ^ prev_dir) & 2) lf1 = sw;
                if ((dir ^ prev_dir) & 4) lf2 = sw;
            }
            prev_dir = dir;
        }
        const bool fx = dir & 1, fy = dir & 2, fz = dir & 4;
        const long long tm0 = tid == 0 ? clock64() : 0;
        // the set of planes (in this direction) holding active points, and their count (the
        // first sweep's was collected with the initial activity)
        const bool first = sw == 0 && !ran_list;
        const bool have0 = first && pm0_ok;   // the plane mask of this direction is in S.plane0
        if (!have0) {
            unsigned long long pm = 0;
            int cnt = 0;
            const uint32_t* sA32 = reinterpret_cast<const uint32_t*>(sA);
            // (every activity byte has bit 0 set: four flags of consecutive a per word fold into
            // four plane bits with one multiply -- ascending a, or descending when x is reflected)
            for (int wd = tid; wd < R3 / 4; wd += NT) {
                const uint32_t y = sA32[wd] & 0x01010101u;
                if (y) {
                    const int a0 = (4 * wd) & (R - 1), b = ((4 * wd) / R) & (R - 1), d = (4 * wd) / (R * R);
                    const int pbd = (fy ? R - 1 - b : b) + (fz ? R - 1 - d : d);
                    if (fx) pm |= (unsigned long long)((y * 0x08040201u) >> 24) << (R - 4 - a0 + pbd);
                    else pm |= (unsigned long long)((y * 0x01020408u) >> 24) << (a0 + pbd);
                    cnt += __popc(y);
                }
            }
            pm = warp_or64(pm);
            cnt = (int)warp_add((uint32_t)cnt);
            if ((tid & 31) == 0 && pm) { atomicOr(&S.plane[sw & 1], pm); atomicAdd(&S.nact2[sw & 1], cnt); }
            __syncthreads();
        }
        const unsigned long long pm = have0 ? S.plane0 : S.plane[sw & 1];
        nact = have0 ? S.nact : S.nact2[sw & 1];
        if (tid == 0) {
            S.plane[(sw + 1) & 1] = 0; S.nact2[(sw + 1) & 1] = 0;
            if (EIK_DIR_VOTE) *M.votes() = 512u | (512u << 10) | (512u << 20);   // (biased zeros; every thread has read the votes)
        }
        const long long tm1 = tid == 0 ? clock64() : 0;
        if (tid == 0) S.tm[4] += (uint32_t)(tm1 - tm0);
        if (pm == 0ull) break;
        if (nact <= LTHR && sw > 0) continue;   // few left: list mode (next iteration)
        if (A.max_sweeps > 0 && nsweeps >= (uint32_t)A.max_sweeps) {
            // sweep cap reached with points still active: save them and continue in a later
            // processing (the cell re-queues itself; correctness is unaffected, values only
            // decrease and every active point is eventually processed)
            uint32_t km = KEY_INF;
            for (int w = tid; w < NWB; w += NT) {
                uint32_t bits = 0;
                for (int l = 0; l < 32; ++l) {
                    const int e = 32 * w + l;
                    if (sA[e]) {
                        bits |= 1u << l;
                        const int a = e % R, b = (e / R) % R, d = e / (R * R);
                        km = min(km, key_bits(sV[(a + 1) + RP * (b + 1) + RP2 * (d + 1)]));
                    }
                }
                __stcg(&A.pend[(int64_t)c * NWB + w], bits);
            }
            for (int o = 16; o > 0; o >>= 1) km = min(km, __shfl_xor_sync(0xffffffffu, km, o));
            if ((tid & 31) == 0) atomicMin(&S.cont_key, km);
            if (tid == 0) {
                S.cont = 1;
                auto age = [&](int l) { return (uint32_t)(sw - l < 63 ? sw - l : 63); };
                S.dstate = (1u << 31) | (uint32_t)dir | ((uint32_t)gi << 3) | (age(lf0) << 9) |
                           (age(lf1) << 15) | (age(lf2) << 21);
            }
            break;
        }
        ++nsweeps;
        uint32_t bwd = 0;
        {
            const bool ungated = first && nact >= R3 / EIK_UNGATED_DIV;
            if constexpr (R < EIK_DIR_TEMPLATE_MIN_R) {
                bwd = sweep_dir<T, R, -1>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_, dir);
            } else if (R == 16 && EIK_SWEEP16 && kap == T(0)) {
                if constexpr (R == 16) bwd = sweep16r<T>(M, A.tab16, dir, pm, ungated, nupd, nwr, nsteps, ltid);
            } else switch (dir) {
            case 0: bwd = sweep_dir<T, R, 0>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            case 1: bwd = sweep_dir<T, R, 1>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            case 2: bwd = sweep_dir<T, R, 2>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            case 3: bwd = sweep_dir<T, R, 3>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            case 4: bwd = sweep_dir<T, R, 4>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            case 5: bwd = sweep_dir<T, R, 5>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            case 6: bwd = sweep_dir<T, R, 6>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            default: bwd = sweep_dir<T, R, 7>(S, M, A.plane_tab, pm, ungated, nupd, nwr, nsteps, kap, dmax_); break;
            }
        }
        if (tid == 0) S.tm[5] += (uint32_t)(clock64() - tm1);
        nact = LCAP + 1;   // unknown until the next scan
        bwd = warp_or(bwd);
        if ((tid & 31) == 0 && bwd) atomicOr(&S.bwd[sw & 1], bwd);
        __syncthreads();
    }
    if (tid == 0) S.tm[7] = (uint32_t)clock64();
    // ---- write back (16-byte vectors; a vector holding any changed point is stored whole,
    // unchanged values are rewritten identically).  Issued before the face summaries, which only
    // read shared memory, so the stores drain while they run (kappa > 0 needs the old values of
    // the global tile in the summaries and writes back after them) ----
    unsigned long long nw = 0;
    if (kap == T(0)) nw = write_back_changed<T, R>(Vt + base, M);
    // ---- face summaries (Eq. (3)): face f is currently downwind iff a border
    // point changed in this processing and ended below its outside neighbour (the staged
    // halo value, an upper bound of the current one: P:718 redundant tags are harmless); the
    // cell key candidate is the smallest such value (A_new of Eq. (3)).
    {
        uint32_t fm = KEY_INF, fx = 0u;
        int f_prev = -1;
        for (int e = tid; e < 6 * R * R; e += NT) {
            const int f = e / (R * R), uv = e - f * R * R, u = uv % R, v = uv / R;
            int a, b, d, ha, hb, hd;
            switch (f) {
            case 0: a = 0; b = u; d = v; ha = -1; hb = b; hd = d; break;
            case 1: a = R - 1; b = u; d = v; ha = R; hb = b; hd = d; break;
            case 2: a = u; b = 0; d = v; ha = a; hb = -1; hd = d; break;
            case 3: a = u; b = R - 1; d = v; ha = a; hb = R; hd = d; break;
            case 4: a = u; b = v; d = 0; ha = a; hb = b; hd = -1; break;
            default: a = u; b = v; d = R - 1; ha = a; hb = b; hd = R; break;
            }
            if (f != f_prev) {
                if (f_prev >= 0 && fm != KEY_INF) {
                    atomicMin(&S.face_min[f_prev], fm);
                    atomicOr(&S.face_flag, 1u << f_prev);
                    if (A.legacy_key) atomicMax(&S.face_max[f_prev], fx);
                }
                fm = KEY_INF;
                fx = 0u;
                f_prev = f;
            }
            const int pp = a + R * b + R * R * d;
            if (M.changed(pp)) {
                const T val = sV[(a + 1) + RP * (b + 1) + RP2 * (d + 1)];
                const T out = habs<R>(sV[(ha + 1) + RP * (hb + 1) + RP2 * (hd + 1)]);   // (HaloNeg)
                // kappa: a border change <= kappa tags no neighbour cell (the tile in
                // global memory still holds the value staged at the start of the processing)
                const bool sig = kap == T(0) || __ldcg(&Vt[base + pp]) - val > kap;
                if (val < out && sig) {
                    fm = min(fm, key_bits(val));
                    fx = max(fx, key_bits(val));
                }
            }
        }
        if (f_prev >= 0 && fm != KEY_INF) {
            atomicMin(&S.face_min[f_prev], fm);
            atomicOr(&S.face_flag, 1u << f_prev);
            if (A.legacy_key) atomicMax(&S.face_max[f_prev], fx);
        }
    }
    __syncthreads();

    if (kap != T(0)) nw = write_back_changed<T, R>(Vt + base, M);
    if (A.stats) {
        // (per-thread counts of one processing are far below 2^32 / 32)
        const unsigned long long u64 = warp_add(nupd), w64 = warp_add(nwr);
        nw = warp_add((uint32_t)nw);
        if ((tid & 31) == 0) {
            atomicAdd(&S.stat[0], u64);
            atomicAdd(&S.stat[1], w64);
            atomicAdd(&S.stat[2], nw);
        }
    }
    n_sweeps_out = nsweeps;
    if (tid == 0 && A.stats) {
        atomicAdd(&A.ctl->dbg[36], (unsigned long long)(uint32_t)(S.tm[3] - S.tm[0]));
        atomicAdd(&A.ctl->dbg[41], (unsigned long long)(uint32_t)(S.tm[1] - S.tm[0]));
        atomicAdd(&A.ctl->dbg[42], (unsigned long long)(uint32_t)(S.tm[2] - S.tm[1]));
        atomicAdd(&A.ctl->dbg[37], (unsigned long long)S.tm[4]);
        atomicAdd(&A.ctl->dbg[38], (unsigned long long)S.tm[5]);
        atomicAdd(&A.ctl->dbg[39], (unsigned long long)(uint32_t)((uint32_t)clock64() - S.tm[7]));
        atomicAdd(&A.ctl->dbg[2], (unsigned long long)nsteps);
        S.nsteps = nsteps;
        atomicAdd(&A.ctl->dbg[40], (unsigned long long)S.tm[6]);
    }
}

// Cell value a tag from face f proposes for the neighbour cell nc (Alg. 1 line 9):
//   Eq. (3) (default): the smallest newly updated inflow value of the face;
//   Eq. (4) (legacy): V_max + D / F(y), V_max the largest newly updated inflow
//   value, D = (h^c + h) / 2 the distance from the face's gridpoints to the centre of nc and
//   F(y) the speed there (the gridpoint (r/2, r/2, r/2) of nc): D / F(y) = (r + 1) / 2 * hf.
template <typename T, int R>
__device__ __forceinline__ uint32_t tag_key(const CellArgs& A, const CellShared<R>& S, int f, int64_t nc)
{
    if (!A.legacy_key) return S.face_min[f];
    const T hfc = __ldcg(reinterpret_cast<const T*>(A.Ht) + nc * (int64_t)(R * R * R) +
                         (R / 2) * (1 + R + R * R));
    const float v = __uint_as_float(S.face_max[f]) + (float)(T(0.5 * (R + 1)) * hfc);
    return key_bits(v);
}

// neighbour cell across face f of c, or -1 outside the grid
__device__ __forceinline__ int64_t face_neighbour(uint32_t c, int f, int cps)
{
    const int cx = (int)(c % (uint32_t)cps), cy = (int)((c / (uint32_t)cps) % (uint32_t)cps),
              cz = (int)(c / ((uint32_t)cps * (uint32_t)cps));
    switch (f) {
    case 0: return cx > 0 ? (int64_t)c - 1 : -1;
    case 1: return cx < cps - 1 ? (int64_t)c + 1 : -1;
    case 2: return cy > 0 ? (int64_t)c - cps : -1;
    case 3: return cy < cps - 1 ? (int64_t)c + cps : -1;
    case 4: return cz > 0 ? (int64_t)c - (int64_t)cps * cps : -1;
    default: return cz < cps - 1 ? (int64_t)c + (int64_t)cps * cps : -1;
    }
}

template <int R>
__device__ __forceinline__ void cell_stats_v(const CellArgs& A, unsigned long long st0, unsigned long long st1,
                                             unsigned long long st2, uint32_t c, unsigned long long nsweeps);
template <int R>
__device__ __forceinline__ void cell_stats(const CellArgs& A, CellShared<R>& S, uint32_t c,
                                           unsigned long long nsweeps)
{
    cell_stats_v<R>(A, S.stat[0], S.stat[1], S.stat[2], c, nsweeps);
}
template <int R>
__device__ __forceinline__ void cell_stats_v(const CellArgs& A, unsigned long long st0, unsigned long long st1,
                                             unsigned long long st2, uint32_t c, unsigned long long nsweeps)
{
    Ctl* ctl = A.ctl;
    const int cps = A.cps;
    const int64_t n1 = A.n1;
    const int cx = (int)(c % (uint32_t)cps), cy = (int)((c / (uint32_t)cps) % (uint32_t)cps),
              cz = (int)(c / ((uint32_t)cps * (uint32_t)cps));
    atomicAdd(&ctl->updates, st0);
    atomicAdd(&ctl->writes, st1);
    atomicAdd(&ctl->bytes_written, st2);
    atomicAdd(&ctl->sweeps, nsweeps);
    const int64_t rx = (n1 - (int64_t)cx * R) < R ? (n1 - (int64_t)cx * R) : R;
    const int64_t ry = (n1 - (int64_t)cy * R) < R ? (n1 - (int64_t)cy * R) : R;
    const int64_t rz = (n1 - (int64_t)cz * R) < R ? (n1 - (int64_t)cz * R) : R;
    atomicAdd(&ctl->real_pts, (unsigned long long)(rx * ry * rz));
    atomicAdd(&ctl->dbg[4 + (nsweeps < 31 ? nsweeps : 31)], 1ull);
}

// ---- round mode: one CTA per cell of this round's list (grid-stride) ------------------
template <typename T, int R>
__global__ void __launch_bounds__(CellCfg<R>::NT, MinBlocks<T, R>::value)
k_cell(CellArgs A)
{
    using C = CellCfg<R>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CellSmem<T, R> Msm(smem_raw);
    __shared__ CellShared<R> S;
    const int tid = threadIdx.x;
    Ctl* ctl = A.ctl;
    // graph body with several rounds: the rounds after the last one are no-ops
    if (A.graph && ctl->done) return;
    const uint32_t cur = ctl->cur, nx = cur ^ 1u;
    // fused: this round's cells are the whole current worklist (Alg. 1 lines 4-5 with an
    // infinite bin); otherwise k_select built the proc list
    const uint32_t nproc = A.fused ? ctl->wl_count[cur] : ctl->proc_count;
    const uint32_t* wl = cur ? A.wl1 : A.wl0;
    uint32_t* wn = nx ? A.wl1 : A.wl0;
    // Fused rounds keep the state bits of the two rounds apart (byte 0 / byte 2 by round
    // parity): a cell takes this round's bits when claimed, and a tag during the round always
    // goes to the next round's byte -- as with k_select, which takes every selected cell's
    // bits before the round starts.  (Merging a tag into a not-yet-claimed cell of this round
    // instead lets it run with faces that are only partly final: measured 13-25 % more
    // processings on the paper's r = 8 suite.)
    const uint32_t sh_cur = (A.fused && EIK_PARITY) ? 16u * (ctl->rounds & 1u) : 0u;
    const uint32_t sh_nx = (A.fused && EIK_PARITY) ? 16u - sh_cur : 0u;
    // dynamic claiming of this round's cells (processing times vary by >10x between cells)
    bool worked = false;
    for (;;) {
        if (tid == 0) {
            const uint32_t w = atomicAdd(&ctl->claim, 1u);
            uint32_t cc = 0xffffffffu, fl = 0;
            if (w < nproc) {
                if (A.fused) {
                    // LIFO: the cells appended last (re-activated by the previous round's
                    // slowest processings: the critical path) are claimed first
                    const uint32_t wi = EIK_LIFO ? nproc - 1u - w : w;
                    cc = wl[wi];
                    // take this round's inflow bits; the cell leaves the list
                    fl = (atomicAnd(&A.state[cc], ~(0xffu << sh_cur)) >> sh_cur) & 0xffu;
                    if (!A.legacy_key) A.key[cc] = KEY_INF;   // V^c <- +inf on removal
                    atomicAdd(&ctl->proc_count, 1u);
                } else {
                    cc = A.proc_cell[w];
                    fl = A.proc_flags[w];
                }
            }
            S.cell = cc;
            S.flags = fl;
        }
        __syncthreads();
        const uint32_t c = S.cell;
        if (c == 0xffffffffu) break;
        if (!worked && tid == 0) atomicMin(&ctl->t_start, gtimer());
        worked = true;
        const long long t0 = clock64();
        EIK_CHECK(c < A.cap, "round cell id");
        const uint32_t flags = S.flags;
        if (tid == 0) S.stat[0] = S.stat[1] = S.stat[2] = 0;
        unsigned long long nsw = 0;
        cell_process<T, R, true>(A, S, Msm, c, flags, nsw);
        __syncthreads();
        // re-activate currently-downwind neighbour cells (Alg. 1 lines 7-10)
        if (S.cont && tid == 7) __stcg(&A.pdir[c], S.dstate);   // read in a later round
        if (tid < 6 && (S.face_flag & (1u << tid))) {
            const int64_t nc = face_neighbour(c, tid, A.cps);
            if (nc >= 0) {
                const uint32_t kb = tag_key<T, R>(A, S, tid, nc);
                atomicMin(&A.key[nc], kb);                                     // Eq. (3) / (4)
                const uint32_t old = atomicOr(&A.state[nc], (1u << (tid ^ 1)) << sh_nx);  // face of nc
                if (((old >> sh_nx) & 0xffu) == 0u) {                                   // Alg. 5
                    const uint32_t sl = atomicAdd(&ctl->wl_count[nx], 1u);
                    wn[sl] = (uint32_t)nc;
                }
                atomicMin(&ctl->kmin[nx], kb);
            }
        }
        if (tid == 0 && S.cont) {   // continue this cell in a later round
            atomicMin(&A.key[c], S.cont_key);
            const uint32_t old = atomicOr(&A.state[c], FLAG_CONT << sh_nx);
            if (((old >> sh_nx) & 0xffu) == 0u) {
                const uint32_t sl = atomicAdd(&ctl->wl_count[nx], 1u);
                wn[sl] = c;
            }
            atomicMin(&ctl->kmin[nx], S.cont_key);
        }
        if (tid == 0 && A.stats) {
            cell_stats<R>(A, S, c, nsw);
            const unsigned long long cyc = (unsigned long long)(clock64() - t0);
            atomicAdd(&ctl->dbg[0], cyc);
            atomicMax(&ctl->dbg[1], cyc);
            atomicAdd(&ctl->dbg[3], 1ull);
            atomicAdd(&ctl->rsum, cyc);
            atomicMax(&ctl->rmax, cyc);
            for (int l = 0; l < 2; ++l) {
                if (l == 1 && cyc <= 100000ull) break;
                atomicAdd(&ctl->lstat[l][0], 1ull);
                atomicAdd(&ctl->lstat[l][1], cyc);
                atomicAdd(&ctl->lstat[l][2], nsw);
                atomicAdd(&ctl->lstat[l][3], (unsigned long long)S.tm[6]);
                atomicAdd(&ctl->lstat[l][4], (unsigned long long)S.nsteps);
                atomicAdd(&ctl->lstat[l][5], (flags & FLAG_CONT) ? 1ull : 0ull);
            }
        }
        __syncthreads();   // smem reuse by the next cell of this CTA
    }
    if (worked && tid == 0) atomicMax(&ctl->t_end, gtimer());
    // fused round end: the last CTA to finish swaps the worklists and decides whether the
    // loop continues (Alg. 3 line 6); every CTA's appends are ordered before its count
    if (A.fused && tid == 0) {
        __threadfence();
        if (atomicAdd(&ctl->cta_done, 1u) == gridDim.x - 1u) {
            __threadfence();
            const bool stop = round_end_body(ctl);
            if (A.graph) cudaGraphSetConditional((cudaGraphConditionalHandle)A.cond, stop ? 0u : 1u);
        }
    }
}

// ---- async mode: persistent CTAs pull cells from a device FIFO (pHCM Alg. 3 analogue) ---
//
// Cell state word: bits 0-5 inflow faces, bit 6 INIT, QUEUED, RUNNING.  A cell is in the
// ring at most once: it is pushed only on the transition to QUEUED while not RUNNING, or by
// its own CTA when it finishes and finds QUEUED set (it was tagged while running).
// ctl->pending = cells queued or running; the solve ends when it reaches 0 (the analogue
// of activeCellCount, Alg. 3 lines 6 and 29).  Value stores are ordered before the tags by
// __threadfence (the flush of P:686-688); readers take the cell with an atomic and read
// tiles through L2 (.cg), so a stale read is only ever a valid upper bound and
// is followed by a re-activation.
enum : uint32_t { ST_QUEUED = 256u, ST_RUNNING = 512u, ST_VISITED = 1024u, Q_EMPTY = 0xffffffffu };
#ifndef EIK_AUTO_RATIO
#define EIK_AUTO_RATIO 6ull   // readiness mode 8: switch to the key order above this processings / cell (measured: 4 slows P2 / P3 / C2d, 6 does not; PMAZE 84 -> 49 ms)
#endif

__device__ __forceinline__ void q_push(Ctl* ctl, uint32_t* ring, uint32_t qmask, uint32_t c)
{
    atomicAdd(&ctl->pending, 1u);
    const uint32_t slot = atomicAdd(&ctl->q_tail, 1u) & qmask;
    while (atomicCAS(&ring[slot], Q_EMPTY, c) != Q_EMPTY) __nanosleep(32);
}

// re-queue a cell that is already counted in pending (a deferral, or a parked cell)
__device__ __forceinline__ void q_repush(Ctl* ctl, uint32_t* ring, uint32_t qmask, uint32_t c)
{
    const uint32_t slot = atomicAdd(&ctl->q_tail, 1u) & qmask;
    while (atomicCAS(&ring[slot], Q_EMPTY, c) != Q_EMPTY) __nanosleep(32);
}

#ifndef EIK_PARK
#define EIK_PARK 0   // 1: a cell deferred by a running neighbour waits on it instead of cycling the ring (measured: C3 7.17 -> 7.57 ms, C5 35.7 -> 36.4; off)
#endif

}  // namespace eik
#include "eik_b2.cuh"
namespace eik {

// cell kernel of the async scheduler: MODE 0 = cell_process (point wavefront), MODE 1 = the
// 2x2x2 micro-block form (r = 16 only, eik_b2.cuh)
template <typename T, int R, int MODE> struct AsyncCfg {
    static constexpr int NT = CellCfg<R>::NT;
    static constexpr int MINB = MinBlocks<T, R>::value;
};
template <typename T> struct AsyncCfg<T, 16, 1> {
    static constexpr int NT = B2::NT;
    static constexpr int MINB = B2Minb<T>::value;
};

template <typename T, int R, int MODE = 0>
__global__ void __launch_bounds__((AsyncCfg<T, R, MODE>::NT), (AsyncCfg<T, R, MODE>::MINB))
k_async(CellArgs A)
{
    constexpr int NTH = AsyncCfg<T, R, MODE>::NT;
    // TAG1: warp 1 re-activates the neighbours and releases the cell while warp 0 is already
    // popping the next one (CTAs of at least two warps)
    constexpr bool TAG1 = NTH >= 64 && EIK_TAG_WARP1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ CellShared<R> S;
    const int tid = threadIdx.x;
    Ctl* ctl = A.ctl;
    uint32_t* ring = A.wl0;
    if (TAG1 && tid == 0) S.stat[0] = S.stat[1] = S.stat[2] = 0;
    uint32_t hpar = 0;   // phase of the hf bulk-copy mbarrier = cells this CTA has staged (EIK_HF_BULK)
    if constexpr (MODE == 0 && CellSmem<T, R>::BULK) {
        if (tid == 0) mbar_init(CellSmem<T, R>(smem_raw).mbar());
        __syncthreads();
    }
    if (tid == 0) atomicMin(&ctl->t_start, gtimer());
    // Warp balance across the SM's four schedulers (r = 16): the plane table fills its columns
    // from 0 up, so the warp of columns 0-31 works in all 46 plane steps of a sweep, the next in
    // 32, then 26, 20, 16 and 10.  With the identity mapping every CTA's busiest warps (0 and 4,
    // 62 of the 150 warp-steps) sit on scheduler 0 (warp w issues on scheduler w mod 4).  The
    // columns are therefore permuted per CTA: the two busiest logical warps go alone on the
    // single-warp schedulers (2, 3), the others pair up as 26 + 10 and 20 + 16, and CTAs of even
    // / odd rank on their SM mirror the assignment.
    uint32_t ltid = (uint32_t)tid;
#if EIK_WARP_BALANCE
    if constexpr (R == 16 && NTH == 192) {
        if (tid == 0) {   // (S.cell as the broadcast word: five CTAs per SM leave no spare shared memory)
            uint32_t smid;
            asm("mov.u32 %0, %%smid;" : "=r"(smid));
            S.cell = atomicAdd(&ctl->sm_rank[smid & 255u], 1u);
        }
        __syncthreads();
        // hardware warp -> logical warp (table columns): even rank {2,3,0,1,5,4}, odd {3,2,1,0,4,5}
        const uint32_t pe = 0x451032u, po = 0x540123u;
#if EIK_WARP_BALANCE == 2
        const uint32_t lw = ((uint32_t)(tid >> 5) + S.cell) % 6u; (void)pe; (void)po;
#elif EIK_WARP_BALANCE == 3
        const uint32_t lw = (pe >> (4 * (tid >> 5))) & 15u; (void)po;
#else
        const uint32_t lw = (((S.cell & 1u) ? po : pe) >> (4 * (tid >> 5))) & 15u;
#endif
        ltid = lw * 32u + ((uint32_t)tid & 31u);
        __syncthreads();   // S.cell is rewritten by the first pop
    }
#endif
    uint32_t tr_pid = 0, tr_tag = 0, tr_pop = 0, tr_swept = 0;   // processing trace (thread 0)
    uint32_t gen_c = 0;                                          // generation of the cell (thread 0)
    uint32_t ost = 0;                                            // state word the claim replaced (thread 0)
    for (;;) {
        if (tid < 32) {   // warp 0 pops the next cell; the other warps wait at the barrier
            const int lane = tid;
            uint32_t got = Q_EMPTY;
            for (;;) {
                // lane 0: ticket pop -- every CTA takes the next head index with one atomicAdd
                // (no CAS retry loop, which serialises 700+ CTAs to one claim per L2 round
                // trip) and waits until the push of the same index has filled the slot, or the
                // solve is over (pending = 0: no push will come)
                uint32_t v = Q_EMPTY;
                int quit = 0;
                if (lane == 0) {
                    // (no pending / abort check before the ticket: the wait below makes it, and a
                    // ticket taken after the end of the solve is harmless -- one round trip less)
                    {
                        const uint32_t h = atomicAdd(&ctl->q_head, 1u);
                        unsigned ns = 32;
                        while ((v = atomicExch(&ring[h & A.qmask], Q_EMPTY)) == Q_EMPTY) {
                            if (__ldcg(&ctl->pending) == 0u || __ldcg(&ctl->abort) != 0u) { quit = 1; break; }
                            if (gtimer() - __ldcg(&ctl->t_solve0) > __ldcg(&ctl->budget_ns)) {   // watchdog
                                atomicOr(&ctl->err, 8u);
                                atomicExch(&ctl->abort, 1u);
                                quit = 1;
                                break;
                            }
                            __nanosleep(ns);
                            ns = ns < EIK_POP_MAXNS ? ns * 2 : EIK_POP_MAXNS;
                        }
                    }
                }
                quit = __shfl_sync(0xffffffffu, quit, 0);
                if (quit) break;
                v = __shfl_sync(0xffffffffu, v, 0);
                EIK_CHECK(v < A.cap, "ring cell id");
                // readiness (the heap order of Alg. 3 approximated locally): lane f checks the
                // neighbour across face f -- all loads of the six checks in one round trip --
                // and v is re-queued while a neighbour runs or is queued ahead of it
                bool d = false, drun = false;
                int64_t nb = -1;
                uint32_t gv0 = 0;   // generation of v (lanes < 6, when a readiness mode is on)
                // mode 8 (automatic): mode 6 until the solve has run more than EIK_AUTO_RATIO
                // processings per processed cell, then mode 2 for the rest (see release below)
                const int dm = A.defer == 8 ? (int)__ldcg(&ctl->auto_mode) : A.defer;
                if (dm && lane < 6) {
                    nb = face_neighbour(v, lane, A.cps);
                    const uint32_t kv = __ldcg(&A.key[v]), sv = __ldcg(&A.state[v]), gv = __ldcg(&A.gen[v]);
                    gv0 = gv;
                    uint32_t sn = 0, kn = KEY_INF, gn = 0;
                    if (nb >= 0) { sn = __ldcg(&A.state[nb]); kn = __ldcg(&A.key[nb]); gn = __ldcg(&A.gen[nb]); }
                    // mode 4: only neighbours across an inflow face of v matter
                    if (nb >= 0 && !(dm == 4 && !(sv & (1u << lane)))) {
                        if (sn & ST_RUNNING) d = drun = true;
                        else if (sn & ST_QUEUED) {
                            if (dm == 5) d = gn < gv;
                            else if (dm == 2) d = kn < kv || (kn == kv && (uint32_t)nb < v);
                            else if (dm == 3) d = __uint_as_float(kn) + A.defer_delta < __uint_as_float(kv);
                            else if (dm == 6 || dm == 9)   // strict total order (no deferral cycles); mode 9: gen = level
                                d = gn < gv || (gn == gv && (kn < kv || (kn == kv && (uint32_t)nb < v)));
                            else if (dm == 7)
                                d = kn < kv || (kn == kv && (gn < gv || (gn == gv && (uint32_t)nb < v)));
                        }
                    }
                }
                if (__any_sync(0xffffffffu, d)) {
                    // Deferred.  Blocked by a RUNNING neighbour: park on it -- set v's bit in the
                    // neighbour's waiter word; its release re-queues v (no cycling through the
                    // ring: a re-push goes behind every other deferred cell, and the critical
                    // path waited a whole ring cycle per cell diagonal, ~30 us on C3).  Whoever
                    // clears the bit pushes v, so v is queued exactly once: if the neighbour
                    // stopped running before v's bit was set, v takes the bit back and re-pushes
                    // itself (Dekker order: bit set, fence, state read / state cleared, fence,
                    // waiter word taken).  Running cells never wait, so parking cannot deadlock.
                    const unsigned rb = EIK_PARK ? __ballot_sync(0xffffffffu, drun) : 0u;
                    const int fp = rb ? __ffs(rb) - 1 : 0;
                    const int64_t nbp = __shfl_sync(0xffffffffu, nb, fp);
                    if (lane == 0) {
                        bool parked = false;
                        if (rb) {
                            const uint32_t bit = 1u << (fp ^ 1);   // face of nbp toward v
                            atomicOr(&A.wait[nbp], bit);
                            __threadfence();
                            if (__ldcg(&A.state[nbp]) & ST_RUNNING) parked = true;
                            else parked = !(atomicAnd(&A.wait[nbp], ~bit) & bit);   // the releaser took it
                        }
                        if (!parked) q_repush(ctl, ring, A.qmask, v);
                        atomicAdd(&ctl->defers, 1ull);
                        if (!parked) __nanosleep(64);
                    }
                    __syncwarp();
                    continue;
                }
                got = v;
                if (lane == 0) gen_c = dm ? gv0 : (A.defer >= 5 ? __ldcg(&A.gen[v]) : 0u);   // (broadcast at the tags)
                break;
            }
            if (lane == 0) {
                if (got != Q_EMPTY) {
                    // the claim: its result (inflow faces + INIT + CONT) is first needed after the
                    // staging loads have been issued, so its round trip overlaps theirs
                    ost = atomicExch(&A.state[got], ST_RUNNING | ST_VISITED);
                    if (!A.legacy_key) A.key[got] = KEY_INF;             // V^c <- +inf
                    // (no fence: the tile loads depend on `got`, which was read from the ring
                    // after its producer fenced the cell's values, and go to L2)
                }
                S.cell = got;
                if constexpr (!TAG1) S.stat[0] = S.stat[1] = S.stat[2] = 0;   // (TAG1: thread 32 resets them)
                if (A.trace && got != Q_EMPTY) {   // (thread 0's registers)
                    tr_pid = atomicAdd(&ctl->trace_n, 1u);
                    tr_tag = __ldcg(&A.tagger[got]);
                    tr_pop = (uint32_t)(gtimer() - __ldcg(&ctl->t_solve0));
                }
            }
        }
        __syncthreads();
        const uint32_t c = S.cell;
        if (c == Q_EMPTY) break;
        const long long t0 = clock64();
        unsigned long long nsw = 0;
        if constexpr (MODE == 1 && R == 16) {
            B2Smem<T> Mb(smem_raw);
            if (tid == 0) S.flags = ost & 255u;
            __syncthreads();
            cell_process_b2<T>(A, S, Mb, c, S.flags, nsw);
        } else {
            CellSmem<T, R> Msm(smem_raw);
            cell_process<T, R, false>(A, S, Msm, c, ost & 255u, nsw, ltid, hpar);   // (thread 0's claim -> S.flags)
            ++hpar;
        }
        if (tid == 0 && !(ost & ST_VISITED)) atomicAdd(&ctl->first_procs, 1u);
        if (A.trace && tid == 0) tr_swept = (uint32_t)(gtimer() - __ldcg(&ctl->t_solve0));
        if (!TAG1 && tid < 32) {
            tr_pid = __shfl_sync(0xffffffffu, tr_pid, 0);
            gen_c = __shfl_sync(0xffffffffu, gen_c, 0);
        }
        // TAG1: thread 0 hands what it holds in registers to warp 1 through S.plane / S.plane0
        // (free once the sweeps are over; five CTAs per SM leave no spare shared memory)
        uint32_t* hand = reinterpret_cast<uint32_t*>(&S.plane[0]);
        if (TAG1 && tid == 0) {
            hand[0] = gen_c; hand[1] = tr_pid; hand[2] = tr_tag; hand[3] = tr_pop;
            reinterpret_cast<uint32_t*>(&S.plane0)[0] = tr_swept;
        }
        __threadfence();   // value stores before the re-activations
        if constexpr (!TAG1) __syncthreads();
        // Re-activations first, then the cell's own release: a neighbour waiting for this cell
        // to stop running must find its tag already set (releasing first let it run without
        // the tag and then again with it: 50 % more processings on C4).  Warp 0 tags and then
        // pops the next cell while thread 32 releases this one (its atomics overlap the pop):
        // named barrier 1 = thread 32 has copied this processing's shared results, barrier 2 =
        // the tags are out.
        // the release of this cell by one thread (counters by value: S may be overwritten)
        auto release = [&](uint32_t cont, uint32_t dstate, uint32_t cont_key, unsigned long long st0,
                           unsigned long long st1, unsigned long long st2) {
            if (cont) {   // sweep cap: save the direction state, continue later
                __stcg(&A.pdir[c], dstate);
                __threadfence();   // before the cell is re-queued below
                atomicMin(&A.key[c], cont_key);
                atomicOr(&A.state[c], FLAG_CONT | ST_QUEUED);
            }
            const uint32_t old = atomicAnd(&A.state[c], ~ST_RUNNING);
            if (old & ST_QUEUED) q_push(ctl, ring, A.qmask, c);   // tagged while running
            if (EIK_PARK) {
                // re-queue the neighbours parked on this cell (they stay counted in pending)
                __threadfence();
                uint32_t w = atomicExch(&A.wait[c], 0u);
                while (w) {
                    const int f = __ffs(w) - 1;
                    w &= w - 1u;
                    const int64_t nbw = face_neighbour(c, f, A.cps);
                    EIK_CHECK(nbw >= 0 && nbw < (int64_t)A.cap, "parked neighbour");
                    q_repush(ctl, ring, A.qmask, (uint32_t)nbw);
                }
            }
            const unsigned long long np = atomicAdd(&ctl->processings, 1ull) + 1ull;
            if (np > A.proc_limit) atomicExch(&ctl->abort, 1u);
            // automatic readiness (mode 8): the generation order keeps the front wide but re-runs
            // cells whose true upwind neighbour arrives later through faster regions; once
            // processings exceed EIK_AUTO_RATIO per processed cell (slow barriers, pinched level
            // sets: P:1644-1648), the rest of the solve takes the key (heap) order of Alg. 3
            if (A.defer == 8 && np > EIK_AUTO_RATIO * (unsigned long long)__ldcg(&ctl->first_procs) + 4096ull &&
                __ldcg(&ctl->auto_mode) != 2u)
                atomicExch(&ctl->auto_mode, 2u);
            if (A.stats) {
                cell_stats_v<R>(A, st0, st1, st2, c, nsw);
                const unsigned long long cyc = (unsigned long long)(clock64() - t0);
                atomicAdd(&ctl->dbg[0], cyc);
                atomicMax(&ctl->dbg[1], cyc);
                atomicAdd(&ctl->dbg[3], 1ull);
            }
            __threadfence();
            atomicSub(&ctl->pending, 1u);
        };
        if constexpr (TAG1) {
            // Every thread has fenced its write-back.  Warp 0 only arrives at the barrier that
            // orders the tags behind those fences and goes on to pop the next cell; warp 1 waits
            // for it, tags (lanes 0-5) and releases (its lane 0); warps 2+ wait at the loop top.
            if (tid < 32) {
                asm volatile("bar.arrive 3, %0;" :: "n"(NTH) : "memory");
            } else {
                asm volatile("bar.sync 3, %0;" :: "n"(NTH) : "memory");
                if (tid < 64) {
                    const int l = tid - 32;
                    const uint32_t cont = S.cont, dstate = S.dstate, cont_key = S.cont_key;
                    const unsigned long long st0 = S.stat[0], st1 = S.stat[1], st2 = S.stat[2];
                    const uint32_t gen_w = hand[0], pid_w = hand[1];
                    __syncwarp();
                    if (l == 0) S.stat[0] = S.stat[1] = S.stat[2] = 0;   // for the next processing
                    if (l < 6 && (S.face_flag & (1u << l))) {
                        const int64_t nc = face_neighbour(c, l, A.cps);
                        if (nc >= 0) {
                            atomicMin(&A.key[nc], tag_key<T, R>(A, S, l, nc));          // Eq. (3) / (4)
                            if (A.defer == 9) atomicMin(&A.gen[nc], gen_w + 1u);   // (mode 9: the smallest level)
                            else if (A.defer >= 5) atomicMax(&A.gen[nc], gen_w + 1u);
                            if (A.trace) A.tagger[nc] = pid_w;
                            const uint32_t old = atomicOr(&A.state[nc], (1u << (l ^ 1)) | ST_QUEUED);
                            if (!(old & (ST_QUEUED | ST_RUNNING))) {
                                q_push(ctl, ring, A.qmask, (uint32_t)nc);
                                __threadfence();   // the push's pending increment before this cell's decrement
                            }
                        }
                    }
                    __syncwarp();
                    if (l == 0) {
                        if (A.trace && pid_w < A.trace_cap) {
                            const uint32_t te = (uint32_t)(gtimer() - __ldcg(&ctl->t_solve0));
                            A.trace[2 * pid_w] = make_uint4(c, hand[2], hand[3], reinterpret_cast<uint32_t*>(&S.plane0)[0]);
                            A.trace[2 * pid_w + 1] = make_uint4(te, (uint32_t)nsw, S.flags, (uint32_t)st1);
                        }
                        release(cont, dstate, cont_key, st0, st1, st2);
                    }
                }
            }
        } else if (tid < 32) {
            if (tid < 6 && (S.face_flag & (1u << tid))) {
                const int64_t nc = face_neighbour(c, tid, A.cps);
                if (nc >= 0) {
                    atomicMin(&A.key[nc], tag_key<T, R>(A, S, tid, nc));          // Eq. (3) / (4)
                    if (A.defer == 9) atomicMin(&A.gen[nc], gen_c + 1u);   // (mode 9: the smallest level)
                    else if (A.defer >= 5) atomicMax(&A.gen[nc], gen_c + 1u);
                    if (A.trace) A.tagger[nc] = tr_pid;
                    const uint32_t old = atomicOr(&A.state[nc], (1u << (tid ^ 1)) | ST_QUEUED);
                    if (!(old & (ST_QUEUED | ST_RUNNING))) {
                        q_push(ctl, ring, A.qmask, (uint32_t)nc);
                        __threadfence();   // the push's pending increment before this cell's decrement
                    }
                }
            }
            __syncwarp();
            if constexpr (NTH >= 64) asm volatile("bar.arrive 2, 64;" ::: "memory");
            if (tid == 0 && A.trace && tr_pid < A.trace_cap) {
                const uint32_t te = (uint32_t)(gtimer() - __ldcg(&ctl->t_solve0));
                A.trace[2 * tr_pid] = make_uint4(c, tr_tag, tr_pop, tr_swept);
                A.trace[2 * tr_pid + 1] = make_uint4(te, (uint32_t)nsw, S.flags, (uint32_t)S.stat[1]);
            }
            if constexpr (NTH >= 64) asm volatile("bar.sync 1, 64;" ::: "memory");   // S may be overwritten now
            else if (tid == 0) release(S.cont, S.dstate, S.cont_key, S.stat[0], S.stat[1], S.stat[2]);
        } else if (NTH >= 64 && tid < 64) {
            // this processing's shared results, before warp 0's pop overwrites them
            const uint32_t cont = S.cont, dstate = S.dstate, cont_key = S.cont_key;
            const unsigned long long st0 = S.stat[0], st1 = S.stat[1], st2 = S.stat[2];
            asm volatile("bar.arrive 1, 64;" ::: "memory");
            asm volatile("bar.sync 2, 64;" ::: "memory");   // tags out
            if (tid == 32) release(cont, dstate, cont_key, st0, st1, st2);
        }
    }
    if (tid == 0) atomicMax(&ctl->t_end, gtimer());
}

// a change as a float rounded up (non-negative: its bits order like the values)
__device__ __forceinline__ float dmax_up(float x) { return x; }
__device__ __forceinline__ float dmax_up(double x) { return __double2float_ru(x); }

// --------------------------------------------------------------------------------------
// Whole-grid sweeping: the paper's comparison methods on the same tiles.
// FSM relaxes every gridpoint once per sweep in one of the 2^3 loop orderings;
// Detrixhe's DFSM visits the planes alpha.(i,j,k) = C of the sweep direction in
// order, the points of a plane in parallel.  Here the ordering is two-level: the cells of one
// cell diagonal a + b + c = D (canonical, i.e. reflected per direction) form one launch and
// run concurrently; inside a cell the CTA visits its point planes in order (sweep_dir).  This
// is another linear extension of the same dependency order -- when a point is relaxed exactly
// its upwind neighbours (smaller canonical i, j or k) already hold this sweep's values, in
// its own cell or in an upwind cell of diagonal D - 1, and its downwind neighbours do not --
// so every sweep produces the same values as the lexicographic FSM sweep of that direction
// and the number of sweeps is the FSM's.  DLSM skips work
// that cannot change anything; here at cell granularity: a cell is relaxed in a sweep only if
// one of its points changed in its last relaxation or a neighbour cell changed a point on the
// shared face since (an update is idempotent when no input changed, so the values, and the
// sweep count, are still the FSM's).
template <typename T, int R>
__global__ void __launch_bounds__(CellCfg<R>::NT, MinBlocks<T, R>::value)
k_dsweep(CellArgs A, int D)
{
    using C = CellCfg<R>;
    constexpr int R3 = C::R3, NPL = C::NPL, NT = C::NT;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    CellSmem<T, R> Msm(smem_raw);
    __shared__ CellShared<R> S;
    const int tid = threadIdx.x;
    Ctl* ctl = A.ctl;
    const int cps = A.cps;
    if (ctl->err != 0u || ctl->n_exits == 0u) return;   // invalid input: no sweeping
    const uint32_t dir = ctl->sweep_idx & 7u;   // set by k_sweep_end (previous launch)
    const uint32_t beg = A.diag_off[D], end = A.diag_off[D + 1];
    T* Vt = reinterpret_cast<T*>(A.Vt);
    const T* Ht = reinterpret_cast<const T*>(A.Ht);
    uint32_t nupd = 0, nwr = 0, nsteps = 0;
    unsigned long long nproc = 0, nw_cta = 0;
    const T kap = (T)A.kappa;
    T dmax = T(0);   // largest change of this thread (the sweep stops once it is <= kappa)
    for (uint32_t w = beg + blockIdx.x; w < end; w += gridDim.x) {
        const uint32_t e = A.diag_cells[w];
        const int a = (int)(e % (uint32_t)cps), b = (int)((e / (uint32_t)cps) % (uint32_t)cps),
                  cc = (int)(e / ((uint32_t)cps * (uint32_t)cps));
        const int cx = (dir & 1u) ? cps - 1 - a : a, cy = (dir & 2u) ? cps - 1 - b : b,
                  cz = (dir & 4u) ? cps - 1 - cc : cc;
        const uint32_t c = (uint32_t)cx + (uint32_t)cps * ((uint32_t)cy + (uint32_t)cps * (uint32_t)cz);
        EIK_CHECK(c < A.cap, "diagonal cell id");
        __syncthreads();   // shared memory of the previous cell is free; S.cell consumed
        if (tid == 0) {
            S.cell = 1u;
            if (A.locked) {
                S.cell = A.cact[c];
                A.cact[c] = 0;    // inputs consumed (re-set below or by a neighbour)
            }
            S.face_flag = 0;
            S.stat[2] = 0;
        }
        __syncthreads();
        if (!S.cell) continue;
        ++nproc;
        stage_cell_async<T, R>(Vt, Ht, Msm, c, cx, cy, cz, cps, A.cap);
        __syncthreads();
        const unsigned long long pm = (1ull << NPL) - 1ull;   // every plane, no gating (FSM)
        if constexpr (R < EIK_DIR_TEMPLATE_MIN_R) {
            sweep_dir<T, R, -1>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax, (int)dir);
        } else switch (dir) {
        case 0: sweep_dir<T, R, 0>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        case 1: sweep_dir<T, R, 1>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        case 2: sweep_dir<T, R, 2>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        case 3: sweep_dir<T, R, 3>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        case 4: sweep_dir<T, R, 4>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        case 5: sweep_dir<T, R, 5>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        case 6: sweep_dir<T, R, 6>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        default: sweep_dir<T, R, 7>(S, Msm, A.plane_tab, pm, true, nupd, nwr, nsteps, kap, dmax); break;
        }
        // (sweep_dir ends with a barrier: every changed point carries the sign bit of hf)
        unsigned long long nw = write_back_changed<T, R>(Vt + (int64_t)c * R3, Msm);
        if (A.locked) {
            // faces holding a changed point: the neighbour across them must run next time
            uint32_t fm = 0;
            for (int q = tid; q < 6 * R * R; q += NT) {
                const int f = q / (R * R), uv = q - f * R * R, u = uv % R, v = uv / R;
                int pa, pb, pd;
                switch (f) {
                case 0: pa = 0; pb = u; pd = v; break;
                case 1: pa = R - 1; pb = u; pd = v; break;
                case 2: pa = u; pb = 0; pd = v; break;
                case 3: pa = u; pb = R - 1; pd = v; break;
                case 4: pa = u; pb = v; pd = 0; break;
                default: pa = u; pb = v; pd = R - 1; break;
                }
                if (Msm.changed(pa + R * pb + R * R * pd)) fm |= 1u << f;
            }
            for (int o = 16; o > 0; o >>= 1) fm |= __shfl_xor_sync(0xffffffffu, fm, o);
            if ((tid & 31) == 0 && fm) atomicOr(&S.face_flag, fm);
        }
        for (int o = 16; o > 0; o >>= 1) nw += __shfl_xor_sync(0xffffffffu, nw, o);
        if ((tid & 31) == 0 && nw) atomicAdd(&S.stat[2], nw);
        __syncthreads();
        if (tid == 0) nw_cta += S.stat[2];
        if (A.locked) {
            if (tid < 6 && (S.face_flag & (1u << tid))) {
                const int64_t nc = face_neighbour(c, tid, cps);
                if (nc >= 0) A.cact[nc] = 1;
            }
            if (tid == 6 && S.stat[2]) A.cact[c] = 1;   // its own points changed: run again
        }
    }
    if (A.stats) {
        unsigned long long u64 = nupd, w64 = nwr;
        for (int o = 16; o > 0; o >>= 1) {
            u64 += __shfl_xor_sync(0xffffffffu, u64, o);
            w64 += __shfl_xor_sync(0xffffffffu, w64, o);
        }
        if ((tid & 31) == 0) {
            if (u64) atomicAdd(&ctl->updates, u64);
            if (w64) atomicAdd(&ctl->writes, w64);
        }
    }
    {
        float dm = dmax_up(dmax);
        for (int o = 16; o > 0; o >>= 1) dm = fmaxf(dm, __shfl_xor_sync(0xffffffffu, dm, o));
        if ((tid & 31) == 0 && dm > 0.f) atomicMax(&ctl->sweep_dmax, __float_as_uint(dm));
    }
    if (tid == 0) {
        if (nw_cta) atomicAdd(&ctl->sweep_writes, nw_cta);
        if (nproc) {
            atomicAdd(&ctl->processings, nproc);
            atomicAdd(&ctl->sweeps, nproc);
            atomicAdd(&ctl->bytes_written, nw_cta);
        }
    }
    (void)R3;
}

// seed the async ring with the initial cells (L <- Q^c, Alg. 1 line 2)
__global__ void k_seed_queue(uint32_t* state, uint32_t* ring, Ctl* ctl, int64_t J)
{
    if (__ldcg(&ctl->err) != 0u || __ldcg(&ctl->n_exits) == 0u) return;   // invalid input: no work
    for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < J;
         base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = base + threadIdx.x;
        const bool q = c < J && state[c] != 0;
        if (q) state[c] |= ST_QUEUED;
        warp_agg_append(&ctl->q_tail, ring, (uint32_t)c, q);
        const unsigned m = __ballot_sync(__activemask(), q);
        if ((threadIdx.x & 31) == 0 && m) atomicAdd(&ctl->pending, (uint32_t)__popc(m));
    }
}

// --------------------------------------------------------------------------------------
// A8: egress, tiles -> lexicographic U_out
// --------------------------------------------------------------------------------------
template <typename T>
__global__ void k_egress(Geom g, const T* __restrict__ Vt, T* __restrict__ U, int64_t M, const Ctl* ctl)
{
    // a device-detected input error or an aborted loop leaves U_out untouched (EIK_EINVAL
    // contract; the host reads the status once, after this kernel)
    if (__ldcg(&ctl->err) != 0u || __ldcg(&ctl->abort) != 0u || __ldcg(&ctl->n_exits) == 0u) return;
    // four consecutive output points of one (j, k) row per thread, flat over the z-plane
    // (blockIdx.y strides over k): one 16-byte tile read, four coalesced scalar writes
    const int r = g.r, lr = g.lr;
    const int64_t n1 = g.n1;
    const uint32_t cps = (uint32_t)g.cps;
    const uint32_t n1v = (uint32_t)((n1 + 3) >> 2);      // vectors per row
    const uint32_t nv = n1v * (uint32_t)n1;              // vectors per z-plane (< 2^32)
    for (int64_t k = blockIdx.y; k < n1; k += gridDim.y) {
        const uint32_t ck = (uint32_t)(k >> lr) * cps;
        const int ek = r * r * (int)(k & (r - 1));
        for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < nv; t += gridDim.x * blockDim.x) {
            const uint32_t j = t / n1v, iv = t - j * n1v;
            const int64_t i0 = (int64_t)iv << 2;
            const uint32_t c = (uint32_t)(i0 >> lr) + cps * ((j >> lr) + ck);
            const int e = (int)(i0 & (r - 1)) + r * (int)(j & (r - 1)) + ek;
            T v[4];
            Vec4T<T>::ld(&Vt[((int64_t)c << (3 * lr)) + e], v);
            T* out = U + (int64_t)j * n1 + n1 * n1 * k + i0;
#pragma unroll
            for (int l = 0; l < 4; ++l)
                if (i0 + l < n1) __stcs(&out[l], v[l]);
        }
    }
}

}  // namespace eik
