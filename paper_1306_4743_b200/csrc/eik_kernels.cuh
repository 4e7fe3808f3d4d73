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
};

enum : uint32_t { FLAG_INIT = 64u };   // state bit: activate every point (first processing)

struct Geom {
    int64_t n1;        // n + 1 points per side
    int32_t cps;       // cells per side
    int32_t r;
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
template <typename T>
__global__ void k_ingest(Geom g, T h, const T* __restrict__ F, const uint8_t* __restrict__ mask,
                         const T* __restrict__ q, T* __restrict__ Vt, T* __restrict__ Ht,
                         uint32_t* __restrict__ key, uint32_t* __restrict__ state, Ctl* ctl,
                         int64_t P)
{
    const int r = g.r, r3 = r * r * r;
    const int64_t n1 = g.n1;
    const int cps = g.cps;
    uint32_t exits = 0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = p / r3;
        const int e = (int)(p - c * r3);
        const int a = e % r, b = (e / r) % r, d = e / (r * r);
        const int cx = (int)(c % cps), cy = (int)((c / cps) % cps), cz = (int)(c / ((int64_t)cps * cps));
        const int64_t i = (int64_t)cx * r + a, j = (int64_t)cy * r + b, k = (int64_t)cz * r + d;
        T v = dinf<T>(), hf = dinf<T>();
        if (i < n1 && j < n1 && k < n1) {
            const int64_t lex = i + n1 * (j + n1 * k);
            const T f = F[lex];
            if (!(f >= T(0)) || !(f < dinf<T>())) atomicOr(&ctl->err, 1u);   // F < 0, NaN, inf
            if (mask[lex]) {
                T qv = q[lex];
                if (!(qv >= T(0)) || !(qv < dinf<T>())) atomicOr(&ctl->err, 2u);
                qv = qv + T(0);   // canonicalise -0 -> +0 (R9)
                v = qv;           // exits: fixed, V = q (hf stays +inf: never updated)
                ++exits;
                const uint32_t kb = key_bits(qv);
                // V^c of a cell in Q^c = min exit value; cells holding a non-exit
                // neighbour of an exit across a cell face are seeded too (R18)
                atomicMin(&key[c], kb);
                atomicOr(&state[c], FLAG_INIT);
                const int64_t cc[6] = {a == 0 && i > 0 ? c - 1 : -1,
                                       a == r - 1 && i + 1 < n1 ? c + 1 : -1,
                                       b == 0 && j > 0 ? c - cps : -1,
                                       b == r - 1 && j + 1 < n1 ? c + cps : -1,
                                       d == 0 && k > 0 ? c - (int64_t)cps * cps : -1,
                                       d == r - 1 && k + 1 < n1 ? c + (int64_t)cps * cps : -1};
#pragma unroll
                for (int f2 = 0; f2 < 6; ++f2)
                    if (cc[f2] >= 0) {
                        atomicMin(&key[cc[f2]], kb);
                        atomicOr(&state[cc[f2]], FLAG_INIT);
                    }
            } else if (f > T(0)) {
                hf = h / f;       // +inf for subnormal-overflow: treated as impassable
            }
        }
        Vt[p] = v;
        Ht[p] = hf;
    }
    // exit count (warp-aggregated)
    for (int o = 16; o > 0; o >>= 1) exits += __shfl_xor_sync(0xffffffffu, exits, o);
    if ((threadIdx.x & 31) == 0 && exits) atomicAdd(&ctl->n_exits, exits);
}

__global__ void k_init_cells(uint32_t* key, uint32_t* state, int64_t J)
{
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < J;
         c += (int64_t)gridDim.x * blockDim.x) {
        key[c] = KEY_INF;
        state[c] = 0;
    }
}

__global__ void k_build_wl(const uint32_t* __restrict__ key, const uint32_t* __restrict__ state,
                           uint32_t* wl0, Ctl* ctl, int64_t J)
{
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
                         uint32_t* proc_flags, uint32_t* key, uint32_t* state, float delta)
{
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
            key[c] = KEY_INF;                 // V^c <- +inf on removal
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
__device__ __forceinline__ bool round_end_body(Ctl* ctl)
{
    const uint32_t cur = ctl->cur, nx = cur ^ 1u;
    ctl->rounds += 1;
    if (ctl->proc_count > ctl->max_proc) ctl->max_proc = ctl->proc_count;
    ctl->processings += ctl->proc_count;
    ctl->proc_count = 0;
    ctl->wl_count[cur] = 0;
    ctl->kmin[cur] = KEY_INF;
    ctl->cur = nx;
    const bool more = ctl->wl_count[nx] != 0;
    if (more && ctl->rounds >= ctl->max_rounds) ctl->err |= 4u;
    ctl->done = (more && ctl->rounds < ctl->max_rounds) ? 0u : 1u;
    return ctl->done != 0u;
}

__global__ void k_round_end(Ctl* ctl) { (void)round_end_body(ctl); }

// --------------------------------------------------------------------------------------
// A3-A6: the cell-sweep kernel
// --------------------------------------------------------------------------------------
template <int R> struct CellCfg {
    static constexpr int R3 = R * R * R;
    static constexpr int RP = R + 2;
    static constexpr int RP2 = RP * RP;
    static constexpr int BOX = RP * RP * RP;
    static constexpr int NPL = 3 * R - 2;                                 // wavefront planes
    static constexpr int NT = R == 16 ? 192 : (R == 8 ? 64 : 32);          // >= largest plane
};

template <typename T, int R>
constexpr size_t cell_smem_bytes()
{
    return sizeof(T) * (CellCfg<R>::BOX + CellCfg<R>::R3) + CellCfg<R>::R3;
}

struct CellArgs {
    Ctl* ctl;
    const uint32_t* proc_cell;
    const uint32_t* proc_flags;
    uint32_t* wl0;
    uint32_t* wl1;
    uint32_t* key;
    uint32_t* state;
    const uint16_t* plane_tab;   // R^3 entries (a | b<<4 | c<<8) sorted by a+b+c
    const int32_t* plane_off;    // NPL + 1 offsets
    void* Vt;
    const void* Ht;
    int64_t n1;
    int32_t cps;
    int32_t stats;
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

template <typename T, int R>
__global__ void __launch_bounds__(CellCfg<R>::NT)
k_cell(CellArgs A)
{
    using C = CellCfg<R>;
    constexpr int NT = C::NT, R3 = C::R3, RP = C::RP, RP2 = C::RP2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* sV = reinterpret_cast<T*>(smem_raw);               // (R+2)^3 box incl. halo faces
    T* sH = sV + C::BOX;                                  // R^3 hf
    uint8_t* sF = reinterpret_cast<uint8_t*>(sH + R3);    // R^3 flags: bit0 active, bit1 changed
    __shared__ uint32_t sFaceMin[6];
    __shared__ uint32_t sFaceFlag;
    __shared__ unsigned long long sCnt[3];

    const int tid = threadIdx.x;
    Ctl* ctl = A.ctl;
    const uint32_t nproc = ctl->proc_count;
    const uint32_t nx = ctl->cur ^ 1u;
    uint32_t* wn = nx ? A.wl1 : A.wl0;
    T* Vt = reinterpret_cast<T*>(A.Vt);
    const T* Ht = reinterpret_cast<const T*>(A.Ht);
    const int cps = A.cps;
    const int64_t n1 = A.n1;
    const T INF = dinf<T>();

    for (uint32_t w = blockIdx.x; w < nproc; w += gridDim.x) {
        const uint32_t c = A.proc_cell[w];
        const uint32_t flags = A.proc_flags[w];
        const int cx = (int)(c % (uint32_t)cps), cy = (int)((c / (uint32_t)cps) % (uint32_t)cps),
                  cz = (int)(c / ((uint32_t)cps * (uint32_t)cps));
        const int64_t base = (int64_t)c * R3;
        if (tid < 6) sFaceMin[tid] = KEY_INF;
        if (tid == 0) { sFaceFlag = 0; sCnt[0] = sCnt[1] = sCnt[2] = 0; }

        // ---- stage tile + hf + flags ----
        const bool init = flags & FLAG_INIT;
        for (int e = tid; e < R3; e += NT) {
            const int a = e % R, b = (e / R) % R, d = e / (R * R);
            sV[(a + 1) + RP * (b + 1) + RP2 * (d + 1)] = Vt[base + e];
            sH[e] = Ht[base + e];
            sF[e] = init ? 1 : 0;
        }
        // ---- halo N(c): 6 faces of r^2 from the neighbour tiles (+inf outside the grid) ----
        for (int e = tid; e < 6 * R * R; e += NT) {
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
            T hv = INF;
            if (ex) hv = Vt[nc * R3 + sa + R * sb + R * R * sd];
            sV[(hx + 1) + RP * (hy + 1) + RP2 * (hz + 1)] = hv;
        }
        __syncthreads();
        if (!init) {
            // re-activation: every point of each face that received new inflow
            for (int e = tid; e < 6 * R * R; e += NT) {
                const int f = e / (R * R), uv = e - f * R * R, u = uv % R, v = uv / R;
                if (!(flags & (1u << f))) continue;
                int a, b, d;
                switch (f) {
                case 0: a = 0; b = u; d = v; break;
                case 1: a = R - 1; b = u; d = v; break;
                case 2: a = u; b = 0; d = v; break;
                case 3: a = u; b = R - 1; d = v; break;
                case 4: a = u; b = v; d = 0; break;
                default: a = u; b = v; d = R - 1; break;
                }
                sF[a + R * b + R * R * d] = 1;
            }
            __syncthreads();
        }

        // ---- gated GS sweeps in wavefront order until no point is active ----
        const uint32_t pref = init ? 0u : pref_dirs(flags & 63u);
        const int gray[8] = {0, 1, 3, 2, 6, 7, 5, 4};
        int gi = 0;
        bool pref_phase = pref != 0;
        uint32_t nsweeps = 0;
        unsigned long long nupd = 0, nwr = 0;
        for (;;) {
            int any = 0;
            const uint32_t* sF32 = reinterpret_cast<const uint32_t*>(sF);
            for (int wd = tid; wd < R3 / 4; wd += NT) any |= (sF32[wd] & 0x01010101u) != 0;
            if (!__syncthreads_or(any)) break;
            int dir;
            if (pref_phase) {
                while (gi < 8 && !(pref & (1u << gray[gi]))) ++gi;
                if (gi < 8) { dir = gray[gi++]; }
                else { pref_phase = false; gi = 0; dir = gray[gi++]; }
            } else {
                dir = gray[gi];
                gi = (gi + 1) & 7;
            }
            ++nsweeps;
            for (int s = 0; s < C::NPL; ++s) {
                const int e = __ldg(&A.plane_off[s]) + tid;
                if (e < __ldg(&A.plane_off[s + 1])) {
                    const uint32_t ent = __ldg(&A.plane_tab[e]);
                    int i = ent & 15, j = (ent >> 4) & 15, k = (ent >> 8) & 15;
                    if (dir & 1) i = R - 1 - i;
                    if (dir & 2) j = R - 1 - j;
                    if (dir & 4) k = R - 1 - k;
                    const int p = i + R * j + R * R * k;
                    uint8_t fl = sF[p];
                    if (fl & 1) {
                        fl &= (uint8_t)~1u;                    // Alg. 2 line 4: set inactive
                        const T hf = sH[p];
                        const int qb = (i + 1) + RP * (j + 1) + RP2 * (k + 1);
                        const T v = sV[qb];
                        const T xm = sV[qb - 1], xp = sV[qb + 1];
                        const T ym = sV[qb - RP], yp = sV[qb + RP];
                        const T zm = sV[qb - RP2], zp = sV[qb + RP2];
                        const T mx = fmin(xm, xp), my = fmin(ym, yp), mz = fmin(zm, zp);
                        const T a1 = fmin(mx, fmin(my, mz));
                        if (hf < INF && a1 < v) {              // fixed points never update
                            ++nupd;
                            const T u = local_solve<T>(mx, my, mz, hf);   // line 5
                            if (u < v) {                                  // line 6
                                sV[qb] = u;                               // line 7
                                fl |= 2u;
                                ++nwr;
                                // lines 8-13: activate larger neighbours; across the cell
                                // border, tag the face as currently downwind (Eq. (3) value)
                                const uint32_t kb = key_bits(u);
                                if (xm > u) { if (i > 0) sF[p - 1] |= 1u; else { atomicOr(&sFaceFlag, 1u); atomicMin(&sFaceMin[0], kb); } }
                                if (xp > u) { if (i < R - 1) sF[p + 1] |= 1u; else { atomicOr(&sFaceFlag, 2u); atomicMin(&sFaceMin[1], kb); } }
                                if (ym > u) { if (j > 0) sF[p - R] |= 1u; else { atomicOr(&sFaceFlag, 4u); atomicMin(&sFaceMin[2], kb); } }
                                if (yp > u) { if (j < R - 1) sF[p + R] |= 1u; else { atomicOr(&sFaceFlag, 8u); atomicMin(&sFaceMin[3], kb); } }
                                if (zm > u) { if (k > 0) sF[p - R * R] |= 1u; else { atomicOr(&sFaceFlag, 16u); atomicMin(&sFaceMin[4], kb); } }
                                if (zp > u) { if (k < R - 1) sF[p + R * R] |= 1u; else { atomicOr(&sFaceFlag, 32u); atomicMin(&sFaceMin[5], kb); } }
                            }
                        }
                        sF[p] = fl;
                    }
                }
                __syncthreads();
            }
        }

        // ---- write back changed values only ----
        unsigned long long nw = 0;
        for (int e = tid; e < R3; e += NT) {
            if (sF[e] & 2u) {
                const int a = e % R, b = (e / R) % R, d = e / (R * R);
                Vt[base + e] = sV[(a + 1) + RP * (b + 1) + RP2 * (d + 1)];
                ++nw;
            }
        }
        if (A.stats) {
            atomicAdd(&sCnt[0], nupd);
            atomicAdd(&sCnt[1], nwr);
            atomicAdd(&sCnt[2], nw);
        }
        __syncthreads();

        // ---- re-activate currently-downwind neighbour cells (Alg. 1 lines 7-10) ----
        if (tid < 6) {
            const int f = tid;
            const bool exists = f == 0 ? cx > 0 : f == 1 ? cx < cps - 1 : f == 2 ? cy > 0
                              : f == 3 ? cy < cps - 1 : f == 4 ? cz > 0 : cz < cps - 1;
            if (exists && (sFaceFlag & (1u << f))) {
                const int64_t nc = f == 0 ? (int64_t)c - 1 : f == 1 ? (int64_t)c + 1
                                 : f == 2 ? (int64_t)c - cps : f == 3 ? (int64_t)c + cps
                                 : f == 4 ? (int64_t)c - (int64_t)cps * cps
                                          : (int64_t)c + (int64_t)cps * cps;
                const uint32_t kb = sFaceMin[f];
                atomicMin(&A.key[nc], kb);                                   // Eq. (3)
                const uint32_t old = atomicOr(&A.state[nc], 1u << (f ^ 1));  // face of nc
                if (old == 0u) {                                             // Alg. 5 analogue
                    const uint32_t s = atomicAdd(&ctl->wl_count[nx], 1u);
                    wn[s] = (uint32_t)nc;
                }
                atomicMin(&ctl->kmin[nx], kb);
            }
        }
        if (tid == 0 && A.stats) {
            atomicAdd(&ctl->updates, sCnt[0]);
            atomicAdd(&ctl->writes, sCnt[1]);
            atomicAdd(&ctl->bytes_written, sCnt[2]);
            atomicAdd(&ctl->sweeps, (unsigned long long)nsweeps);
            // real (non-padding) points of this cell
            const int64_t rx = (n1 - (int64_t)cx * R) < R ? (n1 - (int64_t)cx * R) : R;
            const int64_t ry = (n1 - (int64_t)cy * R) < R ? (n1 - (int64_t)cy * R) : R;
            const int64_t rz = (n1 - (int64_t)cz * R) < R ? (n1 - (int64_t)cz * R) : R;
            atomicAdd(&ctl->real_pts, (unsigned long long)(rx * ry * rz));
        }
        __syncthreads();   // smem reuse by the next cell of this CTA
    }
}

// --------------------------------------------------------------------------------------
// A8: egress, tiles -> lexicographic U_out
// --------------------------------------------------------------------------------------
template <typename T>
__global__ void k_egress(Geom g, const T* __restrict__ Vt, T* __restrict__ U, int64_t M)
{
    const int r = g.r, r3 = r * r * r;
    const int64_t n1 = g.n1;
    const int cps = g.cps;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < M;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx % n1, j = (idx / n1) % n1, k = idx / (n1 * n1);
        const int64_t c = (i / r) + cps * ((j / r) + (int64_t)cps * (k / r));
        const int e = (int)(i % r) + r * (int)(j % r) + r * r * (int)(k % r);
        U[idx] = Vt[c * r3 + e];
    }
}

}  // namespace eik
