// eik_b2.cuh -- r = 16 cell processing on 2x2x2 micro-blocks (the async scheduler's default cell
// kernel for r = 16, kappa = 0, no sweep cap).  PRODUCT PATH; included by eik_kernels.cuh users
// after eik_kernels.cuh.
//
// Same method as cell_process (HCM "perform modified LSM on c until convergence", Alg. 1 line 6,
// P:423-428; Detrixhe wavefront sweeps inside the cell), different thread
// mapping.  A 16^3 cell is 8^3 blocks of 2x2x2 points; a sweep in direction d visits the 22
// block planes A' + B' + C' = S (primes: coordinates reflected per d) in order, one thread per
// block; inside its block the thread relaxes the 8 points in the canonical order of d (levels
// 0, 1, 2, 3 of i' + j' + k'), so every point is relaxed after its upwind neighbours -- the exact
// Gauss-Seidel order of the sweep, as in sweep_dir, but with 8 points per thread-step:
//   * one shared-memory round trip per block-step (24 loads, 2-wide vectors) instead of one
//     per point, and a barrier per 2 point planes;
//   * Alg. 2's activity is kept per block (512 flags instead of 4096): a block is relaxed when
//     its flag is set, a changed point activates the neighbour BLOCK across a face when the
//     neighbour value there is larger (Alg. 2 lines 8-13 at block granularity; conservative:
//     more relaxations, never fewer), and re-activates its own block when an upwind point of
//     the block itself became larger than it;
//   * the per-point bookkeeping of sweep_dir (flag loads, six activation stores, border tests)
//     becomes a few predicated stores per block.
// Values only decrease and every relaxation is exact Eq. (2), so the fixed point is the same
// (P:476-477); the tests compare it with the oracle like every other path.
#pragma once

namespace eik {

struct B2 {
    static constexpr int R = 16, R3 = 4096;
    static constexpr int NB = 8, NB3 = 512, NBP = 3 * NB - 2;   // blocks per side, blocks, block planes
    static constexpr int NT = 64;                                // threads (largest block plane: 48)
    static constexpr int XP = 20, SP = XP * 18, BOX = SP * 18;   // box: x pitch 20 (interior at x = 2)
    static constexpr int ROWS = NBP + 2;                         // table rows (2 trailing dummy planes)
    static constexpr int FL_DUMMY = NB3;                         // flag byte of the dummy block
};
template <typename T> struct B2Minb { static constexpr int value = sizeof(T) == 4 ? 5 : 4; };

// box index of point (a, b, c), a, b, c in [-1, 16]; even for even a (2-wide vector loads)
__host__ __device__ constexpr int b2q(int a, int b, int c) { return (a + 2) + B2::XP * (b + 1) + B2::SP * (c + 1); }

// Per-direction block-plane table (host-built, eik.cu make_tab_b2): tab[d][S][t] = uint2
//   x = q0 | eb << 13 | bm << 23   (q0 = box index of the block's first point, eb = physical
//       block index A + 8 B + 64 C, bm = neighbour blocks that exist in the canonical
//       orientation of d: bit 0 downstream x, 1 upstream x, 2/3 y, 4/5 z)
//   y = h0 = hf index of the block's first point (dense 16^3)
// Threads without a block on a plane get B2_DUMMY: block (0, 0, 0)'s box (reads only), the
// dummy flag byte (always 0), no neighbours.
static constexpr uint32_t B2_DUMMY_X = (uint32_t)b2q(0, 0, 0) | ((uint32_t)B2::FL_DUMMY << 13);

template <typename T> constexpr size_t b2_smem_bytes()
{
    // V box, hf (fp32; fp64 reads hf from global memory), block flags (+ dummy), changed masks
    return sizeof(T) * B2::BOX + (sizeof(T) == 4 ? sizeof(T) * B2::R3 : 0) + (B2::NB3 + 16) + B2::NB3;
}

template <typename T> struct B2Smem {
    T* V;
    T* H;           // fp32: dense 16^3 hf; fp64: null
    uint8_t* fl;    // block activity (Alg. 2 at block granularity), [512] = dummy
    uint8_t* chg;   // changed points of each block (bit ix + 2 jy + 4 kz)
    const T* Hg;    // fp64: this cell's hf tile in global memory
    __device__ explicit B2Smem(unsigned char* raw)
    {
        V = reinterpret_cast<T*>(raw);
        H = sizeof(T) == 4 ? V + B2::BOX : nullptr;
        fl = reinterpret_cast<uint8_t*>(V + B2::BOX + (sizeof(T) == 4 ? B2::R3 : 0));
        chg = fl + B2::NB3 + 16;
        Hg = nullptr;
    }
};

template <typename T> struct Pair;
template <> struct Pair<float> {
    static __device__ __forceinline__ void ld(uint32_t a, float& x, float& y)
    { asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a)); }
    static __device__ __forceinline__ void st(uint32_t a, float x, float y)
    { asm volatile("st.shared.v2.f32 [%0], {%1, %2};" :: "r"(a), "f"(x), "f"(y)); }
};
template <> struct Pair<double> {
    static __device__ __forceinline__ void ld(uint32_t a, double& x, double& y)
    { asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a)); }
    static __device__ __forceinline__ void st(uint32_t a, double x, double y)
    { asm volatile("st.shared.v2.f64 [%0], {%1, %2};" :: "r"(a), "d"(x), "d"(y)); }
};

// Relax canonical point p = ci + 2 cj + 4 ck of the block (compile-time indices: everything
// lives in registers).  The block's values and faces were loaded in the canonical orientation of
// the sweep direction (coordinates reflected per d), so one copy of this code serves all eight
// directions: upwind neighbours are at smaller canonical coordinates -- inside the block (already
// relaxed in this pass) or on the upwind faces (relaxed in the previous block-plane step) --
// downwind ones at larger.  (Eight direction-specialised copies of the step measured 2-3x slower:
// ~10 KB of straight-line code per step each, which the instruction cache cannot hold.)
template <typename T, int CI, int CJ, int CK>
__device__ __forceinline__ void b2_point(T (&P)[8], const T (&H)[8], const T (&XU)[4], const T (&XD)[4],
                                         const T (&YU)[4], const T (&YD)[4], const T (&ZU)[4],
                                         const T (&ZD)[4], bool act, uint32_t& cm, uint32_t& gm)
{
    constexpr int p = CI + 2 * CJ + 4 * CK;
    const T xu = CI ? P[p - 1] : XU[CJ + 2 * CK], xd = CI ? XD[CJ + 2 * CK] : P[p + 1];
    const T yu = CJ ? P[p - 2] : YU[CI + 2 * CK], yd = CJ ? YD[CI + 2 * CK] : P[p + 2];
    const T zu = CK ? P[p - 4] : ZU[CI + 2 * CJ], zd = CK ? ZD[CI + 2 * CJ] : P[p + 4];
    const T mx = vmin(xu, xd), my = vmin(yu, yd), mz = vmin(zu, zd);
    const T v = P[p], hf = H[p];
    const bool gate = act && hf < dinf<T>() && vmin(mx, vmin(my, mz)) < v;   // not fixed, can gain
    const T u = local_solve_fast<T>(mx, my, mz, hf);                          // Alg. 2 line 5
    const bool c = gate && u < v;                                             // line 6
    P[p] = c ? u : v;                                                         // line 7
    cm |= (uint32_t)c << p;
    gm |= (uint32_t)gate << p;
}

template <typename T>
__device__ __forceinline__ void b2_ld_pair(uint32_t a, bool swap, T& c0, T& c1)
{
    T x, y;
    Pair<T>::ld(a, x, y);
    c0 = swap ? y : x;
    c1 = swap ? x : y;
}

// One block-plane sweep in direction dir (bit 0/1/2: x/y/z descending) over the planes in pm.
// Returns the axes (bit 0 x, 1 y, 2 z) along which something behind the wavefront was activated.
template <typename T>
__device__ __forceinline__ uint32_t sweep_b2(const B2Smem<T>& M, const uint2* __restrict__ tab, uint32_t pm,
                                             int dir, uint32_t& nupd_out, uint32_t& nwr_out, uint32_t& nsteps_out)
{
    uint32_t nupd = 0, nwr = 0, nsteps = 0;   // (registers; the caller's counters are updated once)
    constexpr int TS = (int)sizeof(T);
    constexpr int XPB = B2::XP * TS, SPB = B2::SP * TS;   // box row / slice pitch, bytes
    const bool fx = dir & 1, fy = dir & 2, fz = dir & 4;
    // physical offsets (bytes) of the canonical rows / slices 0 and 1 inside a block, of the
    // upwind / downwind face rows, and (block units) of the downwind neighbour blocks
    const uint32_t oy0 = fy ? XPB : 0, oy1 = fy ? 0 : XPB, oz0 = fz ? SPB : 0, oz1 = fz ? 0 : SPB;
    const uint32_t hy0 = fy ? 16 * TS : 0, hy1 = fy ? 0 : 16 * TS, hz0 = fz ? 256 * TS : 0, hz1 = fz ? 0 : 256 * TS;
    const uint32_t oxu = fx ? 2 * TS : (uint32_t)-TS, oxd = fx ? (uint32_t)-TS : 2 * TS;
    const uint32_t oyu = fy ? 2 * XPB : (uint32_t)-XPB, oyd = fy ? (uint32_t)-XPB : 2 * XPB;
    const uint32_t ozu = fz ? 2 * SPB : (uint32_t)-SPB, ozd = fz ? (uint32_t)-SPB : 2 * SPB;
    const uint32_t dbx = fx ? (uint32_t)-1 : 1u, dby = fy ? (uint32_t)-8 : 8u, dbz = fz ? (uint32_t)-64 : 64u;
    const uint32_t vb = smem_u32(M.V), fb = smem_u32(M.fl), cb = smem_u32(M.chg);
    const uint32_t hb = sizeof(T) == 4 ? smem_u32(M.H) : 0u;
    const T* __restrict__ hg = M.Hg;
    const uint2* __restrict__ tp = tab + dir * B2::ROWS * B2::NT + threadIdx.x;
    uint32_t one;
    asm volatile("mov.u32 %0, 1;" : "=r"(one));
    bool fwd = false;
    uint32_t bwd = 0;
    int s = __ffs(pm) - 1;
    uint32_t pmr = pm >> s;
    uint2 en = __ldg(tp + s * B2::NT);
    tp += (s + 1) * B2::NT;
    for (; s < B2::NBP; ++s, pmr >>= 1) {
        if (!((pmr & 1u) | (uint32_t)fwd)) {
            if (pmr == 0u) break;
            en = __ldg(tp);
            tp += B2::NT;
            continue;
        }
        const uint2 ue = en;
        en = __ldg(tp);   // next plane's entry (independent of this step)
        tp += B2::NT;
        const uint32_t q0 = vb + (ue.x & 0x1fffu) * TS;
        const uint32_t eb = (ue.x >> 13) & 1023u;
        // ---- loads in canonical orientation: flag, changed mask, 8 values, 8 hf, 24 faces ----
        const uint32_t act = lds_u8(fb + eb);
        const uint32_t ch0 = lds_u8(cb + (eb & 511u));
        T P[8], H[8], XU[4], XD[4], YU[4], YD[4], ZU[4], ZD[4];
#pragma unroll
        for (int jk = 0; jk < 4; ++jk) {
            const uint32_t row = q0 + ((jk & 1) ? oy1 : oy0) + ((jk >> 1) ? oz1 : oz0);
            b2_ld_pair<T>(row, fx, P[2 * jk], P[2 * jk + 1]);
            XU[jk] = lds<T>(row + oxu);
            XD[jk] = lds<T>(row + oxd);
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint32_t sl = q0 + (k ? oz1 : oz0);
            b2_ld_pair<T>(sl + oyu, fx, YU[2 * k], YU[2 * k + 1]);
            b2_ld_pair<T>(sl + oyd, fx, YD[2 * k], YD[2 * k + 1]);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const uint32_t rw = q0 + (j ? oy1 : oy0);
            b2_ld_pair<T>(rw + ozu, fx, ZU[2 * j], ZU[2 * j + 1]);
            b2_ld_pair<T>(rw + ozd, fx, ZD[2 * j], ZD[2 * j + 1]);
        }
        if constexpr (sizeof(T) == 4) {
#pragma unroll
            for (int jk = 0; jk < 4; ++jk)
                b2_ld_pair<T>(hb + ue.y * TS + ((jk & 1) ? hy1 : hy0) + ((jk >> 1) ? hz1 : hz0), fx,
                              H[2 * jk], H[2 * jk + 1]);
        } else {
            const bool real = eb < 512u;
#pragma unroll
            for (int jk = 0; jk < 4; ++jk) {
                double2 hv = make_double2(dinf<T>(), dinf<T>());
                if (real)
                    hv = __ldg(reinterpret_cast<const double2*>(
                        reinterpret_cast<const char*>(hg + ue.y) + ((jk & 1) ? hy1 : hy0) + ((jk >> 1) ? hz1 : hz0)));
                H[2 * jk] = fx ? hv.y : hv.x;
                H[2 * jk + 1] = fx ? hv.x : hv.y;
            }
        }
        const bool a = act != 0u;
        if (a) sts_u8(fb + eb, 0u);   // Alg. 2 line 4 (nothing else writes this flag during this step)
        bool myfwd = false;
        if (__any_sync(0xffffffffu, a)) {
            uint32_t cm = 0, gm = 0;
            // the 8 points in canonical order: level 0, 1 (3 independent), 2 (3), 3
            b2_point<T, 0, 0, 0>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            b2_point<T, 1, 0, 0>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            b2_point<T, 0, 1, 0>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            b2_point<T, 0, 0, 1>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            b2_point<T, 1, 1, 0>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            b2_point<T, 1, 0, 1>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            b2_point<T, 0, 1, 1>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            b2_point<T, 1, 1, 1>(P, H, XU, XD, YU, YD, ZU, ZD, a, cm, gm);
            nupd += __popc(gm);
            nwr += __popc(cm);
            // write back the changed point pairs (physical order), record them (physical bits)
#pragma unroll
            for (int jk = 0; jk < 4; ++jk)
                if ((cm >> (2 * jk)) & 3u) {
                    const uint32_t row = q0 + ((jk & 1) ? oy1 : oy0) + ((jk >> 1) ? oz1 : oz0);
                    Pair<T>::st(row, fx ? P[2 * jk + 1] : P[2 * jk], fx ? P[2 * jk] : P[2 * jk + 1]);
                }
            if (cm) {
                uint32_t pmk = cm;   // canonical -> physical bit order (reflect the set axes)
                if (fx) pmk = ((pmk & 0x55u) << 1) | ((pmk >> 1) & 0x55u);
                if (fy) pmk = ((pmk & 0x33u) << 2) | ((pmk >> 2) & 0x33u);
                if (fz) pmk = ((pmk & 0x0fu) << 4) | (pmk >> 4);
                sts_u8(cb + eb, ch0 | pmk);
            }
            // activations (Alg. 2 lines 8-13 per block): a changed point whose neighbour across
            // a block face is larger activates that block; a changed point whose upwind
            // neighbour inside the block ended larger re-activates the block itself
            auto C = [&](int p) { return ((cm >> p) & 1u) != 0u; };
            bool xu = false, xd = false, yu = false, yd = false, zu = false, zd = false;
            uint32_t selfax = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int lo = u & 1, hi = u >> 1;
                xu |= C(2 * lo + 4 * hi) && XU[u] > P[2 * lo + 4 * hi];
                xd |= C(1 + 2 * lo + 4 * hi) && XD[u] > P[1 + 2 * lo + 4 * hi];
                yu |= C(lo + 4 * hi) && YU[u] > P[lo + 4 * hi];
                yd |= C(lo + 2 + 4 * hi) && YD[u] > P[lo + 2 + 4 * hi];
                zu |= C(lo + 2 * hi) && ZU[u] > P[lo + 2 * hi];
                zd |= C(lo + 2 * hi + 4) && ZD[u] > P[lo + 2 * hi + 4];
                // internal edges: the upwind endpoint has canonical coordinate 0 on the axis
                if (C(2 * lo + 4 * hi + 1) && P[2 * lo + 4 * hi] > P[2 * lo + 4 * hi + 1]) selfax |= 1u;
                if (C(lo + 4 * hi + 2) && P[lo + 4 * hi] > P[lo + 4 * hi + 2]) selfax |= 2u;
                if (C(lo + 2 * hi + 4) && P[lo + 2 * hi] > P[lo + 2 * hi + 4]) selfax |= 4u;
            }
            const uint32_t bm = ue.x >> 23;   // neighbour blocks that exist (canonical)
            const bool dx = xd && (bm & 1u), ux = xu && (bm & 2u);
            const bool dy = yd && (bm & 4u), uy = yu && (bm & 8u);
            const bool dz = zd && (bm & 16u), uz = zu && (bm & 32u);
            if (dx) sts_u8(fb + eb + dbx, one);
            if (ux) sts_u8(fb + eb - dbx, one);
            if (dy) sts_u8(fb + eb + dby, one);
            if (uy) sts_u8(fb + eb - dby, one);
            if (dz) sts_u8(fb + eb + dbz, one);
            if (uz) sts_u8(fb + eb - dbz, one);
            if (selfax) sts_u8(fb + eb, one);
            myfwd = dx | dy | dz;
            bwd |= (uint32_t)ux | ((uint32_t)uy << 1) | ((uint32_t)uz << 2) | selfax;
        }
        fwd = __syncthreads_or(myfwd);
        ++nsteps;
    }
    nupd_out += nupd;
    nwr_out += nwr;
    nsteps_out += nsteps;
    return bwd;
}

// Process one cell (the B2 form of cell_process; same contract: on return the face summaries
// face_flag / face_min / face_max are in S and the changed values are written back).
template <typename T>
__device__ __forceinline__ void cell_process_b2(const CellArgs& A, CellShared<16>& S, B2Smem<T>& M,
                                                uint32_t c, uint32_t flags, unsigned long long& n_sweeps_out)
{
    constexpr int NT = B2::NT, R = 16, R3 = B2::R3;
    const int tid = threadIdx.x;
    T* Vt = reinterpret_cast<T*>(A.Vt);
    const T* Ht = reinterpret_cast<const T*>(A.Ht);
    const int cps = A.cps;
    const T INF = dinf<T>();
    const int cx = (int)(c % (uint32_t)cps), cy = (int)((c / (uint32_t)cps) % (uint32_t)cps),
              cz = (int)(c / ((uint32_t)cps * (uint32_t)cps));
    const int64_t base = (int64_t)c * R3;
    const bool init = flags & FLAG_INIT;
    if (tid < 6) { S.face_min[tid] = KEY_INF; S.face_max[tid] = 0u; }
    if (tid == 0) {
        S.face_flag = 0;
        S.cont = 0;
        S.cont_key = KEY_INF;
        S.tm[0] = (uint32_t)clock64();
        S.tm[4] = S.tm[5] = S.tm[6] = 0;
    }
    // ---- stage: halo loads first (scattered, one memory round trip with the tile), the tile
    // through L2 in 16-byte vectors (another SM may have written it since this SM cached it),
    // hf (read-only during the solve) by cp.async; flags cleared meanwhile ----
    {
        constexpr int PH = 6 * R * R / NT;     // 24 halo values per thread
        T hv[PH];
#pragma unroll
        for (int m = 0; m < PH; ++m) {
            const int e = tid + m * NT;
            const int f = e >> 8, uv = e & 255, u = uv & 15, v = uv >> 4;
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
            EIK_CHECK(!ex || (nc >= 0 && nc < (int64_t)A.cap), "b2 halo neighbour cell");
            hv[m] = ex ? __ldcg(&Vt[nc * R3 + sa + R * sb + R * R * sd]) : INF;
        }
        using V4 = typename Vec16<T>::type;
        constexpr int EL = 16 / sizeof(T);        // elements per vector
        constexpr int NV = R3 / EL;               // vectors per tile
        constexpr int PV = NV / NT;               // per thread (16 fp32, 32 fp64)
        constexpr int BT = sizeof(T) == 4 ? 8 : 8;
        const V4* Vt4 = reinterpret_cast<const V4*>(Vt + base);
        if constexpr (sizeof(T) == 4) {
            const uint32_t hs = smem_u32(M.H);
            for (int vi = tid; vi < NV; vi += NT) cp_async16(hs + vi * 16, Ht + base + vi * EL);
        } else {
            M.Hg = Ht + base;
        }
        const uint32_t vs = smem_u32(M.V);
#pragma unroll
        for (int m0 = 0; m0 < PV; m0 += BT) {
            V4 va[BT];
#pragma unroll
            for (int m = 0; m < BT; ++m) va[m] = __ldcg(&Vt4[tid + (m0 + m) * NT]);
#pragma unroll
            for (int m = 0; m < BT; ++m) {
                const int vi = tid + (m0 + m) * NT;
                const int e = vi * EL, a = e & 15, b = (e >> 4) & 15, d = e >> 8;
                const uint32_t qa = vs + (uint32_t)b2q(a, b, d) * sizeof(T);
                if constexpr (sizeof(T) == 4) {
                    Pair<T>::st(qa, va[m].x, va[m].y);
                    Pair<T>::st(qa + 8, va[m].z, va[m].w);
                } else {
                    Pair<T>::st(qa, va[m].x, va[m].y);
                }
            }
        }
#pragma unroll
        for (int m = 0; m < PH; ++m) {
            const int e = tid + m * NT;
            const int f = e >> 8, uv = e & 255, u = uv & 15, v = uv >> 4;
            int q;
            switch (f) {
            case 0: q = b2q(-1, u, v); break;
            case 1: q = b2q(R, u, v); break;
            case 2: q = b2q(u, -1, v); break;
            case 3: q = b2q(u, R, v); break;
            case 4: q = b2q(u, v, -1); break;
            default: q = b2q(u, v, R); break;
            }
            M.V[q] = hv[m];
        }
        uint32_t* f32 = reinterpret_cast<uint32_t*>(M.fl);
        const uint32_t fill = init ? 0x01010101u : 0u;
        for (int w = tid; w < B2::NB3 / 4; w += NT) {
            f32[w] = fill;
            reinterpret_cast<uint32_t*>(M.chg)[w] = 0u;
        }
        if (tid == 0) M.fl[B2::FL_DUMMY] = 0;
        cp_async_wait_all();
    }
    __syncthreads();
    if (tid == 0) S.tm[1] = (uint32_t)clock64();
    // ---- initial activity: every block (INIT), otherwise the blocks holding a point of an
    // inflow face whose outside neighbour is smaller (only smaller neighbours enter Eq. (2),
    // P:131) ----
    if (!init && (flags & 63u)) {
        for (int e = tid; e < 6 * R * R; e += NT) {
            const int f = e >> 8;
            if (!(flags & (1u << f))) continue;
            const int uv = e & 255, u = uv & 15, v = uv >> 4;
            int a, b, d, q, qo;
            switch (f) {
            case 0: a = 0; b = u; d = v; qo = b2q(-1, b, d); break;
            case 1: a = R - 1; b = u; d = v; qo = b2q(R, b, d); break;
            case 2: a = u; b = 0; d = v; qo = b2q(a, -1, d); break;
            case 3: a = u; b = R - 1; d = v; qo = b2q(a, R, d); break;
            case 4: a = u; b = v; d = 0; qo = b2q(a, b, -1); break;
            default: a = u; b = v; d = R - 1; qo = b2q(a, b, R); break;
            }
            q = b2q(a, b, d);
            if (M.V[qo] < M.V[q]) M.fl[(a >> 1) + 8 * (b >> 1) + 64 * (d >> 1)] = 1;
        }
        __syncthreads();
    }
    if (tid == 0) S.tm[3] = (uint32_t)clock64();

    // ---- sweeps ----
    int gi = 0, lf0 = -64, lf1 = -64, lf2 = -64;
    const int dir0 = (init || !(flags & 63u)) ? 0 :
        (((flags & 2u) && !(flags & 1u) ? 1 : 0) | ((flags & 8u) && !(flags & 4u) ? 2 : 0) |
         ((flags & 32u) && !(flags & 16u) ? 4 : 0));
    int prev_dir = -1;
    uint32_t nsweeps = 0, nupd = 0, nwr = 0, nsteps = 0;
    const uint2* tab = A.tab_b2;
    for (int sw = 0;; ++sw) {
        int dir;
        {
            const uint32_t gray = 0x45762310u;
            const uint32_t bw = sw > 0 ? S.bwd[(sw - 1) & 1] : 0u;
            if (prev_dir < 0) {
                dir = dir0;
                if (init || !(flags & 63u)) gi = 1;
            } else if (bw) {
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
            prev_dir = dir;
        }
        // active block planes of this direction
        const long long tm0 = tid == 0 ? clock64() : 0;
        if (tid == 0) { S.bwd[sw & 1] = 0; S.plane[sw & 1] = 0; }
        uint32_t pm = 0;
        {
            const uint32_t mx = (dir & 1) ? 7u : 0u, my = (dir & 2) ? 7u : 0u, mz = (dir & 4) ? 7u : 0u;
            const uint32_t w = reinterpret_cast<const uint32_t*>(M.fl)[tid * 2];
            const uint32_t w2 = reinterpret_cast<const uint32_t*>(M.fl)[tid * 2 + 1];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t byte = ((k < 4 ? w : w2) >> (8 * (k & 3))) & 0xffu;
                const uint32_t e = (uint32_t)(tid * 8 + k);
                if (byte) pm |= 1u << (((e & 7u) ^ mx) + (((e >> 3) & 7u) ^ my) + ((e >> 6) ^ mz));
            }
        }
        __syncthreads();   // S.bwd / S.plane reset visible; every flag read
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) pm |= __shfl_xor_sync(0xffffffffu, pm, o);
        if ((tid & 31) == 0 && pm) atomicOr(reinterpret_cast<uint32_t*>(&S.plane[sw & 1]), pm);
        __syncthreads();
        pm = (uint32_t)S.plane[sw & 1];
        if (tid == 0) S.tm[4] += (uint32_t)(clock64() - tm0);
        if (pm == 0u) break;
        ++nsweeps;
        const long long tm1 = tid == 0 ? clock64() : 0;
        uint32_t bwd = sweep_b2<T>(M, tab, pm, dir, nupd, nwr, nsteps);
        if (tid == 0) S.tm[5] += (uint32_t)(clock64() - tm1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bwd |= __shfl_xor_sync(0xffffffffu, bwd, o);
        if ((tid & 31) == 0 && bwd) atomicOr(&S.bwd[sw & 1], bwd);
        __syncthreads();
    }
    if (tid == 0) S.tm[7] = (uint32_t)clock64();
    // ---- face summaries (Eq. (3)): face f is currently downwind iff a border point
    // changed in this processing and ended below its outside neighbour (the staged halo value,
    // an upper bound of the current one: P:718 redundant tags are harmless); the cell key
    // candidate is the smallest such value (A_new of Eq. (3)) ----
    {
        for (int f = 0; f < 6; ++f) {
            uint32_t fm = KEY_INF, fx = 0u;
            for (int uv = tid; uv < R * R; uv += NT) {
                const int u = uv & 15, v = uv >> 4;
                int a, b, d, qo;
                switch (f) {
                case 0: a = 0; b = u; d = v; qo = b2q(-1, b, d); break;
                case 1: a = R - 1; b = u; d = v; qo = b2q(R, b, d); break;
                case 2: a = u; b = 0; d = v; qo = b2q(a, -1, d); break;
                case 3: a = u; b = R - 1; d = v; qo = b2q(a, R, d); break;
                case 4: a = u; b = v; d = 0; qo = b2q(a, b, -1); break;
                default: a = u; b = v; d = R - 1; qo = b2q(a, b, R); break;
                }
                const uint32_t bit = (uint32_t)((a & 1) + 2 * (b & 1) + 4 * (d & 1));
                if ((M.chg[(a >> 1) + 8 * (b >> 1) + 64 * (d >> 1)] >> bit) & 1u) {
                    const T val = M.V[b2q(a, b, d)];
                    if (val < M.V[qo]) {
                        fm = min(fm, key_bits(val));
                        fx = max(fx, key_bits(val));
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                fm = min(fm, __shfl_xor_sync(0xffffffffu, fm, o));
                fx = max(fx, __shfl_xor_sync(0xffffffffu, fx, o));
            }
            if ((tid & 31) == 0 && fm != KEY_INF) {
                atomicMin(&S.face_min[f], fm);
                atomicOr(&S.face_flag, 1u << f);
                if (A.legacy_key) atomicMax(&S.face_max[f], fx);
            }
        }
    }
    // ---- write back: 16-byte vectors holding a changed point (unchanged values are
    // rewritten identically) ----
    unsigned long long nw = 0;
    {
        using V4 = typename Vec16<T>::type;
        constexpr int EL = 16 / sizeof(T);
        constexpr int NV = R3 / EL;
        V4* Vt4 = reinterpret_cast<V4*>(Vt + base);
        const uint32_t vs = smem_u32(M.V);
        for (int vi = tid; vi < NV; vi += NT) {
            const int e = vi * EL, a = e & 15, b = (e >> 4) & 15, d = e >> 8;
            const int sh = 2 * (b & 1) + 4 * (d & 1);
            const int blk = (a >> 1) + 8 * (b >> 1) + 64 * (d >> 1);
            uint32_t m = (M.chg[blk] >> sh) & 3u;
            if constexpr (sizeof(T) == 4) m |= ((M.chg[blk + 1] >> sh) & 3u) << 2;
            if (m) {
                V4 out;
                const uint32_t qa = vs + (uint32_t)b2q(a, b, d) * sizeof(T);
                if constexpr (sizeof(T) == 4) {
                    Pair<T>::ld(qa, out.x, out.y);
                    Pair<T>::ld(qa + 8, out.z, out.w);
                } else {
                    Pair<T>::ld(qa, out.x, out.y);
                }
                __stcg(&Vt4[vi], out);
                nw += __popc(m);
            }
        }
    }
    if (A.stats) {
        unsigned long long u64 = nupd, w64 = nwr;
        for (int o = 16; o > 0; o >>= 1) {
            u64 += __shfl_xor_sync(0xffffffffu, u64, o);
            w64 += __shfl_xor_sync(0xffffffffu, w64, o);
            nw += __shfl_xor_sync(0xffffffffu, nw, o);
        }
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
        atomicAdd(&A.ctl->dbg[37], (unsigned long long)S.tm[4]);
        atomicAdd(&A.ctl->dbg[38], (unsigned long long)S.tm[5]);
        atomicAdd(&A.ctl->dbg[39], (unsigned long long)(uint32_t)((uint32_t)clock64() - S.tm[7]));
        atomicAdd(&A.ctl->dbg[2], (unsigned long long)nsteps);
    }
}

}  // namespace eik
