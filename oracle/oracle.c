/*
 * oracle.c -- CPU reference ("oracle") for the pHCM hot path of arXiv 1306.4743.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing on the product path (paper_1306_4743_b200/, include/)
 * may include, link or call this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header, table or
 * constant with the CUDA path: the only thing both sides share is the *formula* of the local
 * solve, written out independently on each side.
 *
 * Everything is plain, serial, fp64, built with -O3 -ffp-contract=off (no FMA contraction,
 * no fast-math), so that a reader can check it against the paper by eye.
 *
 * Layout: lexicographic, i fastest, idx = i + (n+1)*(j + (n+1)*k).
 *
 * Functions and the passage each follows:
 *   orc_solve_local      Eq. (2) solved for U_ijk given the per-axis minima of
 *                        the neighbour values: sorted 1/2/3-sided quadratic in the shifted
 *                        variable t = U - a1, keep the largest consistent k (C.3,
 *                        readings R1-R4).  Pinned by: S:125-128 worked examples, the closed
 *                        forms of SURVEY C.5, the plug-in residual of Eq. (2) and the
 *                        independent descending-k textbook form (tests/test_oracle_local.py).
 *   orc_fmm              the Fast Marching Method: binary min-heap of TRIAL
 *                        points, accept the smallest, update not-yet-accepted neighbours from
 *                        ACCEPTED neighbours only (R16).  Pinned by value iteration on tiny
 *                        grids, closed forms (axis d*h, W table, plane wave), BFS masks.
 *   orc_value_iteration  the literal definition (C.1): Jacobi iteration of Eq. (2),
 *                        V <- min(V, solve(minima(V))) at every non-exit F > 0 point, from
 *                        V = q on Q', +inf elsewhere, until nothing changes.
 *   orc_bfs              reachability: 6-connected BFS from the exits through non-exit
 *                        F > 0 points (the finite-iff-reachable contract, C.6, R11).
 *   orc_check            invariant checkers on any candidate solution U (C.5/C.6):
 *                        Eq. (2) residual, discrete Lipschitz bound, causal parent.
 *   orc_fsm              the Fast Sweeping Method: Gauss-Seidel sweeps of Eq. (2)
 *                        in the 2^3 standard loop orderings, alternated, until a sweep changes
 *                        nothing; with lsm = 1 the Locking Sweeping Method: a point
 *                        is updated only while "active" (initially the neighbours of the exit
 *                        set; a change activates the neighbours).  Pinned by: the paper's sweep
 *                        count of Ex. 1 (9 at every M, Table 4), LSM = FSM sweeps and
 *                        values, the FSM fixed point = FMM / value iteration on random
 *                        grids (tests/test_oracle_fsm.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_INF (1.0 / 0.0)

/* ---------------------------------------------------------------------------------------
 * Local solve of Eq. (2) for U at one gridpoint.
 *   Given hf = h/F > 0 and the per-axis minima mx, my, mz (each may be +inf):
 *     a1 <= a2 <= a3 = sort(mx, my, mz)
 *     one-sided:   U = a1 + hf                                     (R2)
 *     two-sided:   (U-a1)^2 + (U-a2)^2 = hf^2, used iff hf > a2-a1    (R4: strict >)
 *     three-sided: sum_d (U-a_d)^2 = hf^2, used iff t2 > a3-a1
 *   in the shifted variable t = U - a1 with d2 = a2-a1, d3 = a3-a1:
 *     2-sided: 2t^2 - 2 d2 t + d2^2 - hf^2 = 0  ->  t = (d2 + sqrt(2hf^2 - d2^2)) / 2
 *     3-sided: 3t^2 - 2(d2+d3) t + d2^2 + d3^2 - hf^2 = 0
 *              -> t = (d2 + d3 + sqrt((d2+d3)^2 - 3(d2^2+d3^2-hf^2))) / 3
 *                 with (d2+d3)^2 - 3(d2^2+d3^2) = -(d2^2 + d3^2 + (d3-d2)^2) ... (expanded:
 *                 d2^2+2d2d3+d3^2-3d2^2-3d3^2 = -2d2^2-2d3^2+2d2d3 = -(d2^2+d3^2+(d3-d2)^2))
 *   A negative discriminant from rounding is clamped to 0 (R3).
 * ------------------------------------------------------------------------------------- */
double orc_solve_local(double mx, double my, double mz, double hf)
{
    double a1 = mx, a2 = my, a3 = mz, tmp;
    if (a1 > a2) { tmp = a1; a1 = a2; a2 = tmp; }
    if (a2 > a3) { tmp = a2; a2 = a3; a3 = tmp; }
    if (a1 > a2) { tmp = a1; a1 = a2; a2 = tmp; }
    if (a1 == ORC_INF) return ORC_INF;

    double t = hf;                       /* k = 1: U = a1 + h/F */
    double d2 = a2 - a1;
    if (t > d2) {                        /* k = 2 consistent only if U_1 > a2 */
        double disc = 2.0 * hf * hf - d2 * d2;
        if (disc < 0.0) disc = 0.0;
        t = (d2 + sqrt(disc)) / 2.0;
        double d3 = a3 - a1;
        if (t > d3) {                    /* k = 3 consistent only if U_2 > a3 */
            double disc3 = 3.0 * hf * hf - (d2 * d2 + d3 * d3 + (d3 - d2) * (d3 - d2));
            if (disc3 < 0.0) disc3 = 0.0;
            t = (d2 + d3 + sqrt(disc3)) / 3.0;
        }
    }
    return a1 + t;
}

/* ------------------------------------------------------------------------------------- */
typedef struct { int64_t n1, M; } grid_t;

static inline int64_t gidx(const grid_t* g, int64_t i, int64_t j, int64_t k)
{
    return i + g->n1 * (j + g->n1 * k);
}

/* per-axis minimum of the two axis neighbours; a missing neighbour is +inf (R7) */
static void axis_minima(const grid_t* g, const double* V, int64_t p, double m[3])
{
    int64_t n1 = g->n1;
    int64_t i = p % n1, j = (p / n1) % n1, k = p / (n1 * n1);
    double lo, hi;
    lo = (i > 0) ? V[p - 1] : ORC_INF;
    hi = (i < n1 - 1) ? V[p + 1] : ORC_INF;
    m[0] = lo < hi ? lo : hi;
    lo = (j > 0) ? V[p - n1] : ORC_INF;
    hi = (j < n1 - 1) ? V[p + n1] : ORC_INF;
    m[1] = lo < hi ? lo : hi;
    lo = (k > 0) ? V[p - n1 * n1] : ORC_INF;
    hi = (k < n1 - 1) ? V[p + n1 * n1] : ORC_INF;
    m[2] = lo < hi ? lo : hi;
}

/* up to 6 neighbour indices of p; returns count */
static int neighbours(const grid_t* g, int64_t p, int64_t nb[6])
{
    int64_t n1 = g->n1;
    int64_t i = p % n1, j = (p / n1) % n1, k = p / (n1 * n1);
    int c = 0;
    if (i > 0) nb[c++] = p - 1;
    if (i < n1 - 1) nb[c++] = p + 1;
    if (j > 0) nb[c++] = p - n1;
    if (j < n1 - 1) nb[c++] = p + n1;
    if (k > 0) nb[c++] = p - n1 * n1;
    if (k < n1 - 1) nb[c++] = p + n1 * n1;
    return c;
}

/* ---------------------------------------------------------------------------------------
 * Fast Marching Method.  Binary min-heap keyed on V, with a
 * back-pointer array for decrease-key.  Returns 0 on success, 1 if the accepted values were
 * ever decreasing by more than rounding (S:213 assertion), 2 on allocation failure, 3 if
 * M >= 2^31.
 * n_accepted (optional) receives the number of accepted points.
 * ------------------------------------------------------------------------------------- */
enum { FAR = 0, TRIAL = 1, ACCEPTED = 2 };

typedef struct {
    int32_t* a;      /* heap of point ids */
    int64_t size;
    int32_t* pos;    /* pos[p] = heap slot of p while TRIAL */
    const double* V;
} heap_t;

static void heap_swap(heap_t* h, int64_t x, int64_t y)
{
    int32_t px = h->a[x], py = h->a[y];
    h->a[x] = py; h->a[y] = px;
    h->pos[py] = (int32_t)x; h->pos[px] = (int32_t)y;
}

static void sift_up(heap_t* h, int64_t s)
{
    while (s > 0) {
        int64_t parent = (s - 1) / 2;
        if (h->V[h->a[parent]] <= h->V[h->a[s]]) break;
        heap_swap(h, s, parent);
        s = parent;
    }
}

static void sift_down(heap_t* h, int64_t s)
{
    for (;;) {
        int64_t l = 2 * s + 1, r = l + 1, m = s;
        if (l < h->size && h->V[h->a[l]] < h->V[h->a[m]]) m = l;
        if (r < h->size && h->V[h->a[r]] < h->V[h->a[m]]) m = r;
        if (m == s) break;
        heap_swap(h, s, m);
        s = m;
    }
}

static void heap_push(heap_t* h, int32_t p)
{
    h->a[h->size] = p;
    h->pos[p] = (int32_t)h->size;
    h->size++;
    sift_up(h, h->size - 1);
}

static int32_t heap_pop(heap_t* h)
{
    int32_t top = h->a[0];
    h->size--;
    if (h->size > 0) {
        h->a[0] = h->a[h->size];
        h->pos[h->a[0]] = 0;
        sift_down(h, 0);
    }
    return top;
}

int orc_fmm(int64_t n, double h, const double* F, const uint8_t* mask, const double* q,
            double* V, int64_t* n_accepted)
{
    grid_t g = { n + 1, (n + 1) * (n + 1) * (n + 1) };
    if (g.M >= ((int64_t)1 << 31)) return 3;
    uint8_t* state = (uint8_t*)calloc((size_t)g.M, 1);
    heap_t hp;
    hp.a = (int32_t*)malloc((size_t)g.M * sizeof(int32_t));
    hp.pos = (int32_t*)malloc((size_t)g.M * sizeof(int32_t));
    hp.size = 0;
    hp.V = V;
    if (!state || !hp.a || !hp.pos) { free(state); free(hp.a); free(hp.pos); return 2; }

    /* initialisation: V = q on Q', +inf elsewhere; exits are TRIAL (C.2 step 1) */
    for (int64_t p = 0; p < g.M; ++p) V[p] = ORC_INF;
    for (int64_t p = 0; p < g.M; ++p)
        if (mask[p]) { V[p] = q[p]; state[p] = TRIAL; heap_push(&hp, (int32_t)p); }

    int status = 0;
    int64_t acc = 0;
    double last = -ORC_INF;
    while (hp.size > 0) {
        int32_t p = heap_pop(&hp);                       /* C.2 step 2 */
        state[p] = ACCEPTED;
        acc++;
        /* pops are non-decreasing in exact arithmetic; at the switching tie of R4
           (hf barely > a2 - a1) rounding can place a two-sided value an ulp below a2, so a
           decrease is only an error beyond 64 ulp */
        if (V[p] < last - 64.0 * 2.220446049250313e-16 * last) status = 1;
        if (V[p] > last) last = V[p];
        int64_t nb[6];
        int c = neighbours(&g, p, nb);
        for (int e = 0; e < c; ++e) {                    /* C.2 step 3 */
            int64_t r = nb[e];
            if (state[r] == ACCEPTED || mask[r] || !(F[r] > 0.0)) continue;
            /* minima over ACCEPTED neighbours only (R16) */
            int64_t n1 = g.n1;
            int64_t i = r % n1, j = (r / n1) % n1, k = r / (n1 * n1);
            double m[3] = { ORC_INF, ORC_INF, ORC_INF };
            int64_t off[3] = { 1, n1, n1 * n1 };
            int64_t co[3] = { i, j, k };
            for (int d = 0; d < 3; ++d) {
                if (co[d] > 0 && state[r - off[d]] == ACCEPTED && V[r - off[d]] < m[d])
                    m[d] = V[r - off[d]];
                if (co[d] < n1 - 1 && state[r + off[d]] == ACCEPTED && V[r + off[d]] < m[d])
                    m[d] = V[r + off[d]];
            }
            double u = orc_solve_local(m[0], m[1], m[2], h / F[r]);
            if (u < V[r]) {
                V[r] = u;
                if (state[r] == FAR) { state[r] = TRIAL; heap_push(&hp, (int32_t)r); }
                else sift_up(&hp, hp.pos[r]);           /* decrease-key */
            }
        }
    }
    if (n_accepted) *n_accepted = acc;
    free(state); free(hp.a); free(hp.pos);
    return status;
}

/* ---------------------------------------------------------------------------------------
 * Value iteration (the literal definition, C.1): Jacobi sweeps of
 *   V_p <- min(V_p, solve(minima(V)))   at every non-exit point with F_p > 0,
 * all points reading the previous iterate, until an iteration changes nothing.
 * Returns the number of iterations performed (the last one changes nothing), or -1 if
 * max_iter was reached, -2 on allocation failure.
 * ------------------------------------------------------------------------------------- */
int64_t orc_value_iteration(int64_t n, double h, const double* F, const uint8_t* mask,
                            const double* q, double* V, int64_t max_iter)
{
    grid_t g = { n + 1, (n + 1) * (n + 1) * (n + 1) };
    double* W = (double*)malloc((size_t)g.M * sizeof(double));
    if (!W) return -2;
    for (int64_t p = 0; p < g.M; ++p) V[p] = mask[p] ? q[p] : ORC_INF;
    int64_t it = 0;
    for (;;) {
        if (it >= max_iter) { free(W); return -1; }
        it++;
        int changed = 0;
        for (int64_t p = 0; p < g.M; ++p) {
            W[p] = V[p];
            if (mask[p] || !(F[p] > 0.0)) continue;
            double m[3];
            axis_minima(&g, V, p, m);
            double u = orc_solve_local(m[0], m[1], m[2], h / F[p]);
            if (u < V[p]) { W[p] = u; changed = 1; }
        }
        memcpy(V, W, (size_t)g.M * sizeof(double));
        if (!changed) break;
    }
    free(W);
    return it;
}

/* ---------------------------------------------------------------------------------------
 * BFS reachability from the exits through non-exit F > 0 points (6-connectivity).
 * reach[p] = 1 iff p is an exit or is connected to one through such points.
 * Returns the number of reachable points, or -1 on allocation failure / M >= 2^31.
 * ------------------------------------------------------------------------------------- */
int64_t orc_bfs(int64_t n, const double* F, const uint8_t* mask, uint8_t* reach)
{
    grid_t g = { n + 1, (n + 1) * (n + 1) * (n + 1) };
    if (g.M >= ((int64_t)1 << 31)) return -1;
    int32_t* queue = (int32_t*)malloc((size_t)g.M * sizeof(int32_t));
    if (!queue) return -1;
    int64_t head = 0, tail = 0;
    memset(reach, 0, (size_t)g.M);
    for (int64_t p = 0; p < g.M; ++p)
        if (mask[p]) { reach[p] = 1; queue[tail++] = (int32_t)p; }
    while (head < tail) {
        int64_t p = queue[head++];
        int64_t nb[6];
        int c = neighbours(&g, p, nb);
        for (int e = 0; e < c; ++e) {
            int64_t r = nb[e];
            if (reach[r] || mask[r] || !(F[r] > 0.0)) continue;
            reach[r] = 1;
            queue[tail++] = (int32_t)r;
        }
    }
    free(queue);
    return tail;
}

/* ---------------------------------------------------------------------------------------
 * Invariant checks on a candidate solution U (fp64 view), per SURVEY C.5/C.6:
 *   out[0] = max |res_p| over finite non-exit F>0 points, res_p = sum_d max(U_p - m_d, 0)^2
 *            / hf_p^2 - 1 (Eq. (2) residual)
 *   out[1] = flat index of that max
 *   out[2] = max over finite non-exit F>0 p and finite axis neighbours r of
 *            (U_p - U_r - hf_p) / hf_p  (discrete Lipschitz bound; <= ~0 at a fixed point)
 *   out[3] = number of finite non-exit points with no neighbour strictly smaller (causal
 *            parent violations)
 *   out[4] = number of finite non-exit F>0 points
 *   out[5] = number of non-exit points with F = 0 whose U is finite (must be 0, R11)
 *   out[6] = number of points where isinf(U) disagrees with the "all minima infinite"
 *            condition (U infinite at a non-exit F>0 point with a finite neighbour, or finite
 *            with all neighbours infinite)
 * ------------------------------------------------------------------------------------- */
void orc_check(int64_t n, double h, const double* F, const uint8_t* mask, const double* U,
               double* out)
{
    grid_t g = { n + 1, (n + 1) * (n + 1) * (n + 1) };
    double res_max = 0.0, res_at = -1.0, lip_max = -ORC_INF;
    int64_t causal_bad = 0, n_fin = 0, f0_finite = 0, inf_bad = 0;
    for (int64_t p = 0; p < g.M; ++p) {
        if (mask[p]) continue;
        double Up = U[p];
        if (!(F[p] > 0.0)) { if (Up != ORC_INF) f0_finite++; continue; }
        double m[3];
        axis_minima(&g, U, p, m);
        double amin = m[0] < m[1] ? m[0] : m[1];
        amin = amin < m[2] ? amin : m[2];
        if (Up == ORC_INF) { if (amin != ORC_INF) inf_bad++; continue; }
        if (amin == ORC_INF) { inf_bad++; continue; }
        n_fin++;
        double hf = h / F[p];
        double s = 0.0;
        for (int d = 0; d < 3; ++d) {
            double e = Up - m[d];
            if (e > 0.0) s += e * e;
        }
        double res = fabs(s / (hf * hf) - 1.0);
        if (res > res_max) { res_max = res; res_at = (double)p; }
        if (!(amin < Up)) causal_bad++;
        int64_t nb[6];
        int c = neighbours(&g, p, nb);
        for (int e = 0; e < c; ++e) {
            double Ur = U[nb[e]];
            if (Ur == ORC_INF) continue;
            double l = (Up - Ur - hf) / hf;
            if (l > lip_max) lip_max = l;
        }
    }
    out[0] = res_max; out[1] = res_at; out[2] = lip_max; out[3] = (double)causal_bad;
    out[4] = (double)n_fin; out[5] = (double)f0_finite; out[6] = (double)inf_bad;
}

/* ---------------------------------------------------------------------------------------
 * Scaled residual for results computed in a lower precision (C.6 "fp32: |res_p| <=
 * 8 ulp32(U_p) / hf_p"): returns max over finite non-exit F>0 points of
 *   |res_p| / (k_ulp * u_unit * (U_p + h) / hf_p),   u_unit = unit roundoff of the run dtype.
 * (U_p + h keeps the bound meaningful at U ~ 0 next to exits.)  Also writes the index.
 * ------------------------------------------------------------------------------------- */
double orc_residual_ratio(int64_t n, double h, const double* F, const uint8_t* mask,
                          const double* U, double u_unit, double k_ulp, int64_t* at)
{
    grid_t g = { n + 1, (n + 1) * (n + 1) * (n + 1) };
    double worst = 0.0;
    int64_t wat = -1;
    for (int64_t p = 0; p < g.M; ++p) {
        if (mask[p] || !(F[p] > 0.0)) continue;
        double Up = U[p];
        if (Up == ORC_INF) continue;
        double m[3];
        axis_minima(&g, U, p, m);
        double hf = h / F[p];
        double s = 0.0;
        for (int d = 0; d < 3; ++d) {
            double e = Up - m[d];
            if (e > 0.0) s += e * e;
        }
        double res = fabs(s / (hf * hf) - 1.0);
        double tol = k_ulp * u_unit * (Up + h) / hf;
        double r = res / tol;
        if (r > worst) { worst = r; wat = p; }
    }
    if (at) *at = wat;
    return worst;
}

/* ---------------------------------------------------------------------------------------
 * Fast Sweeping Method: Gauss-Seidel iteration of
 *   V_p <- min(V_p, solve(minima(V)))   (non-exit points with F_p > 0)
 * over the gridpoints in one of the 2^3 standard loop orderings per sweep ("sweep
 * directions").  Sweep s uses direction d = s mod 8 (bit 0: i descending, bit 1:
 * j descending, bit 2: k descending; k outermost, i innermost).  Sweeps continue as long as
 * some gridpoint received an updated value: the last sweep changes nothing and is
 * counted (Ex. 1 converges in 8 + 1 = 9 sweeps, Table 4).
 * lsm = 1: Locking Sweeping Method: active flags, initially set at the non-exit
 * neighbours of the exit set; a point is relaxed only if active, its flag is cleared when it
 * is relaxed, and a changed value activates its neighbours (a value cannot change unless a
 * neighbour changed since its last update).
 * Returns the number of sweeps, -1 if max_sweeps was reached, -2 on allocation failure;
 * *n_updates (if not NULL) = local solves performed.
 * ------------------------------------------------------------------------------------- */
int64_t orc_fsm(int64_t n, double h, const double* F, const uint8_t* mask, const double* q,
                double* V, int lsm, int64_t max_sweeps, int64_t* n_updates)
{
    grid_t g = { n + 1, (n + 1) * (n + 1) * (n + 1) };
    int64_t n1 = g.n1;
    uint8_t* act = NULL;
    for (int64_t p = 0; p < g.M; ++p) V[p] = mask[p] ? q[p] : ORC_INF;
    if (lsm) {
        act = (uint8_t*)calloc((size_t)g.M, 1);
        if (!act) return -2;
        for (int64_t p = 0; p < g.M; ++p) {
            if (!mask[p]) continue;
            int64_t nb[6];
            int c = neighbours(&g, p, nb);
            for (int a = 0; a < c; ++a) if (!mask[nb[a]]) act[nb[a]] = 1;
        }
    }
    int64_t upd = 0, s = 0;
    for (;;) {
        if (s >= max_sweeps) { free(act); return -1; }
        int d = (int)(s % 8);
        s++;
        int changed = 0;
        for (int64_t kk = 0; kk < n1; ++kk) {
            int64_t k = (d & 4) ? n1 - 1 - kk : kk;
            for (int64_t jj = 0; jj < n1; ++jj) {
                int64_t j = (d & 2) ? n1 - 1 - jj : jj;
                for (int64_t ii = 0; ii < n1; ++ii) {
                    int64_t i = (d & 1) ? n1 - 1 - ii : ii;
                    int64_t p = gidx(&g, i, j, k);
                    if (mask[p] || !(F[p] > 0.0)) continue;
                    if (lsm) {
                        if (!act[p]) continue;
                        act[p] = 0;
                    }
                    double m[3];
                    axis_minima(&g, V, p, m);
                    upd++;
                    double u = orc_solve_local(m[0], m[1], m[2], h / F[p]);
                    if (u < V[p]) {
                        V[p] = u;
                        changed = 1;
                        if (lsm) {
                            int64_t nb[6];
                            int c = neighbours(&g, p, nb);
                            for (int a = 0; a < c; ++a) act[nb[a]] = 1;
                        }
                    }
                }
            }
        }
        if (!changed) break;
    }
    free(act);
    if (n_updates) *n_updates = upd;
    return s;
}
