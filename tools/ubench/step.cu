// Microbenchmark of one wavefront plane step (1 CTA of 256 threads, 46 steps x reps).
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1306_4743_b200/csrc/eik_kernels.cuh"
using namespace eik;

__device__ __forceinline__ float sqrt_approx(float x) { float r; asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }
__device__ __forceinline__ float solve_approx(float mx, float my, float mz, float hf)
{
    const float lo = fminf(mx, my), hi = fmaxf(mx, my);
    const float a1 = fminf(lo, mz), a3 = fmaxf(hi, mz), a2 = fmaxf(lo, fminf(hi, mz));
    const float d2 = fminf(a2 - a1, hf), d3 = fminf(a3 - a1, hf), hh = hf * hf;
    const float t2 = (d2 + sqrt_approx(fmaxf(2.f * hh - d2 * d2, 0.f))) * 0.5f;
    const float e = d3 - d2;
    const float t3 = (d2 + d3 + sqrt_approx(fmaxf(3.f * hh - (d2 * d2 + d3 * d3 + e * e), 0.f))) * (1.f / 3.f);
    float t = hf;
    if (hf > d2) t = (t2 > d3) ? t3 : t2;
    return a1 + t;
}

template <int V>
__global__ void k_stepb(float* out, long long* cyc, int reps)
{
    constexpr int R = 16, RP = 18, RP2 = RP * RP, NCOL = 256;
    __shared__ float sV[RP * RP * RP];
    __shared__ float sH[4096];
    __shared__ uint8_t sA[4096];
    const int tid = threadIdx.x, ci = tid % R, cj = tid / R;
    for (int e = tid; e < 4096; e += 256) sH[e] = 0.01f;
    float acc = 0;
    const int qcol = (ci + 1) + RP * (cj + 1);
    const int pbase = ci + cj;
    long long tsum = 0;
    bool fwd = false;
    const float INF = __int_as_float(0x7f800000);
    for (int rep = 0; rep < reps; ++rep) {
        for (int e = tid; e < RP * RP * RP; e += 256) {
            const int a = e % RP, b = (e / RP) % RP, c = e / (RP * RP);
            sV[e] = (a == 0 || b == 0 || c == 0) ? 0.f : INF;
        }
        for (int e = tid; e < 4096; e += 256) sA[e] = 1;
        __syncthreads();
        long long t0 = clock64();
        for (int s = 0; s < 46; ++s) {
            bool myfwd = false;
            const int k = s - pbase;
            if (k >= 0 && k < R) {
                const int p = tid + NCOL * k;
                if (sA[p]) {
                    sA[p] = 0;
                    const int q = qcol + RP2 * (k + 1);
                    const float hf = sH[p];
                    const float v = sV[q];
                    const float xm = sV[q - 1], xp = sV[q + 1], ym = sV[q - RP], yp = sV[q + RP];
                    const float zm = sV[q - RP2], zp = sV[q + RP2];
                    const float mx = fminf(xm, xp), my = fminf(ym, yp), mz = fminf(zm, zp);
                    const float u = V == 7 ? solve_approx(mx, my, mz, hf) : local_solve_par<float>(mx, my, mz, hf);
                    if (u < v) {
                        sV[q] = u;
                        if (xm > u && ci > 0) { sA[p - 1] = 1; }
                        if (xp > u && ci < R - 1) { sA[p + 1] = 1; myfwd = true; }
                        if (ym > u && cj > 0) { sA[p - R] = 1; }
                        if (yp > u && cj < R - 1) { sA[p + R] = 1; myfwd = true; }
                        if (zm > u && k > 0) { sA[p - NCOL] = 1; }
                        if (zp > u && k < R - 1) { sA[p + NCOL] = 1; myfwd = true; }
                    }
                    acc += u;
                }
            }
            fwd = __syncthreads_or(myfwd);
        }
        tsum += clock64() - t0;
        __syncthreads();
    }
    if (tid == 0) cyc[0] = tsum / ((long long)reps * 46);
    out[tid] = acc + fwd;
}

template <int V>
__global__ void k_step(float* out, long long* cyc, int reps)
{
    constexpr int R = 16, RP = 18, RP2 = RP * RP, NCOL = 256;
    __shared__ float sV[RP * RP * RP];
    __shared__ float sH[4096];
    __shared__ uint32_t act[NCOL];
    const int tid = threadIdx.x, ci = tid % R, cj = tid / R;
    for (int e = tid; e < 4096; e += 256) sH[e] = 0.01f;
    float acc = 0;
    const int qcol = (ci + 1) + RP * (cj + 1);
    const int pbase = ci + cj;
    long long tsum = 0;
    bool fwd = false;
    const float INF = __int_as_float(0x7f800000);
    for (int rep = 0; rep < reps; ++rep) {
        // reset: interior +inf, the three lower halo faces 0 (a front enters from the corner side)
        for (int e = tid; e < RP * RP * RP; e += 256) {
            const int a = e % RP, b = (e / RP) % RP, c = e / (RP * RP);
            sV[e] = (a == 0 || b == 0 || c == 0) ? 0.f : INF;
        }
        act[tid] = 0xffffu;
        __syncthreads();
        long long t0 = clock64();
        for (int s = 0; s < 46; ++s) {
            bool myfwd = false;
            const int k = s - pbase;
            if (V >= 1 && k >= 0 && k < R) {
                const uint32_t bit = 1u << k;
                if (V == 1) { myfwd = (act[tid] & bit) != 0; }
                if (V >= 2 && (act[tid] & bit)) {
                    if (V >= 4) atomicAnd(&act[tid], ~bit);
                    const int q = qcol + RP2 * (k + 1);
                    const float hf = sH[tid + NCOL * k];
                    const float v = sV[q];
                    const float xm = sV[q - 1], xp = sV[q + 1], ym = sV[q - RP], yp = sV[q + RP];
                    const float zm = sV[q - RP2], zp = sV[q + RP2];
                    const float mx = fminf(xm, xp), my = fminf(ym, yp), mz = fminf(zm, zp);
                    float u;
                    if (V >= 3) u = local_solve_par<float>(mx, my, mz, hf);
                    else u = fminf(mx, fminf(my, mz)) + hf;
                    if (u < v) {
                        sV[q] = u * 0.999f;
                        if (V >= 4) {
                            if (xm > u && ci > 0) { atomicOr(&act[tid - 1], bit); myfwd = true; }
                            if (xp > u && ci < R - 1) { atomicOr(&act[tid + 1], bit); myfwd = true; }
                            if (ym > u && cj > 0) { atomicOr(&act[tid - R], bit); myfwd = true; }
                            if (yp > u && cj < R - 1) { atomicOr(&act[tid + R], bit); myfwd = true; }
                            if (zm > u && k > 0) { atomicOr(&act[tid], bit >> 1); }
                            if (zp > u && k < R - 1) { atomicOr(&act[tid], bit << 1); myfwd = true; }
                        }
                    }
                    acc += u;
                }
            }
            if (V == 5) { __syncthreads(); fwd = fwd ^ myfwd; }
            else fwd = __syncthreads_or(myfwd);
        }
        tsum += clock64() - t0;
        __syncthreads();
    }
    if (tid == 0) cyc[0] = tsum / ((long long)reps * 46);
    out[tid] = acc + fwd;
}

int main()
{
    float* out; long long* cyc; long long h;
    cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8);
    const char* names[] = {"barrier_or only", "+act bit test", "+7 LDS + cheap solve + STS", "+real solve", "+atomics", "plain syncthreads"};
#define RUN(V) { k_step<V><<<1, 256>>>(out, cyc, 200); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("V%d %-30s %lld cycles/step\n", V, names[V], h); }
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5)
    k_stepb<6><<<1, 256>>>(out, cyc, 200); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("V6 byte flags, IEEE sqrt         %lld cycles/step\n", h);
    k_stepb<7><<<1, 256>>>(out, cyc, 200); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("V7 byte flags, approx sqrt       %lld cycles/step\n", h);
    k_stepb<6><<<148*4, 256>>>(out, cyc, 200); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("V6 x 4 CTAs/SM                   %lld cycles/step\n", h);
    // many CTAs per SM
    printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
