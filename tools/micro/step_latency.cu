// Per-step latency floor of a CTA-wide barrier recurrence (128 threads):
//   v = f(h); buf[par][i] = v; __syncthreads(); h = sum_q buf[par][src_q] + b
#include <cstdio>
#include <cuda_runtime.h>

template <int NQ, int EXTRA>
__global__ void k(const int* __restrict__ srcs, float* out, long long* cyc, int steps) {
    __shared__ float2 buf[2][129];
    const int i = threadIdx.x;
    int src[4];
    for (int q = 0; q < 4; ++q) src[q] = srcs[q * 128 + i];
    if (i == 0) { buf[0][128] = make_float2(0, 0); buf[1][128] = make_float2(0, 0); }
    float hr = i, hi = -i, er = 0.f;
    __syncthreads();
    long long t0 = clock64();
    for (int t = 0; t < steps; ++t) {
        const int par = t & 1;
        buf[par][i] = make_float2(0.9f * hr - 0.1f * hi, 0.9f * hi + 0.1f * hr);
        __syncthreads();
        float2 v[NQ > 0 ? NQ : 1];
#pragma unroll
        for (int q = 0; q < NQ; ++q) v[q] = buf[par][src[q]];
        float ar = 0.f, ai = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) { ar += v[q].x; ai += v[q].y; }
#pragma unroll
        for (int x = 0; x < EXTRA; ++x) er = er * 1.0001f + (float)x;   // independent filler
        hr = ar + 0.5f;
        hi = ai - 0.5f;
    }
    long long t1 = clock64();
    if (i == 0) cyc[blockIdx.x] = (t1 - t0) / steps;
    out[blockIdx.x * 128 + i] = hr + hi + er;
}

int main() {
    int h[512];
    for (int q = 0; q < 4; ++q) for (int i = 0; i < 128; ++i) h[q * 128 + i] = (i * 37 + q * 11) % 129;
    int* d; float* o; long long* c;
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 148 * 128 * 4); cudaMalloc(&c, 148 * 8);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    long long hc[148];
#define RUN(NQ, EX) k<NQ, EX><<<128, 128>>>(d, o, c, 4096); cudaDeviceSynchronize(); cudaMemcpy(hc, c, 8 * 128, cudaMemcpyDeviceToHost); printf("NQ=%d EXTRA=%d cycles/step %lld\n", NQ, EX, hc[0]);
    RUN(0, 0) RUN(1, 0) RUN(2, 0) RUN(4, 0) RUN(4, 20) RUN(4, 40) RUN(4, 80)
    return 0;
}
