// Microbenchmark: L2-resident vs HBM read bandwidth on B200 (design input for
// the scan's second-pass placement).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float4* __restrict__ p, size_t n, int reps, float* out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1234.5f) out[0] = acc;
}

int main() {
    size_t maxb = (size_t)4 << 30;
    float4* p;
    float* o;
    cudaMalloc(&p, maxb);
    cudaMalloc(&o, 4);
    cudaMemset(p, 0, maxb);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    size_t sizes[] = {(size_t)8 << 20, (size_t)16 << 20, (size_t)32 << 20, (size_t)48 << 20, (size_t)64 << 20,
                      (size_t)96 << 20, (size_t)128 << 20, (size_t)256 << 20, (size_t)1 << 30, (size_t)4 << 30};
    for (size_t bytes : sizes) {
        size_t n = bytes / 16;
        int reps = (int)((size_t(8) << 30) / bytes);
        if (reps < 2) reps = 2;
        rd<<<148 * 8, 512>>>(p, n, 1, o);
        cudaEventRecord(a);
        rd<<<148 * 8, 512>>>(p, n, reps, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("bytes=%8zu MB reps=%4d  read GB/s = %.1f\n", bytes >> 20, reps, (double)bytes * reps / (ms * 1e6));
    }
    return 0;
}
