// Shared-memory wavefronts of warp-wide LDS.64 / LDS.32 for given lane address patterns
// (measure under ncu: l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum per launch).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void k64(const int* __restrict__ pat, int iters, float* out) {
    __shared__ float2 buf[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_float2(i, -i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = pat[q * 32 + lane];
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            float2 v = buf[(a[q] + it * 0) & 1023];
            acc += v.x + v.y;
            a[q] ^= (int)(acc == 12345.f);   // keep loads live and in order
        }
    }
    if (acc == 1.f) out[0] = acc;
}
__global__ void k32(const int* __restrict__ pat, int iters, float* out) {
    __shared__ float buf[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    int a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = pat[q * 32 + lane];
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            acc += buf[a[q] & 2047];
            a[q] ^= (int)(acc == 12345.f);
        }
    }
    if (acc == 1.f) out[0] = acc;
}

int main() {
    int* dpat;
    float* dout;
    cudaMalloc(&dpat, 8 * 32 * sizeof(int));
    cudaMalloc(&dout, 4);
    std::vector<int> p(256);
    srand(1);
    auto run = [&](const char* name, bool is64) {
        cudaMemcpy(dpat, p.data(), 256 * 4, cudaMemcpyHostToDevice);
        if (is64) k64<<<1, 32>>>(dpat, 100, dout); else k32<<<1, 32>>>(dpat, 100, dout);
        cudaDeviceSynchronize();
        printf("%s done\n", name);
    };
    // 1 stride-1
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = l;
    run("64_stride1", true);
    // 2 random over 0..128 (distinct per instruction not required)
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = rand() % 129;
    run("64_random129", true);
    // 3 half-warp discriminator: lanes 0-7 -> 0..7, 8-15 -> 16..23, 16-23 -> 8..15, 24-31 -> 24..31
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) {
        int g = l / 8, r = l % 8;
        int base = g == 0 ? 0 : g == 1 ? 16 : g == 2 ? 8 : 24;
        p[q * 32 + l] = base + r;
    }
    run("64_halfwarp_test", true);
    // 4 all same address (broadcast)
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = 128;
    run("64_broadcast", true);
    // 5 16 lanes same bank pair distinct addresses
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = (l % 16) * 16 + (l / 16);
    run("64_16way", true);
    // 6 the swizzled pairing: lanes l and l+16 share bank pair, others distinct
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = (l < 16) ? l : 16 + (l - 16);
    run("64_pairs_l_l16", true);
    // 7 lanes 0..15 -> pairs 0..15; lanes 16..31 -> same pairs 0..15 but +32 (distinct addr)
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = (l % 16) + (l / 16) * 32;
    run("64_two_per_pair_cross_half", true);
    // 8 lanes 2k,2k+1 share a bank pair (distinct addresses): within-half conflicts of 2
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = (l / 2) + (l % 2) * 32;
    run("64_two_per_pair_within_half", true);
    // 32-bit
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = l;
    run("32_stride1", false);
    for (int q = 0; q < 8; ++q) for (int l = 0; l < 32; ++l) p[q * 32 + l] = rand() % 257;
    run("32_random257", false);
    return 0;
}
