// Copy-kernel design sweep (not part of the library): 1 GiB device copy,
// variants of the LSU and TMA bulk paths, CUDA-event timed, best of 10.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint4 ld_nc(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void st_na(void* p, uint4 v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
template <int U, int UNIT>
__global__ void lsu_persistent(const char* __restrict__ s, char* __restrict__ d, uint64_t n) {
    const uint64_t units = n / UNIT;
    for (uint64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const char* src = s + u * UNIT;
        char* dst = d + u * UNIT;
        const uint32_t nv = UNIT / 16;
        for (uint32_t i = threadIdx.x; i < nv; i += U * blockDim.x) {
            uint4 v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) v[k] = ld_nc(src + 16ull * (i + k * blockDim.x));
#pragma unroll
            for (int k = 0; k < U; ++k) st_na(dst + 16ull * (i + k * blockDim.x), v[k]);
        }
    }
}
template <int U>
__global__ void lsu_flat(const uint4* __restrict__ s, uint4* __restrict__ d, uint64_t n16) {
    uint64_t i = (uint64_t(blockIdx.x) * blockDim.x * U) + threadIdx.x;
    uint4 v[U];
#pragma unroll
    for (int k = 0; k < U; ++k) if (i + k * blockDim.x < n16) v[k] = s[i + k * blockDim.x];
#pragma unroll
    for (int k = 0; k < U; ++k) if (i + k * blockDim.x < n16) d[i + k * blockDim.x] = v[k];
}
__device__ __forceinline__ uint32_t su(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
template <int S, int UNIT, int DEFER>
__global__ void tma(const char* s, char* d, uint64_t n) {
    extern __shared__ __align__(128) unsigned char buf[];
    __shared__ __align__(8) uint64_t bar[S];
    if (threadIdx.x) return;
    for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    const uint64_t units = n / UNIT;
    auto load = [&](uint64_t u, int st) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(UNIT));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(buf + st * UNIT)), "l"(s + u * UNIT), "r"(UNIT), "r"(su(&bar[st])) : "memory");
    };
    for (int k = 0; k < S; ++k) { uint64_t u = blockIdx.x + uint64_t(k) * gridDim.x; if (u < units) load(u, k); }
    for (uint64_t k = 0;; ++k) {
        uint64_t u = blockIdx.x + k * gridDim.x;
        if (u >= units) break;
        int st = int(k % S);
        asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}\n" ::"r"(su(&bar[st])), "r"(uint32_t((k / S) & 1)) : "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d + u * UNIT), "r"(su(buf + st * UNIT)), "r"(UNIT) : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (DEFER) {
            if (k >= 1) {
                uint64_t un = blockIdx.x + (k - 1 + S) * gridDim.x;
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                if (un < units) load(un, int((k - 1) % S));
            }
        } else {
            uint64_t un = blockIdx.x + (k + S) * gridDim.x;
            if (un < units) { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); load(un, st); }
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <class F>
void run(const char* name, F f, double bytes) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
        cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (r >= 2 && ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("%-34s %8.1f GB/s (rw)  %s\n", name, 2 * bytes / (best / 1e3) / 1e9, e ? cudaGetErrorString(e) : "");
}

int main() {
    const uint64_t n = 1ull << 30;
    char *s, *d;
    cudaMalloc(&s, n); cudaMalloc(&d, n); cudaMemset(s, 1, n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run("cudaMemcpyAsync d2d", [&] { cudaMemcpyAsync(d, s, n, cudaMemcpyDeviceToDevice); }, n);
    run("lsu persistent U4 16K 8/SM", [&] { lsu_persistent<4, 16384><<<sms * 8, 256>>>(s, d, n); }, n);
    run("lsu persistent U4 16K 4/SM", [&] { lsu_persistent<4, 16384><<<sms * 4, 256>>>(s, d, n); }, n);
    run("lsu persistent U8 32K 8/SM", [&] { lsu_persistent<8, 32768><<<sms * 8, 256>>>(s, d, n); }, n);
    run("lsu persistent U2 8K 8/SM", [&] { lsu_persistent<2, 8192><<<sms * 8, 256>>>(s, d, n); }, n);
    run("lsu flat U1 256t", [&] { lsu_flat<1><<<unsigned(n / 16 / 256), 256>>>((const uint4*)s, (uint4*)d, n / 16); }, n);
    run("lsu flat U2 256t", [&] { lsu_flat<2><<<unsigned(n / 16 / 512), 256>>>((const uint4*)s, (uint4*)d, n / 16); }, n);
    run("lsu flat U4 256t", [&] { lsu_flat<4><<<unsigned(n / 16 / 1024), 256>>>((const uint4*)s, (uint4*)d, n / 16); }, n);
    run("lsu flat U4 512t", [&] { lsu_flat<4><<<unsigned(n / 16 / 2048), 512>>>((const uint4*)s, (uint4*)d, n / 16); }, n);
    cudaFuncSetAttribute(tma<8, 16384, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    cudaFuncSetAttribute(tma<8, 16384, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
    cudaFuncSetAttribute(tma<4, 32768, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    cudaFuncSetAttribute(tma<6, 32768, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    cudaFuncSetAttribute(tma<12, 16384, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
    cudaFuncSetAttribute(tma<4, 16384, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 16384);
    run("tma 8x16K wait0 1/SM", [&] { tma<8, 16384, 0><<<sms, 32, 8 * 16384>>>(s, d, n); }, n);
    run("tma 8x16K defer 1/SM", [&] { tma<8, 16384, 1><<<sms, 32, 8 * 16384>>>(s, d, n); }, n);
    run("tma 4x32K defer 1/SM", [&] { tma<4, 32768, 1><<<sms, 32, 4 * 32768>>>(s, d, n); }, n);
    run("tma 6x32K defer 1/SM", [&] { tma<6, 32768, 1><<<sms, 32, 6 * 32768>>>(s, d, n); }, n);
    run("tma 12x16K defer 1/SM", [&] { tma<12, 16384, 1><<<sms, 32, 12 * 16384>>>(s, d, n); }, n);
    run("tma 4x16K defer 2/SM", [&] { tma<4, 16384, 1><<<sms * 2, 32, 4 * 16384>>>(s, d, n); }, n);
    run("tma 4x16K defer 3/SM", [&] { tma<4, 16384, 1><<<sms * 3, 32, 4 * 16384>>>(s, d, n); }, n);
    return 0;
}
