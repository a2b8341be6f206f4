// Probe: does an event record (or a stream wait on an already-complete event)
// between two kernels of one stream cancel programmatic dependent launch?
// Chain of K short HBM-bound kernels (each reads/writes 64 MiB), timed with
// events, four variants: plain launches, PDL, PDL + cudaEventRecord after each
// kernel, PDL + record + cudaStreamWaitEvent on another stream's old event.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/pdl_probe.cu -o /tmp/pdl_probe && /tmp/pdl_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) step(const float4* __restrict__ a, float4* __restrict__ b, size_t n, int pdl) {
    if (pdl) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
        float4 v = a[i];
        v.x += 1.f;
        b[i] = v;
    }
}

int main() {
    const size_t bytes = 64ull << 20, n = bytes / 16;
    float4 *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaStream_t s, o;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&o, cudaStreamNonBlocking);
    cudaEvent_t e0, e1, old;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreateWithFlags(&old, cudaEventDisableTiming);
    cudaEventRecord(old, o);
    const int K = 200;
    cudaEvent_t evs[K];
    for (int i = 0; i < K; ++i) cudaEventCreateWithFlags(&evs[i], cudaEventDisableTiming);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const unsigned grid = unsigned(sms * 8);
    for (int variant = 0; variant < 4; ++variant)
        for (int rep = 0; rep < 3; ++rep) {
            cudaStreamSynchronize(s);
            cudaEventRecord(e0, s);
            for (int i = 0; i < K; ++i) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute attr[1];
                attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                attr[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = attr;
                cfg.numAttrs = variant > 0 ? 1 : 0;
                cudaLaunchKernelEx(&cfg, step, (const float4*)(i % 2 ? b : a), (i % 2 ? a : b), n, variant > 0 ? 1 : 0);
                if (variant >= 2) cudaEventRecord(evs[i], s);
                if (variant >= 3) cudaStreamWaitEvent(s, old, 0);
            }
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const char* nm[] = {"plain", "pdl", "pdl+record", "pdl+record+wait"};
            printf("%-16s %7.2f us/kernel  (%.0f GB/s)\n", nm[variant], ms * 1e3 / K, 2.0 * bytes / (ms * 1e-3 / K) / 1e9);
        }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
