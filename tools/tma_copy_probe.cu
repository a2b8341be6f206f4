// Probe the TMA tensor-map copy kernel (kernels.cu: tma_copy_add /
// launch_copy_tma) on one strided box shape per process, against a host copy.
//   tma_copy_probe es  sn0 sn1 sn2  dn0 dn1 dn2  so0 so1 so2  do0 do1 do2  e0 e1 e2
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -I include -o tools/tma_copy_probe tools/tma_copy_probe.cu
//        -L paper_2503_10516_b200 -lcel -Xlinker -rpath=$PWD/paper_2503_10516_b200
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_2503_10516_b200/csrc/kernels.cuh"

int main(int argc, char** argv) {
    if (argc != 17) {
        fprintf(stderr, "usage: es sn[3] dn[3] so[3] do[3] ext[3]\n");
        return 2;
    }
    cel::TmaBox b;
    int k = 1;
    b.es = uint32_t(atoi(argv[k++]));
    for (int i = 0; i < 3; ++i) b.sn[i] = atoll(argv[k++]);
    for (int i = 0; i < 3; ++i) b.dn[i] = atoll(argv[k++]);
    for (int i = 0; i < 3; ++i) b.so[i] = atoll(argv[k++]);
    for (int i = 0; i < 3; ++i) b.dof[i] = atoll(argv[k++]);
    for (int i = 0; i < 3; ++i) b.ext[i] = atoll(argv[k++]);
    const size_t sb = size_t(b.sn[0] * b.sn[1] * b.sn[2]) * b.es, db = size_t(b.dn[0] * b.dn[1] * b.dn[2]) * b.es;
    std::vector<unsigned char> hs(sb), hd(db, 0xAB), exp(db, 0xAB);
    for (size_t i = 0; i < sb; ++i) hs[i] = (unsigned char)(i * 131 + 7);
    char *ds, *dd;
    cudaMalloc(&ds, sb);
    cudaMalloc(&dd, db);
    cudaMemcpy(ds, hs.data(), sb, cudaMemcpyHostToDevice);
    cudaMemcpy(dd, hd.data(), db, cudaMemcpyHostToDevice);
    b.src = ds;
    b.dst = dd;
    cel::TmaCopyArgs a;
    memset(&a, 0, sizeof a);
    const int r = cel::tma_copy_add(a, b);
    printf("tma_copy_add = %d", r);
    if (r == 1) printf(" tw %d th %d tiles %u x %u x %u s0 %d %d %d d0 %d %d %d", a.seg[0].tw, a.seg[0].th, a.seg[0].tiles_x,
                       a.seg[0].tiles_y, a.seg[0].planes, a.seg[0].s0[0], a.seg[0].s0[1], a.seg[0].s0[2], a.seg[0].d0[0],
                       a.seg[0].d0[1], a.seg[0].d0[2]);
    printf("\n");
    fflush(stdout);
    if (r != 1) return 0;
    cel::launch_copy_tma(a, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    cudaMemcpy(hd.data(), dd, db, cudaMemcpyDeviceToHost);
    for (int64_t z = 0; z < b.ext[0]; ++z)
        for (int64_t y = 0; y < b.ext[1]; ++y)
            for (int64_t x = 0; x < b.ext[2]; ++x) {
                const size_t so = (((b.so[0] + z) * b.sn[1] + b.so[1] + y) * b.sn[2] + b.so[2] + x) * b.es;
                const size_t dof = (((b.dof[0] + z) * b.dn[1] + b.dof[1] + y) * b.dn[2] + b.dof[2] + x) * b.es;
                memcpy(&exp[dof], &hs[so], b.es);
            }
    size_t bad = 0;
    for (size_t i = 0; i < db; ++i) bad += hd[i] != exp[i];
    printf("mismatched bytes: %zu of %zu\n", bad, db);
    return bad ? 1 : 0;
}
