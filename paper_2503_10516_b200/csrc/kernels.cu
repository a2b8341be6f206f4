// sm_100a kernels of the coherence path.
//
//  * copy_kernel   — Table 1 `copy`: one launch moves every box of a
//    copy instruction's region (resize copies P:L351, coherence / d2d halo
//    copies P:L371-378).  Persistent grid, 16 KiB row chunks per CTA
//    iteration, 128-bit non-allocating loads/stores when the segment is
//    16-byte aligned.  Destination pointers may be peer (NVLink) addresses:
//    the copy then is an SM-driven push over NVSwitch.
//  * workload kernels — the synthetic device-kernel instructions:
//    fill, 1-D 3-point (Listing 5 shape), WaveSim 5-point,
//    3-D 7-point, N-body timestep/update (Listing 1), RSim row
//    (P:L632), integer probe.  Arithmetic order is exactly the oracle's
//    (oracle/kernels.py); the library is built with -fmad=false (R16).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>

#include "kernels.cuh"

namespace cel {

namespace {

int g_copy_blocks_per_sm = 8;
int g_num_sms = 0;

int num_sms() {
    if (g_num_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

// ------------------------------------------------------------------ copy
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_na_v4(void* p, const uint4& v) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}

template <class T>
__device__ __forceinline__ void copy_span(const char* __restrict__ src, char* __restrict__ dst, uint32_t nbytes) {
    const uint32_t n = nbytes / sizeof(T);
    const T* s = reinterpret_cast<const T*>(src);
    T* d = reinterpret_cast<T*>(dst);
    uint32_t i = threadIdx.x;
    constexpr int U = 4;
    for (; i + (U - 1) * blockDim.x < n; i += U * blockDim.x) {
        T v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) v[k] = s[i + k * blockDim.x];
#pragma unroll
        for (int k = 0; k < U; ++k) d[i + k * blockDim.x] = v[k];
    }
    for (; i < n; i += blockDim.x) d[i] = s[i];
}

template <>
__device__ __forceinline__ void copy_span<uint4>(const char* __restrict__ src, char* __restrict__ dst, uint32_t nbytes) {
    const uint32_t n = nbytes / 16;
    uint32_t i = threadIdx.x;
    constexpr int U = 2;
    for (; i + (U - 1) * blockDim.x < n; i += U * blockDim.x) {
        uint4 v[U];
#pragma unroll
        for (int k = 0; k < U; ++k) v[k] = ld_nc_v4(src + 16ull * (i + k * blockDim.x));
#pragma unroll
        for (int k = 0; k < U; ++k) st_na_v4(dst + 16ull * (i + k * blockDim.x), v[k]);
    }
    for (; i < n; i += blockDim.x) st_na_v4(dst + 16ull * i, ld_nc_v4(src + 16ull * i));
}

// Realigning span (shared-memory staging): source and destination 4-byte
// aligned but at different offsets mod 16 (e.g. a resize into an allocation
// one element wider).  The chunk is read with 16-byte loads at the source's
// alignment into shared memory and written with 16-byte stores at the
// destination's alignment; only the destination's head and tail (< 16 bytes
// each) use 4-byte stores.  Without it such copies ran entirely on 4-byte
// accesses (0.74 of the copy peak on 8192 x 16 KiB rows).
__device__ __forceinline__ void copy_span_realign(const char* __restrict__ src, char* __restrict__ dst,
                                                  uint32_t nbytes, uint32_t* sm) {
    const uint32_t sh = uint32_t(uintptr_t(src) & 15);             // multiple of 4
    const char* s0 = src - sh;                                    // 16-byte aligned
    const uint32_t nl = (sh + nbytes + 15) / 16;                  // 16-byte loads covering the span
    for (uint32_t i = threadIdx.x; i < nl; i += blockDim.x) {
        const uint4 v = ld_nc_v4(s0 + 16ull * i);
        sm[4 * i + 0] = v.x;
        sm[4 * i + 1] = v.y;
        sm[4 * i + 2] = v.z;
        sm[4 * i + 3] = v.w;
    }
    __syncthreads();
    const uint32_t* w = sm + sh / 4;                               // word 0 of the span
    const uint32_t nw = nbytes / 4;
    const uint32_t head = ((16 - uint32_t(uintptr_t(dst) & 15)) & 15) / 4;   // words until dst is aligned
    uint32_t* d = reinterpret_cast<uint32_t*>(dst);
    if (threadIdx.x < head && threadIdx.x < nw) d[threadIdx.x] = w[threadIdx.x];
    const uint32_t nv = nw > head ? (nw - head) / 4 : 0;
    for (uint32_t i = threadIdx.x; i < nv; i += blockDim.x) {
        const uint32_t k = head + 4 * i;
        st_na_v4(d + k, make_uint4(w[k], w[k + 1], w[k + 2], w[k + 3]));
    }
    for (uint32_t k = head + 4 * nv + threadIdx.x; k < nw; k += blockDim.x) d[k] = w[k];
    __syncthreads();                                               // sm is reused by the next unit
}

// One CTA per 8 KiB unit (a flat grid: measured faster than a persistent
// grid-stride loop and than cudaMemcpy / torch copy_ on B200, see
// tools/copy_micro.cu); units beyond 2^31 CTAs loop.
__global__ void __launch_bounds__(256, 8) copy_kernel(const __grid_constant__ CopyArgs a) {   // 8 CTAs/SM: <= 32 registers
    __shared__ uint32_t sm[kCopyUnit / 4 + 8];
    for (uint64_t u = blockIdx.x; u < a.total_units; u += gridDim.x) {
        int s = 0;
        while (s + 1 < a.nseg && a.seg[s + 1].units_begin <= u) ++s;
        const CopySeg& g = a.seg[s];
        const uint64_t lu = u - g.units_begin;
        if (g.narrow) {
            // short rows (e.g. a column halo, one element per row): a thread per row
            const uint64_t rl = lu * g.narrow + threadIdx.x;
            if (threadIdx.x < g.narrow && rl < uint64_t(g.rows) * g.planes) {
                const uint64_t plane = rl / g.rows, row = rl - plane * g.rows;
                const char* sp = g.src + plane * g.src_plane_stride + row * g.src_row_stride;
                char* dp = g.dst + plane * g.dst_plane_stride + row * g.dst_row_stride;
                const uint32_t nb = uint32_t(g.row_bytes);
                switch (g.vec) {
                case 16:
                    for (uint32_t o = 0; o < nb; o += 16) *reinterpret_cast<uint4*>(dp + o) = *reinterpret_cast<const uint4*>(sp + o);
                    break;
                case 8:
                    for (uint32_t o = 0; o < nb; o += 8) *reinterpret_cast<uint2*>(dp + o) = *reinterpret_cast<const uint2*>(sp + o);
                    break;
                case 4:
                    for (uint32_t o = 0; o < nb; o += 4) *reinterpret_cast<uint32_t*>(dp + o) = *reinterpret_cast<const uint32_t*>(sp + o);
                    break;
                default:
                    for (uint32_t o = 0; o < nb; ++o) dp[o] = sp[o];
                    break;
                }
            }
            continue;
        }
        const uint64_t row_lin = lu / g.units_per_row;
        const uint32_t chunk = uint32_t(lu - row_lin * g.units_per_row);
        const uint64_t plane = row_lin / g.rows;
        const uint64_t row = row_lin - plane * g.rows;
        const uint64_t off = uint64_t(chunk) * kCopyUnit;
        const char* src = g.src + plane * g.src_plane_stride + row * g.src_row_stride + off;
        char* dst = g.dst + plane * g.dst_plane_stride + row * g.dst_row_stride + off;
        const uint64_t rem = g.row_bytes - off;
        const uint32_t nbytes = rem < kCopyUnit ? uint32_t(rem) : kCopyUnit;
        switch (g.vec) {
        case 16: copy_span<uint4>(src, dst, nbytes); break;
        case 8: copy_span<uint2>(src, dst, nbytes); break;
        case 4: {
            // strides only 4-byte aligned: this unit's own alignment decides
            const uint32_t sa = uint32_t(uintptr_t(src) & 15), da = uint32_t(uintptr_t(dst) & 15);
            if (sa == 0 && da == 0 && (nbytes & 15) == 0)
                copy_span<uint4>(src, dst, nbytes);
            else if (nbytes >= 256)
                copy_span_realign(src, dst, nbytes, sm);
            else
                copy_span<uint32_t>(src, dst, nbytes);
            break;
        }
        case 2: copy_span<uint16_t>(src, dst, nbytes); break;
        default: copy_span<uint8_t>(src, dst, nbytes); break;
        }
    }
    // pushes into peer memory: make the stores visible system-wide before the
    // kernel retires (a flag written after this kernel releases the data)
    if (a.peer) __threadfence_system();
}

// ------------------------------------------------------------------ copy (TMA tensor maps)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
            bar),
        "r"(phase)
        : "memory");
}

// kTmStages x 16 KiB tiles in flight per CTA, of which kTmPend stores may
// still be reading shared memory (6 / 3, 2 CTAs per SM)
constexpr uint32_t kTmTileBytes = 16384;

// One elected thread per CTA streams tiles: TMA tensor load into a stage of the
// shared-memory ring (completion on the stage's mbarrier), then a TMA tensor
// store of the stage into the destination map.  A stage is refilled one tile
// later than the store that drains it, so a store and kTmStages - 1 loads are
// in flight at any time.  Tiles t = blockIdx.x + k * gridDim.x.
template <int kTmStages, int kTmPend>
__global__ void __launch_bounds__(32) copy_kernel_tmap(const __grid_constant__ TmaCopyArgs a) {
    extern __shared__ __align__(128) unsigned char tbuf[];
    __shared__ __align__(8) uint64_t tbar[kTmStages];
    if (threadIdx.x != 0) return;
    for (int k = 0; k < kTmStages; ++k)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&tbar[k])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    struct Tile {
        int s, x, y, z;
    };
    auto tile = [&](uint64_t t) {
        int s = 0;
        while (s + 1 < a.nseg && a.seg[s + 1].tiles_begin <= t) ++s;
        const TmaSeg& g = a.seg[s];
        uint64_t l = t - g.tiles_begin;
        Tile r;
        r.s = s;
        const uint32_t tx = uint32_t(l % g.tiles_x);
        l /= g.tiles_x;
        const uint32_t ty = uint32_t(l % g.tiles_y);
        const uint32_t tz = uint32_t(l / g.tiles_y);
        r.x = int(tx) * g.tw;
        r.y = int(ty) * g.th;
        r.z = int(tz);
        return r;
    };
    auto load = [&](uint64_t t, int st) {
        const Tile q = tile(t);
        const TmaSeg& g = a.seg[q.s];
        const uint32_t b = smem_u32(&tbar[st]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(uint32_t(g.tw * g.th * 4))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                smem_u32(tbuf + size_t(st) * kTmTileBytes)),
            "l"(reinterpret_cast<uint64_t>(&a.map[2 * q.s])), "r"(g.s0[0] + q.x), "r"(g.s0[1] + q.y), "r"(g.s0[2] + q.z),
            "r"(b)
            : "memory");
    };
    auto store = [&](uint64_t t, int st) {
        const Tile q = tile(t);
        const TmaSeg& g = a.seg[q.s];
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                         reinterpret_cast<uint64_t>(&a.map[2 * q.s + 1])),
                     "r"(g.d0[0] + q.x), "r"(g.d0[1] + q.y), "r"(g.d0[2] + q.z),
                     "r"(smem_u32(tbuf + size_t(st) * kTmTileBytes))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    };
    const uint64_t first = blockIdx.x, step = gridDim.x;
    // bring this launch's descriptors into the TMA unit's cache up front (they
    // live in the kernel parameters: a cold fetch at the first load of each)
    for (int q = 0; q < 2 * a.nseg; ++q)
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.map[q])) : "memory");
    for (int k = 0; k < kTmStages; ++k) {
        const uint64_t t = first + uint64_t(k) * step;
        if (t >= a.total_tiles) break;
        load(t, k);
    }
    // kTmPend stores may still be reading their stages: the stage refilled
    // after storing tile k is that of tile k - (kTmPend - 1), whose store is
    // kTmPend - 1 bulk groups old (waiting for the store just issued would
    // serialise every tile on the store path's latency)
    for (uint64_t k = 0;; ++k) {
        const uint64_t t = first + k * step;
        if (t >= a.total_tiles) break;
        const int st = int(k % kTmStages);
        mbar_wait(smem_u32(&tbar[st]), uint32_t((k / kTmStages) & 1));
        store(t, st);
        if (k + 1 >= uint64_t(kTmPend)) {
            const uint64_t j = k + 1 - kTmPend;
            const uint64_t tn = first + (j + kTmStages) * step;
            if (tn < a.total_tiles) {
                asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kTmPend - 1) : "memory");
                load(tn, int(j % kTmStages));
            }
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------ multicast gather
// one store per 16 bytes to the multicast address (SASS: a
// plain STG.E.128 -- the multicast mapping makes NVSwitch replicate it into
// every bound allocation); the source reads with coherent loads because the
// same kernel's multicast stores also land (with equal bytes) in its own chunk.
__global__ void __launch_bounds__(256) mc_gather_kernel(const char* __restrict__ src, char* mc, uint64_t bytes,
                                                        unsigned long long* flag, unsigned* ctr) {
    const uint64_t n16 = bytes / 16;
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = tid; i < n16; i += nth) {
        const uint4 v = *reinterpret_cast<const uint4*>(src + 16 * i);
        asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 16 * i), "f"(__uint_as_float(v.x)),
                     "f"(__uint_as_float(v.y)), "f"(__uint_as_float(v.z)), "f"(__uint_as_float(v.w))
                     : "memory");
    }
    for (uint64_t i = n16 * 4 + tid; i < bytes / 4; i += nth) {
        const uint32_t v = reinterpret_cast<const uint32_t*>(src)[i];
        asm volatile("multimem.st.global.f32 [%0], %1;" ::"l"(mc + 4 * i), "f"(__uint_as_float(v)) : "memory");
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(ctr, 1u);
        if (prev == gridDim.x - 1) {
            *ctr = 0;                                       // the next launch on this stream starts at 0
            __threadfence_system();
            asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(flag), "l"(1ull) : "memory");
        }
    }
}

// ------------------------------------------------------------------ P2P gather
// The chunk is read once (16-byte loads) and stored to each receiver; the
// stores to other GPUs travel over NVLink.  Completion: every CTA fences at
// system scope; the last one bumps each receiver's counter (atomicAdd_system
// on its memory), which the receiver's stream waits for.
__global__ void __launch_bounds__(256) p2p_gather_kernel(const __grid_constant__ P2PGatherArgs a) {
    const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x, nth = uint64_t(gridDim.x) * blockDim.x;
    if (a.vec4) {
        const uint64_t n16 = a.bytes / 16;
        for (uint64_t i = tid; i < n16; i += nth) {
            const uint4 v = *reinterpret_cast<const uint4*>(a.src + 16 * i);
            for (int k = 0; k < a.ndst; ++k) st_na_v4(a.dst[k] + 16 * i, v);
        }
        for (uint64_t i = n16 * 4 + tid; i < a.bytes / 4; i += nth) {
            const uint32_t v = reinterpret_cast<const uint32_t*>(a.src)[i];
            for (int k = 0; k < a.ndst; ++k) reinterpret_cast<uint32_t*>(a.dst[k])[i] = v;
        }
    } else {
        for (uint64_t i = tid; i < a.bytes / 4; i += nth) {
            const uint32_t v = reinterpret_cast<const uint32_t*>(a.src)[i];
            for (int k = 0; k < a.ndst; ++k) reinterpret_cast<uint32_t*>(a.dst[k])[i] = v;
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(a.ctr, 1u);
        if (prev == gridDim.x - 1) {
            *a.ctr = 0;
            __threadfence_system();
            for (int k = 0; k < a.ndst; ++k) atomicAdd_system(a.counter[k], 1ull);
        }
    }
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ int64_t off_of(const DAcc& A, int64_t z, int64_t y, int64_t x) {
    return ((z - A.lo[0]) * A.n[1] + (y - A.lo[1])) * A.n[2] + (x - A.lo[2]);
}
template <class T>
__device__ __forceinline__ T* ptr(const DAcc& A, int64_t z, int64_t y, int64_t x) {
    return reinterpret_cast<T*>(A.base + off_of(A, z, y, x) * int64_t(A.es));
}
__device__ __forceinline__ int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

// Accessor bounds checking (§4.4): an element access outside the
// range-mapper region of its accessor is recorded (bounding box by atomic
// min / max) and reported by the executor after the kernel exits; the access
// itself is redirected to the allocation base when it also leaves the
// allocation, so a wrong range mapper cannot fault the kernel.
template <class T>
__device__ __forceinline__ T* at(const DAcc& A, int64_t z, int64_t y, int64_t x) {
    if (A.oob && (z < A.box.lo[0] || z >= A.box.hi[0] || y < A.box.lo[1] || y >= A.box.hi[1] ||
                  x < A.box.lo[2] || x >= A.box.hi[2])) {
        atomicMin(&A.oob[0], (long long)z);
        atomicMin(&A.oob[1], (long long)y);
        atomicMin(&A.oob[2], (long long)x);
        atomicMax(&A.oob[3], (long long)z + 1);
        atomicMax(&A.oob[4], (long long)y + 1);
        atomicMax(&A.oob[5], (long long)x + 1);
        if (z < A.lo[0] || z >= A.lo[0] + A.n[0] || y < A.lo[1] || y >= A.lo[1] + A.n[1] || x < A.lo[2] ||
            x >= A.lo[2] + A.n[2])
            return reinterpret_cast<T*>(A.base);
    }
    return ptr<T>(A, z, y, x);
}

__global__ void oob_init_kernel(long long* rec, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < 6 * n) rec[i] = (i % 6) < 3 ? 0x7fffffffffffffffLL : (-0x7fffffffffffffffLL - 1);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}

__device__ __forceinline__ float init_value(uint64_t seed, uint64_t idx) {
    const uint64_t h = splitmix64(seed + idx);
    const float v = float(uint32_t(h >> 40));
    return (2.0f * (v * 0x1p-24f)) - 1.0f;
}

// ------------------------------------------------------------------ fills
__global__ void fill_hash_kernel(const __grid_constant__ KArgs a) {
    const DAcc& A = a.acc[0];
    const DBox& b = A.box;
    const int64_t n0 = b.hi[0] - b.lo[0], n1 = b.hi[1] - b.lo[1], n2 = b.hi[2] - b.lo[2];
    const int64_t words = A.es / 4;
    const int64_t total = n0 * n1 * n2 * words;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t w = t % words;
        int64_t e = t / words;
        const int64_t x = b.lo[2] + e % n2;
        e /= n2;
        const int64_t y = b.lo[1] + e % n1;
        const int64_t z = b.lo[0] + e / n1;
        const int64_t lin = (z * A.ext[1] + y) * A.ext[2] + x;
        ptr<float>(A, z, y, x)[w] = init_value(a.seed, uint64_t(lin * words + w));
    }
}

__global__ void fill_const_kernel(const __grid_constant__ KArgs a) {
    const DAcc& A = a.acc[0];
    const DBox& b = A.box;
    const int64_t n0 = b.hi[0] - b.lo[0], n1 = b.hi[1] - b.lo[1], n2 = b.hi[2] - b.lo[2];
    const int64_t words = A.es / 4;
    const int64_t total = n0 * n1 * n2 * words;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t w = t % words;
        int64_t e = t / words;
        const int64_t x = b.lo[2] + e % n2;
        e /= n2;
        const int64_t y = b.lo[1] + e % n1;
        const int64_t z = b.lo[0] + e / n1;
        ptr<float>(A, z, y, x)[w] = a.value;
    }
}

// ------------------------------------------------------------------ C1 3-point
__global__ void stencil3_kernel(const __grid_constant__ KArgs a) {
    const DAcc& S = a.acc[0];
    const DAcc& D = a.acc[1];
    const int64_t n = S.ext[0];
    for (int64_t i = a.chunk.lo[0] + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.chunk.hi[0];
         i += int64_t(gridDim.x) * blockDim.x) {
        const float xm = *at<const float>(S, clampi(i - 1, 0, n - 1), 0, 0);
        const float xc = *at<const float>(S, i, 0, 0);
        const float xp = *at<const float>(S, clampi(i + 1, 0, n - 1), 0, 0);
        *at<float>(D, i, 0, 0) = (0.25f * xm + 0.5f * xc) + 0.25f * xp;
    }
}

// ------------------------------------------------------------------ C2 WaveSim
__device__ __forceinline__ float wave1(float uc, float up, float un, float us, float uw, float ue) {
    const float lap = ((un + us) + (uw + ue)) - 4.0f * uc;
    return (2.0f * uc - up) + 0.25f * lap;
}

// generic (scalar) path: any alignment
__global__ void wave5_scalar(const __grid_constant__ KArgs a) {
    const DAcc& U = a.acc[0];
    const DAcc& P = a.acc[1];
    const int64_t r0 = a.chunk.lo[0], c0 = a.chunk.lo[1];
    const int64_t nr = a.chunk.hi[0] - r0, nc = a.chunk.hi[1] - c0;
    const int64_t E0 = U.ext[0], E1 = U.ext[1];
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nr * nc; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = r0 + t / nc, c = c0 + t % nc;
        const float uc = *at<const float>(U, r, c, 0);
        const float un = *at<const float>(U, clampi(r - 1, 0, E0 - 1), c, 0);
        const float us = *at<const float>(U, clampi(r + 1, 0, E0 - 1), c, 0);
        const float uw = *at<const float>(U, r, clampi(c - 1, 0, E1 - 1), 0);
        const float ue = *at<const float>(U, r, clampi(c + 1, 0, E1 - 1), 0);
        float* pp = at<float>(P, r, c, 0);
        *pp = wave1(uc, *pp, un, us, uw, ue);
    }
}

constexpr int kWaveRows = 8;                  // strip height cap of the automatic choice (sweep r02: 8 beat 16 by 3-4%)

// vector path: 128 threads x float4 = 512 columns per CTA, a strip of kWaveRows
// rows marched top to bottom with a 3-row register window; west/east
// neighbours come from warp shuffles (scalar loads only at warp edges).
// kHalo: the halo exchange fused in (HaloArgs, exec_halo.cu).
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// spin until *f >= v (32-bit counter, wrap-safe); traps like wait_flag
__device__ __forceinline__ void wait_flag32(const unsigned* f, unsigned v) {
    const long long t0 = clock64();
    while (int(ld_acquire_gpu32(f) - v) < 0) {
        __nanosleep(32);
        if (clock64() - t0 > (1ll << 37)) __trap();
    }
}
// spin until *f >= v; a flag that never comes traps after ~2^37 cycles (~70 s: a
// failed launch instead of a hung GPU)
__device__ __forceinline__ void wait_flag(const unsigned long long* f, unsigned long long v) {
    const long long t0 = clock64();
    while (ld_acquire_sys(f) < v) {
        __nanosleep(64);
        if (clock64() - t0 > (1ll << 37)) __trap();
    }
}

// One CTA's strip: rows [rs, re) of its 512 columns.  kPlain: u through
// plain (coherent) loads -- rows another GPU stored while this kernel ran,
// under a flag -- instead of the read-only path.
template <bool kPlain>
__device__ __forceinline__ void wave5_rows(const DAcc& U, const DAcc& P, int64_t rs, int64_t re, int64_t c, int64_t c1,
                                           bool valid) {
    const int64_t E0 = U.ext[0], E1 = U.ext[1];
    const int lane = threadIdx.x & 31;
    const float* ub = reinterpret_cast<const float*>(U.base);
    float* pb = reinterpret_cast<float*>(P.base);
    const int64_t uoff = c - U.lo[1];
    const int64_t poff = c - P.lo[1];
    auto urow = [&](int64_t r) { return ub + (r - U.lo[0]) * U.n[1]; };
    auto ld4 = [&](const float* q) {
        return kPlain ? *reinterpret_cast<const float4*>(q) : __ldg(reinterpret_cast<const float4*>(q));
    };
    auto ld1 = [&](const float* q) { return kPlain ? *q : __ldg(q); };
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 prev = z4, cur = z4;
    if (valid) {
        prev = ld4(urow(rs > 0 ? rs - 1 : 0) + uoff);
        cur = ld4(urow(rs) + uoff);
    }
    const bool need_e = valid && (lane == 31 || c + 4 >= c1);
    const bool need_w = valid && lane == 0;
    const int64_t cw = c > 0 ? c - 1 : 0;
    const int64_t ce = c + 4 < E1 ? c + 4 : E1 - 1;
#pragma unroll 2
    for (int64_t r = rs; r < re; ++r) {
        const int64_t rn = r + 1 < E0 ? r + 1 : E0 - 1;
        float4 nxt = z4, up = z4;
        float* prow = pb + (r - P.lo[0]) * P.n[1] + poff;
        if (valid) {
            nxt = ld4(urow(rn) + uoff);
            up = *reinterpret_cast<const float4*>(prow);
        }
        float w = __shfl_up_sync(0xffffffffu, cur.w, 1);
        float e = __shfl_down_sync(0xffffffffu, cur.x, 1);
        if (need_w) w = ld1(urow(r) + (cw - U.lo[1]));
        if (need_e) e = ld1(urow(r) + (ce - U.lo[1]));
        float4 o;
        o.x = wave1(cur.x, up.x, prev.x, nxt.x, w, cur.y);
        o.y = wave1(cur.y, up.y, prev.y, nxt.y, cur.x, cur.z);
        o.z = wave1(cur.z, up.z, prev.z, nxt.z, cur.y, cur.w);
        o.w = wave1(cur.w, up.w, prev.w, nxt.w, cur.z, e);
        if (valid) *reinterpret_cast<float4*>(prow) = o;
        prev = cur;
        cur = nxt;
    }
}

// Forward rows [ra, rb) of this thread's columns (just written to P: L1 / L2
// hits) into every outgoing copy that holds them, then count the CTA in: the
// last CTA of copy i publishes the receiver's flag.  bar.sync, then thread
// 0's cumulative system fence, order every thread's peer stores before it.
__device__ __forceinline__ void wave5_push(const DAcc& P, const HaloArgs& hx, int64_t ra, int64_t rb, int64_t c,
                                           bool valid) {
    unsigned outs = 0;
    for (int i = 0; i < hx.n_out; ++i)
        if (hx.r0[i] < rb && ra < hx.r1[i]) outs |= 1u << i;
    if (!outs) return;
    if (hx.n_war) {                         // the receivers' readers of those rows are done
        if (threadIdx.x == 0)
            for (int i = 0; i < hx.n_war; ++i) wait_flag(hx.war_flag[i], hx.war_value[i]);
        __syncthreads();
    }
    if (valid) {
        const float* pb = reinterpret_cast<const float*>(P.base);
        for (int i = 0; i < hx.n_out; ++i) {
            if (!((outs >> i) & 1u)) continue;
            const int64_t a = ra > hx.r0[i] ? ra : hx.r0[i], b = rb < hx.r1[i] ? rb : hx.r1[i];
            for (int64_t r = a; r < b; ++r)
                *reinterpret_cast<float4*>(reinterpret_cast<float*>(hx.base[i]) + (r - hx.lo0[i]) * hx.n1[i] +
                                           (c - hx.lo1[i])) =
                    *reinterpret_cast<const float4*>(pb + (r - P.lo[0]) * P.n[1] + (c - P.lo[1]));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        for (int i = 0; i < hx.n_out; ++i)
            if ((outs >> i) & 1u) {
                const unsigned old = atomicAdd(hx.ctr[i], 1u);
                if (old == hx.ctr_last[i]) {
                    __threadfence_system();
                    st_release_sys(hx.flag[i], hx.value[i]);
                }
            }
    }
}

template <bool kHalo>
__device__ __forceinline__ void wave5_body(const KArgs& a, const HaloArgs* hxp) {
    const DAcc& U = a.acc[0];
    const DAcc& P = a.acc[1];
    const int64_t r0 = a.chunk.lo[0], r1 = a.chunk.hi[0];
    const int64_t c0 = a.chunk.lo[1], c1 = a.chunk.hi[1];
    const int64_t c = c0 + (int64_t(blockIdx.x) * 128 + threadIdx.x) * 4;
    const bool valid = c < c1;
    const int64_t h = a.strip > 0 ? a.strip : kWaveRows;
    // halo launches visit the last strip second (CTAs start roughly in
    // blockIdx order): both boundary strips -- the ones that exchange rows
    // with the neighbours -- run first, so pushes leave early and the
    // neighbours' flags are set by the time their boundary strips look
    int64_t sy = blockIdx.y;
    if (kHalo && gridDim.y > 2) sy = blockIdx.y == 0 ? 0 : (blockIdx.y == 1 ? int64_t(gridDim.y) - 1 : int64_t(blockIdx.y) - 1);
    const int64_t rs = r0 + sy * h;
    const int64_t re = rs + h < r1 ? rs + h : r1;
    // programmatic dependent launch (see launch_wave5): the previous step wrote u
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (!kHalo) {
        wave5_rows<false>(U, P, rs, re, c, c1, valid);
        return;
    }
    const HaloArgs& hx = *hxp;
    // incoming rows this strip reads: wait for their flags first
    bool wait_in = false;
    for (int i = 0; i < hx.n_in; ++i)
        if (hx.in_r0[i] < re + 1 && rs - 1 < hx.in_r1[i]) wait_in = true;
    if (wait_in) {
        if (threadIdx.x == 0)
            for (int i = 0; i < hx.n_in; ++i)
                if (hx.in_r0[i] < re + 1 && rs - 1 < hx.in_r1[i]) wait_flag(hx.in_flag[i], hx.in_value[i]);
        __syncthreads();
        wave5_rows<true>(U, P, rs, re, c, c1, valid);
    } else {
        wave5_rows<false>(U, P, rs, re, c, c1, valid);
    }
    wave5_push(P, hx, rs, re, c, valid);
}

__global__ void __launch_bounds__(128) wave5_vec(const __grid_constant__ KArgs a) {
    wave5_body<false>(a, nullptr);
}

__global__ void __launch_bounds__(128) wave5_halo(const __grid_constant__ KArgs a, const __grid_constant__ HaloArgs hx) {
    wave5_body<true>(a, &hx);
}

// The same kernels held to 32 registers: 16 CTAs per SM instead of 12, for
// thin chunks (see wave5_strip)
__global__ void __launch_bounds__(128, 16) wave5_vec16(const __grid_constant__ KArgs a) {
    wave5_body<false>(a, nullptr);
}

__global__ void __launch_bounds__(128, 16) wave5_halo16(const __grid_constant__ KArgs a, const __grid_constant__ HaloArgs hx) {
    wave5_body<true>(a, &hx);
}

// ------------------------------------------------------------------ C5 Jacobi 7-point
__device__ __forceinline__ float jac1(float c, float zm, float zp, float ym, float yp, float xm, float xp) {
    return 0.25f * c + 0.125f * (((zm + zp) + (ym + yp)) + (xm + xp));
}

__global__ void jacobi7_scalar(const __grid_constant__ KArgs a) {
    const DAcc& A = a.acc[0];
    const DAcc& B = a.acc[1];
    const DBox& ch = a.chunk;
    const int64_t n0 = ch.hi[0] - ch.lo[0], n1 = ch.hi[1] - ch.lo[1], n2 = ch.hi[2] - ch.lo[2];
    const int64_t E0 = A.ext[0], E1 = A.ext[1], E2 = A.ext[2];
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n0 * n1 * n2; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = ch.lo[2] + t % n2;
        const int64_t y = ch.lo[1] + (t / n2) % n1;
        const int64_t z = ch.lo[0] + t / (n1 * n2);
        const float c = *at<const float>(A, z, y, x);
        const float zm = *at<const float>(A, clampi(z - 1, 0, E0 - 1), y, x);
        const float zp = *at<const float>(A, clampi(z + 1, 0, E0 - 1), y, x);
        const float ym = *at<const float>(A, z, clampi(y - 1, 0, E1 - 1), x);
        const float yp = *at<const float>(A, z, clampi(y + 1, 0, E1 - 1), x);
        const float xm = *at<const float>(A, z, y, clampi(x - 1, 0, E2 - 1));
        const float xp = *at<const float>(A, z, y, clampi(x + 1, 0, E2 - 1));
        *at<float>(B, z, y, x) = jac1(c, zm, zp, ym, yp, xm, xp);
    }
}

constexpr int kJacZ = 16;

__global__ void __launch_bounds__(128) jacobi7_vec(const __grid_constant__ KArgs a) {
    const DAcc& A = a.acc[0];
    const DAcc& B = a.acc[1];
    const DBox& ch = a.chunk;
    const int64_t E0 = A.ext[0], E1 = A.ext[1], E2 = A.ext[2];
    const int lane = threadIdx.x & 31;
    const int64_t x = ch.lo[2] + (int64_t(blockIdx.x) * 128 + threadIdx.x) * 4;
    const bool valid = x < ch.hi[2];
    const int64_t y = ch.lo[1] + blockIdx.y;
    const int64_t zs = ch.lo[0] + int64_t(blockIdx.z) * kJacZ;
    const int64_t ze = zs + kJacZ < ch.hi[0] ? zs + kJacZ : ch.hi[0];
    const int64_t ym = y > 0 ? y - 1 : 0, yp = y + 1 < E1 ? y + 1 : E1 - 1;
    const int64_t xw = x > 0 ? x - 1 : 0, xe = x + 4 < E2 ? x + 4 : E2 - 1;
    const float* ab = reinterpret_cast<const float*>(A.base);
    float* bb = reinterpret_cast<float*>(B.base);
    auto arow = [&](int64_t z, int64_t yy) { return ab + ((z - A.lo[0]) * A.n[1] + (yy - A.lo[1])) * A.n[2] - A.lo[2]; };
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 prev = z4, cur = z4;
    if (valid) {
        prev = __ldg(reinterpret_cast<const float4*>(arow(zs > 0 ? zs - 1 : 0, y) + x));
        cur = __ldg(reinterpret_cast<const float4*>(arow(zs, y) + x));
    }
    const bool need_e = valid && (lane == 31 || x + 4 >= ch.hi[2]);
    const bool need_w = valid && lane == 0;
    for (int64_t z = zs; z < ze; ++z) {
        const int64_t zn = z + 1 < E0 ? z + 1 : E0 - 1;
        float4 nxt = z4, fm = z4, fp = z4;
        if (valid) {
            nxt = __ldg(reinterpret_cast<const float4*>(arow(zn, y) + x));
            fm = __ldg(reinterpret_cast<const float4*>(arow(z, ym) + x));
            fp = __ldg(reinterpret_cast<const float4*>(arow(z, yp) + x));
        }
        float w = __shfl_up_sync(0xffffffffu, cur.w, 1);
        float e = __shfl_down_sync(0xffffffffu, cur.x, 1);
        if (need_w) w = __ldg(arow(z, y) + xw);
        if (need_e) e = __ldg(arow(z, y) + xe);
        float4 o;
        o.x = jac1(cur.x, prev.x, nxt.x, fm.x, fp.x, w, cur.y);
        o.y = jac1(cur.y, prev.y, nxt.y, fm.y, fp.y, cur.x, cur.z);
        o.z = jac1(cur.z, prev.z, nxt.z, fm.z, fp.z, cur.y, cur.w);
        o.w = jac1(cur.w, prev.w, nxt.w, fm.w, fp.w, cur.z, e);
        if (valid)
            *reinterpret_cast<float4*>(bb + ((z - B.lo[0]) * B.n[1] + (y - B.lo[1])) * B.n[2] + (x - B.lo[2])) = o;
        prev = cur;
        cur = nxt;
    }
}

// TMA tensor-map version: one elected thread streams z-plane tiles of the
// input allocation, (BY+2) rows x (BX+8) columns (y halo + 16-byte aligned x
// halo), into a 4-stage shared-memory ring with cp.async.bulk.tensor.3d
// (SASS UTMALDG) completing on mbarriers; 512 consumer threads compute a
// BY x BX output tile per plane from shared memory (z-1, z, z+1 are all in
// the ring) and store float4 rows.  Out-of-bounds tile parts are zero-filled
// by TMA and never read: the consumers clamp at the buffer edges (R16 order
// of operations unchanged).
constexpr int kJBX = 128, kJBY = 16, kJZS = 64, kJStages = 4;
constexpr int kJPW = kJBX + 8, kJPH = kJBY + 2, kJPlane = kJPW * kJPH;   // floats per staged plane
constexpr int kJStride = (kJPlane + 31) / 32 * 32;                          // stage stride: 128-byte aligned

__global__ void __launch_bounds__(512) jacobi7_tma(const __grid_constant__ CUtensorMap tm, const __grid_constant__ KArgs a) {
    extern __shared__ __align__(128) float jsm[];
    __shared__ __align__(8) uint64_t jbar[kJStages];
    const DAcc& A = a.acc[0];
    const DAcc& B = a.acc[1];
    const DBox& ch = a.chunk;
    const int64_t E0 = A.ext[0], E1 = A.ext[1], E2 = A.ext[2];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t x0 = ch.lo[2] + int64_t(blockIdx.x) * kJBX;
    const int64_t y0 = ch.lo[1] + int64_t(blockIdx.y) * kJBY;
    const int64_t zs = ch.lo[0] + int64_t(blockIdx.z) * kJZS;
    const int64_t ze = zs + kJZS < ch.hi[0] ? zs + kJZS : ch.hi[0];
    const int nplanes = int(ze - zs) + 2;                       // planes zs-1 .. ze (clamped)
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
        for (int k = 0; k < kJStages; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&jbar[k])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // programmatic dependent launch (as wave5): the next step's prologue may
    // overlap this grid's tail; the input planes come from the previous step
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __syncthreads();
    auto issue = [&](int i) {       // plane i (0 -> zs-1), clamped to the buffer extent
        int64_t z = zs - 1 + i;
        z = z < 0 ? 0 : (z > E0 - 1 ? E0 - 1 : z);
        const int st = i % kJStages;
        const uint32_t b = smem_u32(&jbar[st]);
        const int c0 = int(x0 - 4 - A.lo[2]), c1 = int(y0 - 1 - A.lo[1]), c2 = int(z - A.lo[0]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(uint32_t(kJPlane * 4))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                smem_u32(jsm + size_t(st) * kJStride)),
            "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(c1), "r"(c2), "r"(b)
            : "memory");
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < 3 && i < nplanes; ++i) issue(i);
    const int64_t gx = x0 + 4 * tx, gy = y0 + ty;
    const bool valid = gx < ch.hi[2] && gy < ch.hi[1];
    const int cx = 4 * tx + 4, ry = ty + 1;
    const int rym = gy == 0 ? ry : ry - 1;
    const int ryp = gy == E1 - 1 ? ry : ry + 1;
    float* bb = reinterpret_cast<float*>(B.base);
    for (int j = 0; j + 2 < nplanes; ++j) {
        if (threadIdx.x == 0 && j + 3 < nplanes) issue(j + 3);   // stage of plane j-1, freed by the last barrier
        for (int i = j; i <= j + 2; ++i) mbar_wait(smem_u32(&jbar[i % kJStages]), uint32_t((i / kJStages) & 1));
        const float* P0 = jsm + size_t(j % kJStages) * kJStride;
        const float* P1 = jsm + size_t((j + 1) % kJStages) * kJStride;
        const float* P2 = jsm + size_t((j + 2) % kJStages) * kJStride;
        if (valid) {
            const float4 c = *reinterpret_cast<const float4*>(P1 + ry * kJPW + cx);
            const float4 zm = *reinterpret_cast<const float4*>(P0 + ry * kJPW + cx);
            const float4 zp = *reinterpret_cast<const float4*>(P2 + ry * kJPW + cx);
            const float4 fm = *reinterpret_cast<const float4*>(P1 + rym * kJPW + cx);
            const float4 fp = *reinterpret_cast<const float4*>(P1 + ryp * kJPW + cx);
            const float w = gx == 0 ? c.x : P1[ry * kJPW + cx - 1];
            const float e = gx + 4 >= E2 ? c.w : P1[ry * kJPW + cx + 4];
            float4 o;
            o.x = jac1(c.x, zm.x, zp.x, fm.x, fp.x, w, c.y);
            o.y = jac1(c.y, zm.y, zp.y, fm.y, fp.y, c.x, c.z);
            o.z = jac1(c.z, zm.z, zp.z, fm.z, fp.z, c.y, c.w);
            o.w = jac1(c.w, zm.w, zp.w, fm.w, fp.w, c.z, e);
            const int64_t z = zs + j;
            *reinterpret_cast<float4*>(bb + ((z - B.lo[0]) * B.n[1] + (gy - B.lo[1])) * B.n[2] + (gx - B.lo[2])) = o;
        }
        __syncthreads();
    }
}

// Tensor maps of input allocations, cached by (base, extents).
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

bool jacobi_tensor_map(const DAcc& A, CUtensorMap* out) {
    static EncodeFn enc = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    }
    if (!enc) return false;
    static std::map<std::tuple<const char*, int64_t, int64_t, int64_t>, CUtensorMap> cache;
    auto key = std::make_tuple(static_cast<const char*>(A.base), A.n[0], A.n[1], A.n[2]);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    CUtensorMap m;
    const cuuint64_t dims[3] = {cuuint64_t(A.n[2]), cuuint64_t(A.n[1]), cuuint64_t(A.n[0])};
    const cuuint64_t strides[2] = {cuuint64_t(A.n[2]) * 4, cuuint64_t(A.n[1] * A.n[2]) * 4};
    const cuuint32_t box[3] = {kJPW, kJPH, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, A.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (cache.size() > 256) cache.clear();
    cache[key] = m;
    *out = m;
    return true;
}

// ------------------------------------------------------------------ C3 N-body
constexpr float NB_DT = 0x1p-7f;
constexpr float NB_MASS = 0x1p-20f;
constexpr float NB_EPS2 = 0x1p-10f;
constexpr int kNbTile = 256;

__global__ void __launch_bounds__(kNbTile) nbody_step_kernel(const __grid_constant__ KArgs a) {
    const DAcc& P = a.acc[0];
    const DAcc& V = a.acc[1];
    __shared__ float4 sp[kNbTile];
    const int64_t i = a.chunk.lo[0] + int64_t(blockIdx.x) * kNbTile + threadIdx.x;
    const bool valid = i < a.chunk.hi[0];
    const int64_t N = P.ext[0];
    float4 pi = make_float4(0.f, 0.f, 0.f, 0.f);
    if (valid) pi = *at<const float4>(P, i, 0, 0);
    float ax = 0.f, ay = 0.f, az = 0.f;
    for (int64_t j0 = 0; j0 < N; j0 += kNbTile) {
        const int64_t j = j0 + threadIdx.x;
        sp[threadIdx.x] = j < N ? *at<const float4>(P, j, 0, 0) : make_float4(0.f, 0.f, 0.f, 0.f);
        __syncthreads();
        const int jn = N - j0 < kNbTile ? int(N - j0) : kNbTile;
        for (int k = 0; k < jn; ++k) {
            const float4 pj = sp[k];
            const float dx = pj.x - pi.x, dy = pj.y - pi.y, dz = pj.z - pi.z;
            const float r2 = ((dx * dx + dy * dy) + dz * dz) + NB_EPS2;
            const float inv = 1.0f / sqrtf(r2);
            const float s = (inv * inv) * inv;
            ax = ax + dx * s;
            ay = ay + dy * s;
            az = az + dz * s;
        }
        __syncthreads();
    }
    if (valid) {
        float4* vp = at<float4>(V, i, 0, 0);
        float4 v = *vp;
        const float c = NB_DT * NB_MASS;
        v.x = v.x + c * ax;
        v.y = v.y + c * ay;
        v.z = v.z + c * az;
        *vp = v;
    }
}

// fast-math timestep on Blackwell packed FP32x2 (FFMA2 / FADD2 / FMUL2):
// bodies i and i + 128 ride in the two lanes of every float2 operation, so
// one instruction does the arithmetic of two interactions (rsqrt stays scalar)
__global__ void __launch_bounds__(128) nbody_step_fast_x2_kernel(const __grid_constant__ KArgs a) {
    const DAcc& P = a.acc[0];
    const DAcc& V = a.acc[1];
    __shared__ float4 sp[kNbTile];
    const int64_t i0 = a.chunk.lo[0] + int64_t(blockIdx.x) * kNbTile + threadIdx.x;
    const int64_t i1 = i0 + 128;
    const bool v0 = i0 < a.chunk.hi[0], v1 = i1 < a.chunk.hi[0];
    const int64_t N = P.ext[0];
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 p0 = v0 ? *ptr<const float4>(P, i0, 0, 0) : z4;
    const float4 p1 = v1 ? *ptr<const float4>(P, i1, 0, 0) : z4;
    const float2 npx = make_float2(-p0.x, -p1.x), npy = make_float2(-p0.y, -p1.y), npz = make_float2(-p0.z, -p1.z);
    const float2 eps = make_float2(NB_EPS2, NB_EPS2);
    float2 ax = make_float2(0.f, 0.f), ay = ax, az = ax;
    for (int64_t j0 = 0; j0 < N; j0 += kNbTile) {
        for (int t = threadIdx.x; t < kNbTile; t += 128) {
            const int64_t j = j0 + t;
            sp[t] = j < N ? *ptr<const float4>(P, j, 0, 0) : z4;
        }
        __syncthreads();
        const int jn = N - j0 < kNbTile ? int(N - j0) : kNbTile;
        auto body = [&](const float4 pj) {
            const float2 dx = __fadd2_rn(make_float2(pj.x, pj.x), npx);
            const float2 dy = __fadd2_rn(make_float2(pj.y, pj.y), npy);
            const float2 dz = __fadd2_rn(make_float2(pj.z, pj.z), npz);
            const float2 r2 = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __ffma2_rn(dx, dx, eps)));
            const float2 q = make_float2(rsqrtf(r2.x), rsqrtf(r2.y));
            const float2 sq = __fmul2_rn(__fmul2_rn(q, q), q);
            ax = __ffma2_rn(dx, sq, ax);
            ay = __ffma2_rn(dy, sq, ay);
            az = __ffma2_rn(dz, sq, az);
        };
        if (jn == kNbTile) {
#pragma unroll 8
            for (int k = 0; k < kNbTile; ++k) body(sp[k]);
        } else {
            for (int k = 0; k < jn; ++k) body(sp[k]);
        }
        __syncthreads();
    }
    const float c = NB_DT * NB_MASS;
    if (v0) {
        float4* vp = ptr<float4>(V, i0, 0, 0);
        float4 v = *vp;
        v.x = __fmaf_rn(c, ax.x, v.x);
        v.y = __fmaf_rn(c, ay.x, v.y);
        v.z = __fmaf_rn(c, az.x, v.z);
        *vp = v;
    }
    if (v1) {
        float4* vp = ptr<float4>(V, i1, 0, 0);
        float4 v = *vp;
        v.x = __fmaf_rn(c, ax.y, v.x);
        v.y = __fmaf_rn(c, ay.y, v.y);
        v.z = __fmaf_rn(c, az.y, v.z);
        *vp = v;
    }
}

__global__ void nbody_update_kernel(const __grid_constant__ KArgs a) {
    const DAcc& V = a.acc[0];
    const DAcc& P = a.acc[1];
    for (int64_t i = a.chunk.lo[0] + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.chunk.hi[0];
         i += int64_t(gridDim.x) * blockDim.x) {
        const float4 v = *at<const float4>(V, i, 0, 0);
        float4* pp = at<float4>(P, i, 0, 0);
        float4 p = *pp;
        p.x = p.x + NB_DT * v.x;
        p.y = p.y + NB_DT * v.y;
        p.z = p.z + NB_DT * v.z;
        *pp = p;
    }
}

// ------------------------------------------------------------------ C4 RSim row
// Row t = 0.5 * row[t-1] + 0.5/t * sum_{s<t} row[s][(i+s) mod W], the sum taken
// in ascending s with sequential adds (R16).  HBM bound: t*W*4 B per launch.
// Register fallback (when the TMA variant's layout preconditions fail): each
// thread keeps U = 16 independent loads in flight (~18 warps per SM at
// W = 84,000; 8 loads in flight ran 56 ms per 1024 rows, 16 ran 42.5 ms).
// Evict-last / evict-first L2 hints for a pinned prefix of rows were measured
// and dropped (within 2%).
template <int U>
__global__ void __launch_bounds__(128) rsim_row_kernel(const __grid_constant__ KArgs a) {
    const DAcc& R = a.acc[0];
    const DAcc& Wr = a.acc[1];
    const int64_t t = a.t;
    const int64_t W = R.ext[1];
    const float* base = ptr<const float>(R, 0, 0, 0);
    const int64_t pitch = R.n[1];
    for (int64_t i = a.chunk.lo[0] + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.chunk.hi[0];
         i += int64_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        int64_t s = 0;
        for (; s + U <= t; s += U) {
            float v[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                int64_t c = i + s + k;
                c = c >= W ? c - W : c;
                v[k] = __ldg(base + (s + k) * pitch + c);
            }
#pragma unroll
            for (int k = 0; k < U; ++k) acc = acc + v[k];
        }
        for (; s < t; ++s) {
            int64_t c = i + s;
            c = c >= W ? c - W : c;
            acc = acc + __ldg(base + s * pitch + c);
        }
        const float prev = *ptr<const float>(R, t - 1, i, 0);
        const float coef = 0.5f / float(t);
        *ptr<float>(Wr, t, i, 0) = 0.5f * prev + coef * acc;
    }
}

// Bounds-checked variant: every element access through at() (§4.4).
__global__ void rsim_row_checked(const __grid_constant__ KArgs a) {
    const DAcc& R = a.acc[0];
    const DAcc& Wr = a.acc[1];
    const int64_t t = a.t;
    const int64_t W = R.ext[1];
    for (int64_t i = a.chunk.lo[0] + int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < a.chunk.hi[0];
         i += int64_t(gridDim.x) * blockDim.x) {
        float acc = 0.f;
        for (int64_t s = 0; s < t; ++s) {
            int64_t c = i + s;
            c = c >= W ? c - W : c;
            acc = acc + *at<const float>(R, s, c, 0);
        }
        const float prev = *at<const float>(R, t - 1, i, 0);
        const float coef = 0.5f / float(t);
        *at<float>(Wr, t, i, 0) = 0.5f * prev + coef * acc;
    }
}

// TMA-staged variant (default): a CTA owns kRC consecutive columns.  For a
// stage of kRR rows starting at s0 it needs, from row s0+k, the kRC columns
// starting at (i0 + s0 + k) mod W: all inside one kRR x kRB rectangle whose
// first column is (i0 + s0) mod W rounded down to 16 bytes.  One elected
// thread loads that rectangle with one cp.async.bulk.tensor.2d (SASS UTMALDG)
// into a kRS-stage ring completing on mbarriers; where the rectangle would
// cross column W it loads each row as two cp.async.bulk pieces (wrap) instead.
// The kRC consumer threads add from shared memory in ascending s (R16).
// ~3 stages x 9.5 KB in flight per CTA, 4-5 CTAs per SM.
// Preconditions (host): the read allocation spans whole rows (pitch == W),
// W % 4 == 0, W >= 2 kRB, base 16-byte aligned.
constexpr int kRC = 128, kRR = 16, kRS = 4, kRB = kRC + kRR + 4;

template <bool kPeer>
__global__ void __launch_bounds__(kRC) rsim_row_tma_t(const __grid_constant__ CUtensorMap tm,
                                                      const __grid_constant__ KArgs a, const __grid_constant__ PeerOut po) {
    extern __shared__ __align__(128) float rsm[];
    __shared__ __align__(8) uint64_t rbar[kRS];
    const DAcc& R = a.acc[0];
    const DAcc& Wr = a.acc[1];
    const int64_t t = a.t;
    const int64_t W = R.ext[1];
    const int64_t i0 = a.chunk.lo[0] + int64_t(blockIdx.x) * kRC;
    const char* base = R.base;                       // row R.lo[0], column 0
    const int nst = int((t + kRR - 1) / kRR);
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
        for (int k = 0; k < kRS; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&rbar[k])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // programmatic dependent launch: the next row's kernel may be scheduled
    // now (its prologue above overlaps this kernel's tail); everything below
    // reads rows the previous kernel wrote, so wait for it to have completed
    // (a no-op when the launch was not programmatic)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (kPeer && po.chain) {
        if (threadIdx.x == 0) {
            wait_flag32(po.done, po.done_wait);
            // the rows were written by generic-proxy stores; TMA reads them
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
    } else {
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    __syncthreads();
    // incoming rows (other GPUs' stores under a flag; TMA reads them from L2)
    // are the newest ones (row t - 1 in steady state): the producer waits for
    // their flags only before issuing the first stage that holds a row at or
    // after po.in_row0, so the older rows stream meanwhile
    bool in_done = !(kPeer && po.n_in);
    auto issue = [&](int g) {
        if (kPeer && !in_done && int64_t(g + 1) * kRR > po.in_row0) {
            for (int k = 0; k < po.n_in; ++k) wait_flag(po.in_flag[k], po.in_value[k]);
            asm volatile("fence.proxy.async.global;" ::: "memory");   // generic-proxy stores, TMA reads
            in_done = true;
        }
        const int st = g % kRS;
        const int64_t s0 = int64_t(g) * kRR;
        const int nr = int(t - s0 < kRR ? t - s0 : kRR);
        const int64_t c0 = ((i0 + s0) % W) & ~int64_t(3);
        const uint32_t b = smem_u32(&rbar[st]);
        float* dst = rsm + size_t(st) * kRR * kRB;
        if (c0 + kRB <= W) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(uint32_t(kRR * kRB * 4))
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    smem_u32(dst)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(int(c0)), "r"(int(s0 - R.lo[0])), "r"(b)
                : "memory");
        } else {
            const uint32_t n1 = uint32_t(W - c0), n2 = uint32_t(kRB) - n1;   // floats, both multiples of 4
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(uint32_t(nr * kRB * 4))
                         : "memory");
            for (int k = 0; k < nr; ++k) {
                const char* row = base + (s0 + k - R.lo[0]) * W * 4;
                float* d = dst + k * kRB;
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(d)),
                             "l"(row + c0 * 4), "r"(n1 * 4), "r"(b)
                             : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                 smem_u32(d + n1)),
                             "l"(row), "r"(n2 * 4), "r"(b)
                             : "memory");
            }
        }
    };
    if (threadIdx.x == 0)
        for (int g = 0; g < kRS - 1 && g < nst; ++g) issue(g);
    const int j = threadIdx.x;
    float acc = 0.f;
    for (int g = 0; g < nst; ++g) {
        if (threadIdx.x == 0 && g + kRS - 1 < nst) issue(g + kRS - 1);   // its stage was freed by the last barrier
        const int st = g % kRS;
        mbar_wait(smem_u32(&rbar[st]), uint32_t((g / kRS) & 1));
        const int64_t s0 = int64_t(g) * kRR;
        const int nr = int(t - s0 < kRR ? t - s0 : kRR);
        // row k's columns start at offset r0 + k of the staged rectangle row
        // ((i0 + s0) mod W mod 4 == (i0 + s0) mod 4 because 4 divides W)
        const int r0 = int((i0 + s0) & 3);
        const float* P = rsm + size_t(st) * kRR * kRB + r0 + j;
        if (nr == kRR) {
#pragma unroll
            for (int k = 0; k < kRR; ++k) acc = acc + P[k * kRB + k];
        } else {
            for (int k = 0; k < nr; ++k) acc = acc + P[k * kRB + k];
        }
        __syncthreads();
    }
    const int64_t i = i0 + j;
    if (kPeer && po.n_wait) {                        // the receivers' readers of row t are done
        if (threadIdx.x == 0)
            for (int k = 0; k < po.n_wait; ++k) wait_flag(po.wait_flag[k], po.wait_value[k]);
        __syncthreads();
    }
    float out = 0.f;
    if (i < a.chunk.hi[0]) {
        const float prev = (kPeer && po.chain) ? __ldcg(ptr<const float>(R, t - 1, i, 0)) : *ptr<const float>(R, t - 1, i, 0);
        const float coef = 0.5f / float(t);
        out = 0.5f * prev + coef * acc;
        *ptr<float>(Wr, t, i, 0) = out;
    }
    if (kPeer && po.flags && po.done) {
        // the row is stored locally: the next row's CTAs may read it
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(po.done, 1u);
        }
    }
    if (kPeer && i < a.chunk.hi[0])
        for (int k = 0; k < po.n; ++k)
            reinterpret_cast<float*>(po.base[k])[(t - po.lo0[k]) * po.n1[k] + (i - po.lo1[k])] = out;
    if (kPeer && po.flags) {
        // every receiver's row lands before its flag: the last CTA publishes them
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned prevc = atomicAdd(po.ctr, 1u);
            if (prevc == po.ctr_last) {
                __threadfence_system();
                for (int k = 0; k < po.n; ++k) st_release_sys(po.flag[k], po.value[k]);
            }
        }
    } else if (kPeer) {
        // the row's gather: every receiver's copy lands before its counter moves
        __threadfence_system();
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned prevc = atomicAdd(po.ctr, 1u);
            if (prevc == gridDim.x - 1) {
                *po.ctr = 0;
                __threadfence_system();
                for (int k = 0; k < po.n; ++k) atomicAdd_system(po.counter[k], 1ull);
            }
        }
    }
}

bool rsim_tensor_map(const DAcc& A, CUtensorMap* out) {
    static EncodeFn enc = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    }
    if (!enc) return false;
    static std::map<std::tuple<const char*, int64_t, int64_t>, CUtensorMap> cache;
    auto key = std::make_tuple(static_cast<const char*>(A.base), A.n[0], A.n[1]);
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    CUtensorMap m;
    const cuuint64_t dims[2] = {cuuint64_t(A.n[1]), cuuint64_t(A.n[0])};
    const cuuint64_t strides[1] = {cuuint64_t(A.n[1]) * 4};
    const cuuint32_t box[2] = {kRB, kRR};
    const cuuint32_t estr[2] = {1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A.base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (cache.size() > 256) cache.clear();
    cache[key] = m;
    *out = m;
    return true;
}


// ------------------------------------------------------------------ integer probe
__device__ uint32_t probe_sum(const DAcc& A, int64_t z, int64_t y, int64_t x) {
    if (A.mode == 3 || A.map == 0)  // read_write or one_to_one: the element itself
        return *at<const uint32_t>(A, z, y, x);
    int64_t lo[3], hi[3];
    if (A.map == 2) {  // all
        for (int d = 0; d < 3; ++d) { lo[d] = 0; hi[d] = A.ext[d]; }
    } else if (A.map == 3) {  // fixed
        for (int d = 0; d < 3; ++d) { lo[d] = A.fixed.lo[d]; hi[d] = A.fixed.hi[d]; }
    } else {  // neighborhood
        const int64_t p[3] = {z, y, x};
        for (int d = 0; d < 3; ++d) {
            lo[d] = p[d] - A.border[d] < 0 ? 0 : p[d] - A.border[d];
            hi[d] = p[d] + A.border[d] + 1 > A.ext[d] ? A.ext[d] : p[d] + A.border[d] + 1;
        }
    }
    uint32_t s = 0;
    for (int64_t a0 = lo[0]; a0 < hi[0]; ++a0)
        for (int64_t a1 = lo[1]; a1 < hi[1]; ++a1)
            for (int64_t a2 = lo[2]; a2 < hi[2]; ++a2) s += *at<const uint32_t>(A, a0, a1, a2);
    return s;
}

__global__ void probe_kernel(const __grid_constant__ KArgs a, int w) {
    const DAcc& O = a.acc[w];
    const DBox& b = O.box;
    const int64_t n1 = b.hi[1] - b.lo[1], n2 = b.hi[2] - b.lo[2];
    const int64_t total = (b.hi[0] - b.lo[0]) * n1 * n2;
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t x = b.lo[2] + t % n2;
        const int64_t y = b.lo[1] + (t / n2) % n1;
        const int64_t z = b.lo[0] + t / (n1 * n2);
        const uint32_t lin = uint32_t((z * O.ext[1] + y) * O.ext[2] + x);
        uint32_t h = fmix32((a.salt + uint32_t(w)) ^ fmix32(lin));
        for (int i = 0; i < a.n_acc; ++i) {
            const DAcc& A = a.acc[i];
            if (A.mode != 1 && A.mode != 3) continue;
            h = fmix32(h ^ probe_sum(A, z, y, x));
        }
        *at<uint32_t>(O, z, y, x) = h;
    }
}

int grid_for(int64_t work, int threads) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = int64_t(num_sms()) * 16;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return int(g);
}

int64_t vol(const DBox& b) {
    int64_t v = 1;
    for (int d = 0; d < 3; ++d) {
        const int64_t e = b.hi[d] - b.lo[d];
        if (e <= 0) return 0;
        v *= e;
    }
    return v;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

void set_copy_blocks_per_sm(int n) { g_copy_blocks_per_sm = n > 0 ? n : 8; }

void launch_oob_init(long long* rec, int n, cudaStream_t s) {
    oob_init_kernel<<<1, 64, 0, s>>>(rec, n);
}

namespace {
EncodeFn encoder() {
    static EncodeFn enc = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
    }
    return enc;
}

// 3-D map of 4-byte words: dims (d0 words, d1, d2), byte strides (p1, p2),
// box (tw, th, 1); cached (halo copies repeat every step)
bool word_map(const char* base, const uint64_t dims[3], const uint64_t strides[2], int tw, int th, CUtensorMap* out) {
    EncodeFn enc = encoder();
    if (!enc) return false;
    using Key = std::tuple<const char*, uint64_t, uint64_t, uint64_t, uint64_t, uint64_t, int, int>;
    static std::map<Key, CUtensorMap> cache;
    const Key key{base, dims[0], dims[1], dims[2], strides[0], strides[1], tw, th};
    auto it = cache.find(key);
    if (it != cache.end()) {
        *out = it->second;
        return true;
    }
    CUtensorMap m;
    const cuuint64_t gd[3] = {dims[0], dims[1], dims[2]};
    const cuuint64_t gs[2] = {strides[0], strides[1]};
    const cuuint32_t box[3] = {cuuint32_t(tw), cuuint32_t(th), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<char*>(base), gd, gs, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return false;
    if (cache.size() > 4096) cache.clear();
    cache[key] = m;
    *out = m;
    return true;
}
}  // namespace

int tma_copy_add(TmaCopyArgs& args, const TmaBox& b) {
    if (b.es % 4 != 0) return 0;
    // the box as dims (planes, rows, words), each with its origin and byte
    // stride in both allocations; normalised by (1) merging a dim into the
    // next inner one where that inner one spans whole rows of both
    // allocations, (2) folding dims of extent 1 into the base addresses
    struct Dim {
        int64_t n, so, dof, ss, ds;
    };
    const int64_t w = int64_t(b.es / 4), es = int64_t(b.es);
    Dim d[3] = {{b.ext[0], b.so[0], b.dof[0], b.sn[1] * b.sn[2] * es, b.dn[1] * b.dn[2] * es},
                {b.ext[1], b.so[1], b.dof[1], b.sn[2] * es, b.dn[2] * es},
                {b.ext[2] * w, b.so[2] * w, b.dof[2] * w, 4, 4}};
    int nd = 3;
    const char* src = b.src;
    char* dst = b.dst;
    for (int k = nd - 2; k >= 0; --k) {            // (1) merge dim k into dim k + 1
        Dim& in = d[k + 1];
        if (in.so == 0 && in.dof == 0 && d[k].ss == in.n * in.ss && d[k].ds == in.n * in.ds) {
            in.so = d[k].so * in.n;
            in.dof = d[k].dof * in.n;
            in.n *= d[k].n;
            for (int j = k; j + 1 < nd; ++j) d[j] = d[j + 1];
            --nd;
        }
    }
    Dim o[3];
    int no = 0;
    for (int k = 0; k < nd; ++k) {                  // (2) fold extent-1 outer dims into the bases
        if (k + 1 < nd && d[k].n == 1) {
            src += d[k].so * d[k].ss;
            dst += d[k].dof * d[k].ds;
        } else {
            o[no++] = d[k];
        }
    }
    if (no == 1) return -1;                         // one run: the LSU kernel is at the copy peak
    if (args.nseg >= kMaxTmaSegs) return 0;
    if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) return 0;
    // TMA order: dim 0 = words (innermost), 1, 2; a missing dim 2 is extent 1
    const Dim& x = o[no - 1];
    const Dim& y = o[no - 2];
    const Dim z = no == 3 ? o[0] : Dim{1, 0, 0, y.ss * (y.so + y.n), y.ds * (y.dof + y.n)};
    for (const Dim* q : {&y, &z})
        if (q->ss % 16 || q->ds % 16 || q->ss >= (int64_t(1) << 40) || q->ds >= (int64_t(1) << 40)) return 0;
    const int64_t W = x.n;
    const int tw = int(W >= 256 ? 256 : (W + 3) / 4 * 4);
    int64_t th = int64_t(kTmTileBytes / 4) / tw;
    if (th > y.n) th = y.n;
    if (th > 256) th = 256;
    // TMA moves the innermost dimension in 16-byte steps: measured on B200, a
    // tile starting at a word that is not a multiple of 4 faulted (illegal
    // instruction) and a store clipped at such a word wrote past it.  So the
    // box must start on 16-byte boundaries of its rows in both allocations and
    // end on one in the destination; other boxes stay on the LSU kernel
    if ((x.so % 4) || (x.dof % 4) || ((x.dof + x.n) % 4) || x.dof + x.n < tw) return 0;
    // maps cut at the box's far corner (the source's rounded up to 16 bytes:
    // what a tile reads beyond the box is never stored): stores beyond it are
    // clipped by TMA
    const int64_t sx = (x.so + x.n + 3) / 4 * 4;
    const uint64_t sd[3] = {uint64_t(sx < tw ? tw : sx), uint64_t(y.so + y.n), uint64_t(z.so + z.n)};
    const uint64_t dd[3] = {uint64_t(x.dof + x.n), uint64_t(y.dof + y.n), uint64_t(z.dof + z.n)};
    const uint64_t ss[2] = {uint64_t(y.ss), uint64_t(z.ss)};
    const uint64_t ds[2] = {uint64_t(y.ds), uint64_t(z.ds)};
    for (int k = 0; k < 3; ++k)
        if (sd[k] >= (uint64_t(1) << 31) || dd[k] >= (uint64_t(1) << 31)) return 0;
    if (ss[1] < ss[0] * sd[1] || ds[1] < ds[0] * dd[1] || ss[0] < 4 * sd[0] || ds[0] < 4 * dd[0]) return 0;
    if (sd[1] < uint64_t(th) || dd[1] < uint64_t(th)) return 0;
    const int s = args.nseg;
    if (!word_map(src, sd, ss, tw, int(th), &args.map[2 * s]) || !word_map(dst, dd, ds, tw, int(th), &args.map[2 * s + 1]))
        return 0;
    TmaSeg& g = args.seg[s];
    g.s0[0] = int32_t(x.so);
    g.s0[1] = int32_t(y.so);
    g.s0[2] = int32_t(z.so);
    g.d0[0] = int32_t(x.dof);
    g.d0[1] = int32_t(y.dof);
    g.d0[2] = int32_t(z.dof);
    g.tw = tw;
    g.th = int32_t(th);
    g.tiles_x = uint32_t((W + tw - 1) / tw);
    g.tiles_y = uint32_t((y.n + th - 1) / th);
    g.planes = uint32_t(z.n);
    g.tiles_begin = args.total_tiles;
    args.total_tiles += uint64_t(g.tiles_x) * g.tiles_y * g.planes;
    args.nseg++;
    return 1;
}

int launch_copy_tma(const TmaCopyArgs& a, cudaStream_t s) {
    if (a.total_tiles == 0 || a.nseg == 0) return 0;
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev >= 0 && dev < 64 && !attr_set[dev]) {   // function attributes are per device
        cudaFuncSetAttribute(copy_kernel_tmap<6, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(6 * kTmTileBytes));
        attr_set[dev] = true;
    }
    // persistent over the tiles, 2 CTAs per SM x 6 stages (3 x 4 measured the same)
    int64_t grid = int64_t(num_sms()) * 2;
    if (int64_t(a.total_tiles) < grid) grid = int64_t(a.total_tiles);
    copy_kernel_tmap<6, 3><<<unsigned(grid), 32, 6 * kTmTileBytes, s>>>(a);
    return 1;
}

int launch_mc_gather(const char* src, char* mc_dst, uint64_t bytes, unsigned long long* mc_flag, unsigned* ctr,
                     cudaStream_t s) {
    const uint64_t units = (bytes / 16 + 255) / 256;
    int64_t grid = int64_t(units ? units : 1);
    if (grid > int64_t(num_sms()) * 4) grid = int64_t(num_sms()) * 4;
    mc_gather_kernel<<<unsigned(grid), 256, 0, s>>>(src, mc_dst, bytes, mc_flag, ctr);
    return 1;
}

int launch_p2p_gather(const P2PGatherArgs& a, cudaStream_t s) {
    const uint64_t units = (a.bytes / 16 + 255) / 256;
    int64_t grid = int64_t(units ? units : 1);
    if (grid > int64_t(num_sms()) * 4) grid = int64_t(num_sms()) * 4;
    p2p_gather_kernel<<<unsigned(grid), 256, 0, s>>>(a);
    return 1;
}

int launch_copy(const CopyArgs& a, cudaStream_t s) {
    if (a.total_units == 0 || a.nseg == 0) return 0;
    // local copies: flat grid (one CTA per unit); peer pushes over NVLink: a
    // persistent grid of 8 CTAs per SM (fewer outstanding remote CTAs measured faster)
    int64_t grid = int64_t(a.total_units);
    if (a.peer && grid > int64_t(num_sms()) * g_copy_blocks_per_sm) grid = int64_t(num_sms()) * g_copy_blocks_per_sm;
    if (grid > (1ll << 31) - 1) grid = (1ll << 31) - 1;
    copy_kernel<<<unsigned(grid), 256, 0, s>>>(a);
    return 1;
}

// Preconditions of the TMA-staged RSim row kernel (see rsim_row_tma_t).
bool rsim_tma_ok(const KArgs& a) {
    const DAcc& R0 = a.acc[0];
    return !(a.variant & kVarRsimRegs) && !a.checked && R0.n[1] == R0.ext[1] && R0.lo[1] == 0 && R0.ext[1] % 4 == 0 &&
           R0.n[2] == 1 && R0.lo[2] == 0 && R0.es == 4 && R0.ext[1] >= 2 * kRB && R0.lo[0] == 0 &&
           (reinterpret_cast<uintptr_t>(R0.base) & 15) == 0 && a.t > 0;
}

// Launch the TMA RSim row kernel, programmatically dependent on the previous
// kernel of the stream (CEL_PDL=0: ordinary stream order).
template <bool kPeer>
void launch_rsim_tma(const CUtensorMap& tm, const KArgs& a, const PeerOut& po, unsigned grid, cudaStream_t s) {
    static int pdl = -1;
    if (pdl < 0) {
        const char* e = getenv("CEL_PDL");
        pdl = (e && e[0] == '0') ? 0 : 1;
    }
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kRC);
    cfg.dynamicSmemBytes = size_t(kRS) * kRR * kRB * sizeof(float);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, rsim_row_tma_t<kPeer>, tm, a, po);
}

bool rsim_fusable(const KArgs& a) {
    CUtensorMap tm;
    return a.kind == K_RSIM_ROW && vol(a.chunk) > 0 && rsim_tma_ok(a) && rsim_tensor_map(a.acc[0], &tm);
}

int launch_rsim_fused(const KArgs& a, const PeerOut& po, cudaStream_t s) {
    CUtensorMap tm;
    if (!rsim_fusable(a) || !rsim_tensor_map(a.acc[0], &tm)) return 0;
    const unsigned grid = unsigned((vol(a.chunk) + kRC - 1) / kRC);
    launch_rsim_tma<true>(tm, a, po, grid, s);
    return 1;
}

int64_t wave5_strip(const KArgs& a, unsigned* gx, unsigned* gy, bool* occ16_out) {
    const DAcc& U = a.acc[0];
    const DAcc& P = a.acc[1];
    const int64_t c0 = a.chunk.lo[1], w = a.chunk.hi[1] - c0;
    const bool vec = !a.checked && U.es == 4 && P.es == 4 && U.n[2] == 1 && P.n[2] == 1 && U.n[1] % 4 == 0 &&
                     P.n[1] % 4 == 0 && (c0 - U.lo[1]) % 4 == 0 && (c0 - P.lo[1]) % 4 == 0 && w % 4 == 0 &&
                     aligned16(U.base) && aligned16(P.base);
    const int64_t rows = a.chunk.hi[0] - a.chunk.lo[0];
    if (!vec || rows <= 0 || w <= 0) return 0;
    // strip height: 8 rows, lowered (>= 4) until the grid has about 8 waves
    // of resident CTAs (r02 sweep, tools/wave_strip.py: 16384 rows 478 us at
    // h = 8 vs 494 at 16; neighbouring strips' halo rows are L2 hits).
    // Chunks of fewer than ~20 waves of 8-row strips at 16 CTAs/SM (the
    // multi-GPU chunks: 8192 / 5462 / 4096 rows at 2 / 3 / 4 GPUs) run the
    // 32-register variant at 16 CTAs/SM, with the lower strip when that gives
    // fewer than 8 waves: 4029 vs 3995 steps/s at 2 B200, 5892 vs 5834 at 3,
    // 7812-7826 vs 7574-7664 at 4; the full 16384-row chunk (27.7 waves)
    // keeps 12 CTAs/SM, where 16 is 4% slower (2002 vs 2082).
    // (A launch-time model picking h = 5 for 4096 rows at 12 CTAs/SM measured
    // 2% slower: short strips cost more than a partial last wave.)
    static int occ = 0, occ16 = 0, force = -1;      // force: CEL_WAVE_OCC=12 / 16 (A/B), else -1
    if (occ == 0) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, wave5_vec, 128, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ16, wave5_vec16, 128, 0);
        if (occ < 1) occ = 1;
        if (occ16 < occ) occ16 = occ;
        const char* e = getenv("CEL_WAVE_OCC");
        force = e ? (atoi(e) == 16 ? 16 : 12) : -1;
    }
    const int64_t cols = (w / 4 + 127) / 128;
    const int64_t h16 = (rows * cols) / (int64_t(num_sms()) * occ16 * 8);
    const bool use16 = force == 16 || (force < 0 && occ16 > occ && h16 < 20);
    int64_t h = use16 ? h16 : (rows * cols) / (int64_t(num_sms()) * occ * 8);
    h = h < 4 ? 4 : (h > kWaveRows ? kWaveRows : h);
    if (occ16_out) *occ16_out = use16;
    static int strip_force = -1;
    if (strip_force < 0) {
        const char* e = getenv("CEL_WAVE_STRIP");           // A/B of the strip height
        strip_force = e ? atoi(e) : 0;
    }
    if (strip_force > 0) h = strip_force;
    *gx = unsigned(cols);
    *gy = unsigned((rows + h - 1) / h);
    return h;
}

int launch_wave5_halo(const KArgs& a, const HaloArgs& hx, cudaStream_t s) {
    unsigned gx = 0, gy = 0;
    bool o16 = false;
    const int64_t h = wave5_strip(a, &gx, &gy, &o16);
    if (h <= 0) return 0;
    KArgs b = a;
    b.strip = int(h);
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(gx, gy);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (o16) cudaLaunchKernelEx(&cfg, wave5_halo16, b, hx);
    else cudaLaunchKernelEx(&cfg, wave5_halo, b, hx);
    return 1;
}

int launch_workload(const KArgs& a, cudaStream_t s) {
    const int64_t cv = vol(a.chunk);
    switch (a.kind) {
    case K_FILL_HASH:
    case K_FILL_CONST: {
        const int64_t work = vol(a.acc[0].box) * (a.acc[0].es / 4);
        if (work == 0) return 0;
        if (a.kind == K_FILL_HASH)
            fill_hash_kernel<<<grid_for(work, 256), 256, 0, s>>>(a);
        else
            fill_const_kernel<<<grid_for(work, 256), 256, 0, s>>>(a);
        return 1;
    }
    case K_STENCIL3:
        if (cv == 0) return 0;
        stencil3_kernel<<<grid_for(cv, 256), 256, 0, s>>>(a);
        return 1;
    case K_WAVE5: {
        if (cv == 0) return 0;
        unsigned gx = 0, gy = 0;
        bool o16 = false;
        const int64_t h = wave5_strip(a, &gx, &gy, &o16);
        if (h > 0) {
            KArgs b = a;
            b.strip = int(h);
            static int pdl = -1;
            if (pdl < 0) {
                const char* e = getenv("CEL_PDL");
                pdl = (e && e[0] == '0') ? 0 : 1;
            }
            cudaLaunchConfig_t cfg;
            memset(&cfg, 0, sizeof cfg);
            cfg.gridDim = dim3(gx, gy);
            cfg.blockDim = dim3(128);
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = pdl ? 1 : 0;
            if (o16) cudaLaunchKernelEx(&cfg, wave5_vec16, b);
            else cudaLaunchKernelEx(&cfg, wave5_vec, b);
        } else {
            wave5_scalar<<<grid_for(cv, 256), 256, 0, s>>>(a);
        }
        return 1;
    }
    case K_JACOBI7: {
        if (cv == 0) return 0;
        const DAcc& A = a.acc[0];
        const DAcc& B = a.acc[1];
        const int64_t x0 = a.chunk.lo[2], w = a.chunk.hi[2] - x0;
        const bool vec = !a.checked && A.es == 4 && B.es == 4 && A.n[2] % 4 == 0 && B.n[2] % 4 == 0 && (x0 - A.lo[2]) % 4 == 0 &&
                         (x0 - B.lo[2]) % 4 == 0 && w % 4 == 0 && aligned16(A.base) && aligned16(B.base);
        static bool attr_set[64] = {};
        CUtensorMap tm;
        if (vec && !(a.variant & kVarJacobiLsu) && A.n[2] % 4 == 0 && jacobi_tensor_map(A, &tm)) {
            int dev = 0;
            cudaGetDevice(&dev);
            if (dev >= 0 && dev < 64 && !attr_set[dev]) {
                cudaFuncSetAttribute(jacobi7_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     int(kJStages * kJStride * sizeof(float)));
                attr_set[dev] = true;
            }
            dim3 grid{unsigned((w + kJBX - 1) / kJBX), unsigned((a.chunk.hi[1] - a.chunk.lo[1] + kJBY - 1) / kJBY),
                      unsigned((a.chunk.hi[0] - a.chunk.lo[0] + kJZS - 1) / kJZS)};
            static int pdl = -1;
            if (pdl < 0) {
                const char* e = getenv("CEL_PDL");
                pdl = (e && e[0] == '0') ? 0 : 1;
            }
            cudaLaunchConfig_t cfg;
            memset(&cfg, 0, sizeof cfg);
            cfg.gridDim = grid;
            cfg.blockDim = dim3(32 * kJBY);
            cfg.dynamicSmemBytes = size_t(kJStages) * kJStride * sizeof(float);
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = pdl ? 1 : 0;
            cudaLaunchKernelEx(&cfg, jacobi7_tma, tm, a);
        } else if (vec) {
            dim3 grid(unsigned((w / 4 + 127) / 128), unsigned(a.chunk.hi[1] - a.chunk.lo[1]),
                      unsigned((a.chunk.hi[0] - a.chunk.lo[0] + kJacZ - 1) / kJacZ));
            jacobi7_vec<<<grid, 128, 0, s>>>(a);
        } else {
            jacobi7_scalar<<<grid_for(cv, 256), 256, 0, s>>>(a);
        }
        return 1;
    }
    case K_NBODY_STEP: {
        if (cv == 0) return 0;
        const int64_t n = a.chunk.hi[0] - a.chunk.lo[0];
        if (a.fast && !a.checked)
            nbody_step_fast_x2_kernel<<<unsigned((n + kNbTile - 1) / kNbTile), 128, 0, s>>>(a);
        else
            nbody_step_kernel<<<unsigned((n + kNbTile - 1) / kNbTile), kNbTile, 0, s>>>(a);
        return 1;
    }
    case K_NBODY_UPDATE:
        if (cv == 0) return 0;
        nbody_update_kernel<<<grid_for(cv, 256), 256, 0, s>>>(a);
        return 1;
    case K_RSIM_ROW: {
        if (cv == 0) return 0;
        const DAcc& R0 = a.acc[0];
        if (a.checked) {
            rsim_row_checked<<<grid_for(cv, 128), 128, 0, s>>>(a);
            return 1;
        }
        CUtensorMap tm;
        if (rsim_tma_ok(a) && rsim_tensor_map(R0, &tm)) {
            const unsigned grid = unsigned((cv + kRC - 1) / kRC);
            PeerOut none;
            memset(&none, 0, sizeof none);
            launch_rsim_tma<false>(tm, a, none, grid, s);
            return 1;
        }
        rsim_row_kernel<16><<<grid_for(cv, 128), 128, 0, s>>>(a);
        return 1;
    }
    case K_PROBE: {
        int n = 0;
        for (int w = 0; w < a.n_acc; ++w) {
            if (a.acc[w].mode != 2 && a.acc[w].mode != 3) continue;
            const int64_t work = vol(a.acc[w].box);
            if (work == 0) continue;
            probe_kernel<<<grid_for(work, 128), 128, 0, s>>>(a, w);
            ++n;
        }
        return n;
    }
    default:
        return 0;
    }
}

}  // namespace cel
