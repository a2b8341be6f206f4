// Device kernels of the coherence path (sm_100a).  Launch wrappers are
// called by the executor; no torch types anywhere.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace cel {

// ---- copy instruction (Table 1 `copy`): a region = several boxes,
// each lowered to a strided segment  planes x rows x row_bytes.
struct CopySeg {
    const char* src;
    char* dst;
    uint64_t row_bytes;
    uint64_t src_row_stride, dst_row_stride;
    uint64_t src_plane_stride, dst_plane_stride;
    uint32_t rows, planes;
    uint64_t units_begin;      // prefix sum of work units (exclusive)
    uint32_t units_per_row;
    uint32_t vec;              // 16, 8, 4, 2 or 1 byte accesses
    uint32_t narrow;           // > 0: rows of <= kNarrowBytes, a unit = `narrow` whole rows, one per thread
};

constexpr int kMaxSegs = 24;
constexpr uint64_t kNarrowBytes = 256;     // rows this short are packed 256 per CTA (e.g. column halos)
constexpr uint32_t kCopyUnit = 8192;      // bytes of one row chunk = one CTA (256 threads x 2 x 16 B)

struct CopyArgs {
    CopySeg seg[kMaxSegs];
    int nseg;
    int peer;                  // destination is another GPU's memory: fence before exit
    uint64_t total_units;
};

// ---- TMA tensor-map copy of strided boxes (north_star: "TMA tensor-map box
// loads and stores for 2D/3D strided regions").  Each box of a copy region is
// described by two 3-D tensor maps of 4-byte words, one over the source and
// one over the destination allocation, both cut at the box's far corner (TMA
// stores clip there, so a tile hanging over the box edge never writes outside
// it); a tile is (tw words x th rows x 1 plane), moved global -> shared ->
// global by cp.async.bulk.tensor (SASS UTMALDG / UTMASTG).
constexpr int kMaxTmaSegs = 8;
struct TmaSeg {
    int32_t s0[3];             // box origin in the source map (words, rows, planes)
    int32_t d0[3];             // box origin in the destination map
    uint32_t tiles_x, tiles_y, planes;
    int32_t tw, th;            // tile = tensor-map box (tw words, th rows, 1 plane)
    uint64_t tiles_begin;      // prefix sum of tiles (exclusive)
};
struct TmaCopyArgs {
    CUtensorMap map[2 * kMaxTmaSegs];   // 2 s: source of segment s, 2 s + 1: its destination
    TmaSeg seg[kMaxTmaSegs];
    int nseg;
    uint64_t total_tiles;
};
// One strided box of a local copy: allocation bases (16-byte aligned), their
// extents and the box (planes, rows, elements), element size (multiple of 4).
struct TmaBox {
    const char* src;
    char* dst;
    int64_t sn[3], dn[3];      // allocation extents (planes, rows, elements)
    int64_t so[3], dof[3];     // box origin inside each allocation
    int64_t ext[3];            // box extent
    uint32_t es;
};
// Adds the box to args (encoding / reusing its tensor maps): 1 added; -1 the
// box is one contiguous run (not strided: left to the LSU kernel); 0 TMA
// cannot express it (alignment, pitch or size limits) or args is full.
int tma_copy_add(TmaCopyArgs& args, const TmaBox& b);
int launch_copy_tma(const TmaCopyArgs& a, cudaStream_t s);

// NVLS all-gather: `bytes` (multiple of 4; src and mc_dst
// 16-byte aligned) from this device's chunk to the multicast address of the
// set's allocations; the last CTA then adds 1 to the multicast flag (release,
// system scope).  ctr: a zeroed per-device word the CTAs count on.
int launch_mc_gather(const char* src, char* mc_dst, uint64_t bytes, unsigned long long* mc_flag, unsigned* ctr,
                     cudaStream_t s);

// P2P all-gather (SURVEY §8 a7 / §8(e) "P2P stores over NVSwitch"): one
// source's chunk stored into every receiver's allocation (peer pointers:
// another GPU's memory over NVLink, IPC-mapped in multi-process runs); the
// last CTA then adds 1 (system scope) to each receiver's gather counter.
constexpr int kMaxGatherDst = 15;
struct P2PGatherArgs {
    const char* src;
    char* dst[kMaxGatherDst];
    unsigned long long* counter[kMaxGatherDst];
    int ndst;
    uint64_t bytes;            // multiple of 4; src and every dst 16-byte aligned, or 4-byte with vec4 = 0
    int vec4;
    unsigned* ctr;             // zeroed word of the source device: CTAs done
};
int launch_p2p_gather(const P2PGatherArgs& a, cudaStream_t s);



// ---- accessor (allocation pointer interpolated into the accessor)
struct DBox {
    int64_t lo[3], hi[3];
};

struct DAcc {
    char* base;                // allocation base
    int64_t lo[3];             // allocation box min
    int64_t n[3];              // allocation box extent
    int64_t ext[3];            // buffer extent
    uint32_t es;               // element size in bytes
    int mode;                  // 1 read, 2 write, 3 read_write
    int map;                   // mapper kind
    int64_t border[3];
    DBox fixed;
    DBox box;                  // mapped box of this access for the chunk
    long long* oob;            // accessor bounds checking (§4.4): [min z,y,x, max+1 z,y,x] of
                               // accesses outside `box`, or null when checking is off
};

constexpr int kMaxAcc = 6;

struct KArgs {
    int kind;
    int n_acc;
    DBox chunk;
    uint64_t seed;
    float value;
    uint32_t t;
    uint32_t salt;
    int fast;                  // fast-math variant (FMA + rsqrt) of ALU-bound kernels
    int strip;                 // rows per CTA of the stencil kernels (0 = default)
    int checked;               // bounds checking: scalar kernels whose accesses go through at()
    int variant;               // A/B switches of the runtime (Executor: CEL_JACOBI / CEL_RSIM env):
                               // kVarJacobiLsu, kVarRsimRegs
    DAcc acc[kMaxAcc];
};

constexpr int kVarJacobiLsu = 1;   // 3-D 7-point: LSU register-window kernel instead of TMA
constexpr int kVarRsimRegs = 2;    // RSim row: register kernel instead of the TMA-staged one

// kernel kinds (mirror include/cel.h cel_kernel)
enum : int {
    K_FILL_HASH = 0,
    K_FILL_CONST = 1,
    K_STENCIL3 = 2,
    K_WAVE5 = 3,
    K_JACOBI7 = 4,
    K_NBODY_STEP = 5,
    K_NBODY_UPDATE = 6,
    K_RSIM_ROW = 7,
    K_PROBE = 8,
    K_CALLBACK = 9,
    K_NUM = 10,
};

// Work units of a segment (fields src .. vec set): a unit is one <= kCopyUnit
// chunk of a row, or, for many short rows, 256 whole rows (one per thread).
inline uint64_t seg_units(CopySeg& g) {
    const uint64_t nrows = uint64_t(g.rows) * g.planes;
    if (g.row_bytes <= kNarrowBytes && nrows >= 64) {
        g.narrow = 256;
        g.units_per_row = 0;
        return (nrows + g.narrow - 1) / g.narrow;
    }
    g.narrow = 0;
    g.units_per_row = uint32_t((g.row_bytes + kCopyUnit - 1) / kCopyUnit);
    return uint64_t(g.units_per_row) * nrows;
}

// Returns the number of kernel launches issued (0 if nothing to do).
int launch_copy(const CopyArgs& a, cudaStream_t s);
// bounds-check records: n accessors x [min z,y,x = +inf, max z,y,x = -inf]
void launch_oob_init(long long* rec, int n, cudaStream_t s);
int launch_workload(const KArgs& a, cudaStream_t s);

void set_copy_blocks_per_sm(int n);

// RSim row kernel with the row's all-gather fused into its epilogue: each
// thread also stores its element into every receiver's allocation (same
// buffer coordinates, the receiver's allocation layout), then the last CTA
// bumps each receiver's gather counter -- the P2P gather without its own
// launch.  Used by the executor when a row kernel is followed by the gather
// set of the row it writes (exec_fuse.cu).
struct PeerOut {
    int n;
    char* base[kMaxGatherDst];
    int64_t lo0[kMaxGatherDst], lo1[kMaxGatherDst], n1[kMaxGatherDst];   // receiver allocation box (rows, cols)
    unsigned long long* counter[kMaxGatherDst];
    unsigned* ctr;
    // flag mode (exec_halo.cu, one process per GPU): the outputs are plain
    // coherence copies -- the last CTA writes each receiver's flag slot with
    // the copy's id instead of bumping a gather counter -- and the incoming
    // copies of the rows this kernel reads are awaited in the kernel
    int flags;
    unsigned long long* flag[kMaxGatherDst];
    unsigned long long value[kMaxGatherDst];
    int n_wait;                                    // flags awaited before the (remote) writes: WAR dependencies
    const unsigned long long* wait_flag[kMaxGatherDst];
    unsigned long long wait_value[kMaxGatherDst];
    int n_in;                                      // incoming copies: awaited before loading rows >= in_row0
    const unsigned long long* in_flag[kMaxGatherDst];
    unsigned long long in_value[kMaxGatherDst];
    int64_t in_row0;                               // the lowest row they write
    unsigned ctr_last;                             // flag mode: CTA counter value before the last CTA's increment
    // row chain (flag mode): every CTA counts itself into *done once its row
    // is stored locally; a chained launch waits for *done >= done_wait (the
    // previous row's CTAs) instead of for the whole previous grid, so this
    // row runs while the previous one's CTAs wait for their NVLink stores
    unsigned* done;
    unsigned done_wait;
    int chain;
};
bool rsim_fusable(const KArgs& a);                       // the TMA row kernel applies (it carries the epilogue)
int launch_rsim_fused(const KArgs& a, const PeerOut& po, cudaStream_t s);

// WaveSim halo exchange fused into the stencil (exec_halo.cu; SURVEY §7 step
// 6, NEXT-2).  Outgoing: coherence copies of rows this launch writes, stored
// by the CTAs that compute them straight into the receiver's allocation (peer
// memory over NVLink), after the copies' remote dependencies (war flags); the
// last CTA of each copy writes the receiver's flag slot.  Incoming: copies
// into rows the launch reads, awaited by the CTAs that read them (flag slots
// in this device's memory), not by the stream.
constexpr int kHaloMax = 4;
struct HaloArgs {
    int n_out;
    char* base[kHaloMax];                          // receiver allocation
    int64_t lo0[kHaloMax], lo1[kHaloMax], n1[kHaloMax];   // its box origin (rows, cols), row pitch (elements)
    int64_t r0[kHaloMax], r1[kHaloMax];            // rows copied, all chunk columns
    unsigned long long* flag[kHaloMax];            // receiver's signal slot for the copy (peer memory)
    unsigned long long value[kHaloMax];            // the copy's instruction id
    unsigned* ctr[kHaloMax];                       // this device's CTA counter of copy i
    unsigned ctr_last[kHaloMax];                   // counter value before the last CTA's increment
    int n_war;
    const unsigned long long* war_flag[kHaloMax];  // remote dependencies of the outgoing copies
    unsigned long long war_value[kHaloMax];
    int n_in;
    const unsigned long long* in_flag[kHaloMax];   // incoming copies: flag slot, instruction id,
    unsigned long long in_value[kHaloMax];
    int64_t in_r0[kHaloMax], in_r1[kHaloMax];      // rows they write
};
// strip height and grid of the vectorised wave5 launch for this chunk (0 rows
// if the vector kernel does not apply)
int64_t wave5_strip(const KArgs& a, unsigned* gx, unsigned* gy, bool* occ16 = nullptr);
int launch_wave5_halo(const KArgs& a, const HaloArgs& h, cudaStream_t s);

}  // namespace cel
