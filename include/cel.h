/*
 * cel.h — C-ABI of the B200-native Celerity instruction-graph coherence path
 * (Knorr et al., "Concurrent Scheduling of High-Level Parallel Programs on
 * Multi-GPU Systems", arXiv 2503.10516).
 *
 * The calls follow the paper's user model (§2): a
 * queue to which tasks are submitted; each task launches one kernel over an
 * index space and declares accesses to virtual buffers through range mappers;
 * epochs synchronise with the caller.  Behind the calls the library
 * splits each task over the devices (§3.1), evaluates the range
 * mappers, diffs the per-device read/write regions against the buffers'
 * up-to-date / original-producer region maps (§3.3), generates
 * alloc / resize-copy / copy / free / kernel / horizon / epoch instructions
 * (Table 1; §3.2; §3.5) with the lookahead
 * of §4.3, and executes them on B200 (sm_100a): copies by SM
 * kernels (peer pushes over NVLink/NVSwitch), kernels on per-device streams.
 *
 * Conventions
 *   - Boxes are half-open [min, max) in 3 dimensions; dimensions beyond a
 *     buffer's `dims` are [0, 1).  Dimension 0 is the slowest (row-major).
 *   - Buffers are dense row-major arrays of `elem_size`-byte elements.
 *   - Status: 0 = OK; > 0 = warning (the call took effect); < 0 = error (the
 *     call had no effect, except CEL_E_CUDA / CEL_E_OOM during execution,
 *     which poison the runtime: every later call except cel_runtime_destroy
 *     returns the same error).  cel_last_error() gives a thread-local message.
 *   - All calls on one runtime come from one thread (Celerity's single user
 *     thread).  Pointers passed in are only read during the call
 *     unless stated otherwise.
 */
#ifndef CEL_H
#define CEL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CEL_OK 0
#define CEL_W_UNINIT_READ 1          /* §4.4 uninitialised-read warning */
#define CEL_E_INVALID (-1)           /* malformed argument */
#define CEL_E_OUT_OF_BOUNDS (-2)     /* one_to_one chunk / fixed / remap box outside the buffer */
#define CEL_E_OVERLAPPING_WRITE (-3) /* §4.4 overlapping-write error */
#define CEL_E_OOM (-4)               /* device arena or pinned host memory exhausted (sticky) */
#define CEL_E_CUDA (-5)              /* CUDA error, or no GPU (sticky) */
#define CEL_E_NCCL (-6)
#define CEL_E_STATE (-7)             /* call not valid in this state (e.g. after shutdown) */

typedef struct cel_runtime cel_runtime; /* opaque: owns all device memory, streams, events */
typedef uint32_t cel_buffer;
typedef uint64_t cel_task;

typedef struct {
    uint64_t min[3];
    uint64_t max[3];
} cel_box;

/* Range mappers (R5 of DESIGN.md):
 *   ONE_TO_ONE   buffer region = kernel chunk (error if outside the buffer)
 *   NEIGHBORHOOD chunk inflated by border[d] per dim, clamped to the buffer
 *   ALL          the whole buffer ("always spans the entire buffer range")
 *   FIXED        the box `fixed` regardless of the chunk
 *   REMAP        buffer dim k takes the chunk's interval of kernel dim
 *                from_kernel_dim[k], or fixed's interval if that is -1
 *                (e.g. RSim "append row t": fixed=[t,t+1)x., map={-1,0,-1}) */
/* CEL_NEIGHBORHOOD_AXES: the axis-only neighbourhood -- the chunk inflated by
 * border[d] along one dimension d at a time (a cross, no corners), e.g. a
 * 5-point stencil; the allocation still spans the cross's bounding box. */
typedef enum {
    CEL_ONE_TO_ONE = 0,
    CEL_NEIGHBORHOOD = 1,
    CEL_ALL = 2,
    CEL_FIXED = 3,
    CEL_REMAP = 4,
    CEL_NEIGHBORHOOD_AXES = 5
} cel_mapper_kind;

typedef struct {
    int32_t kind;              /* cel_mapper_kind */
    uint32_t border[3];        /* NEIGHBORHOOD */
    cel_box fixed;             /* FIXED, REMAP */
    int32_t from_kernel_dim[3];/* REMAP */
} cel_range_mapper;

typedef enum { CEL_READ = 1, CEL_WRITE = 2, CEL_READ_WRITE = 3 } cel_mode;
typedef enum { CEL_SPLIT_1D = 0, CEL_SPLIT_2D = 1 } cel_split; /* §3.1 split along dim 0, or dims 0 and 1 */

typedef struct {
    cel_buffer buf;
    int32_t mode;              /* cel_mode */
    cel_range_mapper map;
} cel_access;

/* Built-in sm_100a device kernels (synthetic workloads); the
 * accessor order each expects is given in brackets.  CALLBACK calls `fn`. */
typedef enum {
    CEL_K_FILL_HASH = 0,   /* [write]               word w of element x = init(seed, lin(x)*words+w) */
    CEL_K_FILL_CONST = 1,  /* [write]               every 32-bit word = value */
    CEL_K_STENCIL3 = 2,    /* [read nbhd(1), write]  1-D 3-point (Listing 5 shape) */
    CEL_K_WAVE5 = 3,       /* [read u nbhd(1,1), read_write up] WaveSim 5-point leapfrog */
    CEL_K_JACOBI7 = 4,     /* [read nbhd(1,1,1), write] 3-D 7-point */
    CEL_K_NBODY_STEP = 5,  /* [read P all, read_write V] float4 bodies */
    CEL_K_NBODY_UPDATE = 6,/* [read V, read_write P] */
    CEL_K_RSIM_ROW = 7,    /* [read fixed rows [0,t), write remap row t] */
    CEL_K_PROBE = 8,       /* u32 coherence probe, any accessors, one written */
    CEL_K_CALLBACK = 9
} cel_kernel;

/* What a kernel sees of one accessor: its backing allocation. */
typedef struct {
    void* base;                /* device pointer of the allocation (element alloc_box.min) */
    cel_box alloc_box;         /* buffer box the allocation covers, dense row-major */
    uint32_t elem_size;
    cel_box range;             /* the range mapper's region for this chunk: what the kernel may access */
    long long* oob;            /* bounds checking on (cel_config.bounds_check): device record
                                  [min z,y,x, max+1 z,y,x] of accesses outside `range`, to be
                                  updated with cel_check_access() (include/cel_device.cuh);
                                  NULL when off */
} cel_accessor;

/* User kernel: called on the scheduling thread with the device's stream; it
 * must only enqueue work on `cuda_stream` (a cudaStream_t). */
typedef void (*cel_kernel_fn)(void* user, int device, const cel_box* chunk, const cel_accessor* acc, int n_acc,
                              void* cuda_stream);

typedef struct {
    uint64_t seed;             /* FILL_HASH */
    float value;               /* FILL_CONST */
    uint32_t t;                /* RSIM_ROW: row index */
    uint32_t salt;             /* PROBE */
} cel_kernel_params;

typedef struct {
    int32_t dims;              /* kernel index space dimensionality 1..3 */
    cel_box range;             /* kernel index space */
    int32_t split;             /* cel_split */
    int32_t kernel;            /* cel_kernel */
    cel_kernel_params params;
    cel_kernel_fn fn;          /* CALLBACK only; must outlive the task */
    void* fn_user;
    const cel_access* acc;     /* n_acc accessors, copied during the call */
    int32_t n_acc;
} cel_task_desc;

typedef struct {
    const int* cuda_devices;   /* physical CUDA device of each virtual device; repeats allowed
                                  (several virtual devices on one GPU); NULL = 0..n_devices-1 */
    int32_t n_devices;         /* G: devices the work is split over */
    int32_t execute;           /* 0 = generate the instruction graph only (no GPU touched) */
    int32_t lookahead;         /* 0 none, 1 auto (default), 2 infinite */
    int32_t horizon_step;      /* critical-path horizon step (R7), default 4 */
    int32_t checks;            /* §4.4 checks (uninitialised read, overlapping write) */
    const char* instr_log_path;/* JSONL instruction log (one record per instruction) or NULL */
    uint64_t arena_bytes;      /* device memory reserved per device; 0 = 16 GiB */
    int32_t rank;              /* multi-process: this process's rank; device `rank` is its own */
    int32_t world;             /* multi-process: number of processes (= n_devices), 1 = single process */
    int32_t fast_math;         /* 1: ALU-bound kernels (N-body) use FMA + rsqrt; results then match the
                                  oracle within a tolerance instead of bit for bit (R16) */
    int32_t collective;        /* 1: a task's all-gather copy set (buffer read through `all` / `fixed`,
                                  every device receiving every other device's contiguous chunk; SURVEY
                                  §8 a7) runs as one group of NCCL broadcasts when the
                                  devices are distinct GPUs; 0: as peer pushes.  The instruction graph
                                  is the same either way.  NCCL (libnccl.so.2) is opened at run time;
                                  a failed communicator setup is CEL_E_NCCL (sticky). */
    int32_t bounds_check;      /* §4.4 accessor bounds checking: kernels run their
                                  scalar variants, every element access is checked against the
                                  range mapper's region, and the bounding box of the accesses
                                  outside it is reported after the kernel exits as a sticky
                                  CEL_E_OUT_OF_BOUNDS error ("task T device D accessor A ...").
                                  Debug aid: slower kernels, results unchanged. */
    int32_t n_nodes;           /* virtual-node mode (§3.4, §4.2): > 1 runs
                                  n_nodes node schedulers of n_devices devices each in this process;
                                  cuda_devices then lists n_nodes * n_devices entries (node-major).
                                  Nodes exchange data only through push / await-push commands lowered
                                  to send, receive, split receive and await receive instructions
                                  staged in pinned host memory (M1), with pilot messages and receive
                                  arbitration.  Node k's instruction log goes to
                                  "<instr_log_path>.<k>"; readbacks gather on node 0.
                                  Each node's M1 arena is arena_bytes of pinned host
                                  memory (256 MiB when arena_bytes is 0).
                                  0 or 1 = one node (the default). */
} cel_config;

/* Counters since runtime creation.  Instruction counts are the node's IDAG
 * (every rank of a multi-process run replays the whole node's graph); executor
 * counters are this process's.  Virtual-node mode: totals over the nodes. */
typedef struct cel_stats_s {
    uint64_t n_alloc, n_free, n_copy, n_kernel, n_horizon, n_epoch;
    uint64_t copies_resize, copies_coherence, copies_readback;
    uint64_t bytes_resize, bytes_coherence, bytes_readback, bytes_d2d_peer;
    uint64_t alloc_bytes_peak;
    uint64_t flushes;          /* lookahead queue flushes */
    uint64_t kernel_launches;  /* CUDA kernels launched by this process (workload + copy) */
    uint64_t copy_launches, memcpy_calls, event_waits, remote_waits, signals, host_syncs;
    uint64_t gen_ns;           /* host time spent in scheduling + issue (incl. epoch waits) */
    uint64_t exec_ns_alloc, exec_ns_free, exec_ns_copy, exec_ns_kernel, exec_ns_horizon, exec_ns_epoch;
                               /* host time of the executor per instruction kind (part of gen_ns) */
    uint64_t signal_ns, remote_wait_ns; /* host time in cross-process flag writes / waits */
    uint64_t copies_elided, bytes_elided; /* resize copies made no-ops by in-place allocation growth */
    uint64_t coll_groups, coll_copies;    /* all-gather copy sets run as NCCL collectives, and their copies */
    uint64_t gather_sets;                 /* coherence copy sets the scheduler found to be all-gathers */
    uint64_t n_send, n_receive, n_split_receive, n_await_receive;   /* virtual-node mode (n_nodes > 1) */
    uint64_t pulls, pull_bytes;           /* virtual-node mode: pilot-matched transfers executed, bytes */
    uint64_t coll_allgathers;             /* all-gather sets run as one in-place ncclAllGather */
    uint64_t tma_copy_launches;           /* copy launches of the TMA tensor-map kernel (strided boxes) */
    uint64_t vmm_maps, vmm_mapped_bytes;  /* VMM allocations: physical granules mapped (creation + in-place growth) */
    uint64_t coll_multicast;              /* all-gather sets run as NVLS multicast stores (CEL_COLL_MC=1) */
    uint64_t staging_elided;              /* virtual-node mode: push staging copies (device -> M1) not executed:
                                             their sends published the device allocation (device-direct) */
    uint64_t staging_materialized;        /* ... of which executed late (their M1 bytes were needed after all) */
    uint64_t coll_p2p;                    /* all-gather sets run as P2P gather kernels (stores into every receiver) */
    uint64_t coll_fused;                  /* ... fused into the RSim row kernels that produce them */
    uint64_t halo_fused;                  /* coherence copies stored by the stencil launch that writes their rows */
    uint64_t halo_in_waits;               /* incoming copies awaited by the reading CTAs of a fused launch */
    uint64_t halo_chained;                /* fused RSim rows that waited for the previous row's local stores, not its grid */
    uint64_t memo_hits, memo_misses;      /* task compiles replayed from the steady-state memo / recorded into it
                                             (CEL_SCHED_MEMO=0 disables it; the instructions are the same) */
} cel_stats_t;

/* Create a runtime.  With execute != 0 every device reserves arena_bytes of
 * device memory and gets its own streams; peer access is enabled between
 * distinct GPUs.  Fails with CEL_E_CUDA if no GPU is visible. */
int cel_runtime_create(const cel_config* cfg, cel_runtime** out);

/* Multi-process (world > 1, one process per GPU): export this rank's blob
 * (cel_ipc_blob_size() bytes into blob: the arena's CUDA IPC handle and, from
 * rank 0, the NCCL unique id of the all-gather communicator), then import every
 * other rank's before submitting work.  Copies into another rank's memory are
 * pushed by SM stores over NVLink; cross-process dependencies are flags in GPU
 * memory; the communicator is built when the first all-gather set executes. */
size_t cel_ipc_blob_size(void);
int cel_ipc_export(cel_runtime* rt, void* blob);
int cel_ipc_import(cel_runtime* rt, int32_t rank, const void* blob);

/* Virtual buffer: only the parts the devices access are ever
 * allocated.  host_init (nullable) holds extent[0]*..*extent[dims-1]*elem_size
 * bytes and is copied before the call returns. */
int cel_buffer_create(cel_runtime* rt, int32_t dims, const uint64_t extent[3], uint32_t elem_size,
                      const void* host_init, cel_buffer* out);

/* Same, with flags.  CEL_BUFFER_BORROW_HOST: host_init is NOT copied; the
 * caller keeps it valid and unmodified until the buffer is destroyed (or the
 * runtime is); page-locked memory is then uploaded by DMA at full speed with
 * no staging copy and no pinning cost. */
#define CEL_BUFFER_BORROW_HOST 1u
int cel_buffer_create_ex(cel_runtime* rt, int32_t dims, const uint64_t extent[3], uint32_t elem_size,
                         const void* host_init, uint32_t flags, cel_buffer* out);

/* Submit a task ("submit command groups to a queue"; one kernel
 * over desc->range with the accessors' range mappers).  The task
 * is split over the devices (§3.1), checked (§4.4) and
 * lowered to instructions (§3.2-3.5) that are issued to the GPUs before the
 * call returns; it does not wait for them (asynchronous).  desc and
 * desc->acc are copied; *out (nullable) receives the task id.
 * Returns 0, or CEL_W_UNINIT_READ (>0, accepted: a read of never-written
 * elements), or <0 with no effect: CEL_E_INVALID (malformed desc),
 * CEL_E_OUT_OF_BOUNDS (one_to_one / fixed / remap region outside a buffer),
 * CEL_E_OVERLAPPING_WRITE (two devices write the same element), or
 * the runtime's sticky error. */
int cel_task_submit(cel_runtime* rt, const cel_task_desc* desc, cel_task* out);

/* Epoch: flush the lookahead queue, block until all work is done. */
int cel_wait(cel_runtime* rt);

/* Read back `box` of a buffer into host_dst (dense row-major over box,
 * elem_size bytes per element, caller-owned, written before the call
 * returns): coherence copies into host memory (§3.3, the user
 * pointer acting as an M0 allocation over `box`; R13) followed by an epoch
 * (P:L304); blocking.  Elements never written and not host-initialised are
 * left untouched.  Multi-process: only the elements whose up-to-date copy
 * lives on this rank's device are written.  CEL_E_INVALID: unknown buffer or
 * null pointer; CEL_E_OUT_OF_BOUNDS: box outside the buffer. */
int cel_buffer_read(cel_runtime* rt, cel_buffer buf, const cel_box* box, void* host_dst);

/* Drop the buffer: its allocations are freed once the last user has finished. */
int cel_buffer_destroy(cel_runtime* rt, cel_buffer buf);

/* Counters (cel_stats_t above) into *out; the executor's counters are as of
 * the last epoch or a few hundred instructions ago.  cel_stats_get is the
 * round-1 name of the same call. */
int cel_stats(cel_runtime* rt, cel_stats_t* out);
int cel_stats_get(cel_runtime* rt, cel_stats_t* out);

/* Device-time profile of the kernels this process launched, measured with
 * CUDA events on the launching streams: ms[k], count[k] for k = cel_kernel
 * kinds 0..9, k = 10 for copy kernels within one GPU (resize, copies between
 * virtual devices of one GPU), k = 11 for peer pushes to another GPU and
 * k = 12 for the boundary (shell) launches of stencil kernels that are split
 * for halo overlap (their interiors count under the kernel's kind) and k = 13
 * for NCCL all-gather groups (per device, broadcast group start to end).
 * n = array length (14).  cel_profile_enable(rt, k): k = 0 off, k >= 1 times
 * every k-th launch of each kind (count[] = timed launches, so ms/count stays
 * the average launch duration with 1/k of the event overhead). */
int cel_profile_enable(cel_runtime* rt, int32_t on);
int cel_profile_read(cel_runtime* rt, double* ms, uint64_t* count, int32_t n);

/* Write the launches profiled since cel_profile_enable(rt, 1) as JSONL, one
 * record per launch: {"iid", "rank", "device", "stream", "kind", "start_us",
 * "end_us"} with times from CUDA events relative to the enable call, per
 * device (the instruction trace of SURVEY §5 / S:L528). */
int cel_trace_dump(cel_runtime* rt, const char* path);

/* Shutdown epoch, free everything. */
int cel_runtime_destroy(cel_runtime* rt);

const char* cel_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CEL_H */
