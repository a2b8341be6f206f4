// Instruction executor (§4.1 "Out-of-Order Instruction Dispatch").
//
// The paper's out-of-order engine issues an instruction *directly* when its
// dependencies are complete or *eagerly* when all incomplete dependencies sit
// on the same in-order queue.  On B200 the in-order queues are CUDA streams and
// cross-queue dependencies become cudaStreamWaitEvent, so every instruction is
// issued eagerly at generation time: a dependency on the same stream costs
// nothing, one on another stream of this process costs one event wait, one on
// a device owned by another process (one process per GPU) costs a stream
// memory-op wait on a flag that the producer's process writes into this GPU's
// memory over NVLink.  The host only blocks at epochs and when too
// many events are in flight.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <array>
#include <deque>
#include <functional>
#include <mutex>
#include <tuple>
#include <thread>
#include <map>
#include <memory>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "kernels.cuh"
#include "sched.hpp"

namespace cel {

// completion token of an instruction: per local stream the sequence number of
// the event recorded after it, plus (rank, iid) pairs whose completion another
// process signals.
struct TokEntry {
    int stream;
    uint64_t seq;
    cudaEvent_t ev;
};
struct Token {
    std::vector<TokEntry> local;
    std::vector<std::pair<int, uint64_t>> remote;
    bool empty() const { return local.empty() && remote.empty(); }
};

// Virtual-node mode: the "communicator" between the node
// executors of one process.  Pilots arrive from the schedulers at
// compile time; a send publishes its staged M1 box and the event
// after its staging copy.  Receive arbitration happens on the receiver's
// executor thread: a receive (or await receive) waits until the pilots covering
// its region have arrived and their sends have been issued, then pulls each box
// into its M1 allocation with a copy kernel on its own stream; completion is
// "as soon as its subregion or a superset thereof has been received".
// A send completes with the pull of its box; the sender resolves that event
// lazily, when an instruction depending on the send is issued.  No GPU-side
// waits on flags: every cross-node edge is an event of a pull already issued
// (host-side ordering by task order keeps this deadlock-free).
class Communicator {
public:
    struct Mem {
        char* base = nullptr;   // device-accessible (pinned + mapped host) allocation base
        Box box;                // allocation box, row-major
        uint32_t es = 0;
    };
    explicit Communicator(int nodes) : nodes_(nodes) {}
    void add_pilot(const Pilot& p);
    void post_send(int node, uint64_t msg, const Mem& src, cudaEvent_t ready);
    // receiver thread: pull every pilot of transfer (node, tid, buf) that
    // intersects `reg` and was not pulled yet into `dst`, on `stream`
    int pull_region(int node, int64_t tid, uint32_t buf, const Region& reg, const Mem& dst, cudaStream_t stream);
    // sender thread: event after the pull of (node, msg); blocks until issued
    cudaEvent_t wait_pulled(int node, uint64_t msg);
    uint64_t pulls() const { return pulls_; }
    uint64_t pull_bytes() const { return pull_bytes_; }
    void abort();                               // wake blocked threads on shutdown / error

private:
    using Key = std::tuple<int, int64_t, uint32_t>;     // (receiver, tid, buffer)
    struct PilotRec {
        int sender;
        uint64_t msg;
        Box box;
        bool pulled = false;
    };
    struct Send {
        Mem src;
        cudaEvent_t ready = nullptr;
    };
    std::mutex m_;
    std::condition_variable cv_;
    int nodes_;
    bool abort_ = false;
    std::map<Key, std::vector<PilotRec>> pilots_;
    std::map<std::pair<int, uint64_t>, Send> sends_;          // posted, not yet pulled
    std::map<std::pair<int, uint64_t>, cudaEvent_t> pulled_;  // pull done events, until the sender takes them
    uint64_t pulls_ = 0, pull_bytes_ = 0;
};

struct ExecConfig {
    std::vector<int> cuda_devices;     // physical device of each virtual device
    int rank = 0, world = 1;           // world > 1: device d is owned by rank d
    uint64_t arena_bytes = 0;          // per device; 0 = auto
    bool profile = false;
    bool fast_math = false;
    bool collective = true;            // run all-gather copy sets as grouped NCCL broadcasts (§8 a7)
    int node = 0;                      // virtual-node mode: this executor's node
    std::shared_ptr<Communicator> comm;
    std::vector<int> all_devices;               // virtual-node mode: every node's GPUs (peer access for device-direct sends)
    uint64_t host_arena_bytes = 256ull << 20;   // M1 (pinned, mapped) staging arena, virtual-node mode
    bool bounds_check = false;                  // §4.4 accessor bounds checking
};

struct ExecStats {
    uint64_t kernel_launches = 0;      // our CUDA kernels (workload + copy + signal)
    uint64_t workload_launches = 0;
    uint64_t copy_launches = 0;
    uint64_t tma_copy_launches = 0;    // ... of which TMA tensor-map copy kernels
    uint64_t vmm_maps = 0, vmm_mapped_bytes = 0;   // VMM: physical granule mappings and their bytes
    uint64_t coll_multicast = 0;                    // all-gather sets run as NVLS multicast stores
    uint64_t coll_p2p = 0;                          // ... as P2P gather kernels
    uint64_t coll_fused = 0;                        // ... fused into the RSim row kernels that produce them
    uint64_t halo_fused = 0;                        // coherence copies stored by the stencil launch that writes them
    uint64_t halo_in_waits = 0;                     // incoming copies awaited inside the consuming launch
    uint64_t halo_chained = 0;                      // fused RSim rows chained to the previous row's local stores
    uint64_t staging_elided = 0, staging_materialized = 0;   // device-direct sends (virtual-node mode)
    uint64_t memcpy_calls = 0;         // cudaMemcpy3DAsync (H2D / D2H)
    uint64_t bytes_copy[6] = {};       // 0 resize, 1 d2d same GPU, 2 d2d peer, 3 h2d, 4 d2h, 5 other
    uint64_t event_waits = 0, remote_waits = 0, signals = 0;
    uint64_t copies_elided = 0, bytes_elided = 0;   // resize copies made no-ops by in-place growth
    uint64_t coll_groups = 0, coll_copies = 0;      // all-gather copy sets run as NCCL collectives
    uint64_t coll_allgathers = 0;                   // ... of which as one in-place ncclAllGather
    uint64_t host_syncs = 0;
    uint64_t exec_ns[kNumIKinds] = {}; // host time in on_instr per instruction kind (IKind order)
    uint64_t signal_ns = 0, remote_wait_ns = 0;
};

constexpr int kProfSlots = K_NUM + 4;

class Executor : public InstrSink {
public:
    Executor(const ExecConfig& cfg, Scheduler* sched);
    ~Executor() override;

    int init(std::string* err);
    // Called by the scheduler (API thread) in iid order.  With the executor
    // thread running (default), the instruction is queued and issued by that
    // thread (scheduler and executor decoupled over a queue).
    void on_instr(const Instr& ins) override;
    void on_instr_impl(const Instr& ins);
    // Wait until the executor thread has processed everything queued so far
    // (after an epoch instruction: until the epoch's GPU work is complete).
    void drain();
    // Run fn on the executor thread, in queue order.
    void post(std::function<void()> fn);
    void add_buffer(uint32_t bid, const Box& extent, uint32_t es);

    // host data of a host-initialised buffer: copied into pinned memory, or
    // borrowed (size 0 marks a borrowed pointer; the caller keeps it valid)
    int set_host_init(uint32_t bid, const void* data, size_t bytes, bool borrow);
    void drop_host_init(uint32_t bid);
    void drop_host_init_later(uint32_t bid) {
        post([this, bid] { host_drop_.push_back(bid); });
    }
    void set_scheduler(Scheduler* s) { sched_ = s; }
    void set_readback(int64_t rb, void* dst, const Box& box, uint32_t elem_size);

    // multi-process plumbing: blob = arena IPC handle | flag | NCCL unique id
    static constexpr size_t kBlobBytes = 64 + 1 + 128;
    size_t ipc_blob_size() const;
    int ipc_export(void* blob) const;
    int ipc_import(int rank, const void* blob);

    int error() const { return err_.load(); }
    const std::string& error_msg() const { return errmsg_; }
    // counters as of the last drain (or the last few hundred instructions):
    // the executor thread publishes a copy, the API thread reads the copy
    ExecStats stats() {
        if (!threaded_) return st_;
        std::lock_guard<std::mutex> l(smu_);
        return pub_;
    }

    // profiling: per kernel kind, accumulated device ms and launch count
    // stride k > 0: time every k-th launch of each kind (unbiased average, less
    // event overhead in the timed region); 0: off
    void set_profile(int stride);
    int profile_read(double* ms, uint64_t* count, int n);
    // JSONL trace of the profiled launches (S:L528 format): iid, device,
    // stream, kind, start_us, end_us relative to profile_enable, per device
    int trace_dump(const char* path);
    void profile_reset();
    int device_count() const { return G_; }
    // multicast gathers run sets of any size: the scheduler should flag small ones too
    // (multi-process: P2P gathers replace NCCL for the sets NCCL would take;
    // small sets stay pushes -- measured faster across processes for RSim rows)
    bool gathers_any_size() const { return mc_enabled_ || (p2p_gather_ && cfg_.world == 1); }
    int owned(int d) const { return owner_rank(d) == cfg_.rank; }
    void sync_all();

private:
    struct Stream {
        cudaStream_t s = nullptr;
        int dev = 0;
        uint64_t seq = 0;
        uint64_t done = 0;
        std::deque<std::pair<uint64_t, cudaEvent_t>> inflight;
        std::unordered_set<uint64_t> waited_remote;   // (rank, iid) flags already waited on this stream
        uint64_t waits = 0;                           // waits enqueued (event / flag)
    };
    struct FreeRange {
        uint64_t len;
        Token tok;
    };
    struct Arena {
        char* base = nullptr;          // local mapping (owned device) or IPC mapping
        uint64_t size = 0;
        uint64_t data_off = 0;         // after the signal area
        std::map<uint64_t, FreeRange> free_;
        bool alloc(uint64_t bytes, uint64_t* off, Token* tok);
        // grow [off, off + old_bytes) in place to new_bytes if the range right
        // after it is free; tok receives that range's completion token
        bool extend(uint64_t off, uint64_t old_bytes, uint64_t new_bytes, Token* tok);
        Token& release(uint64_t off, uint64_t bytes, Token tok);   // the coalesced free range's token
    };
    // VMM allocation: its own reserved VA range,
    // physical memory mapped in granules as the allocation grows in place
    struct VmmRegion {
        CUdeviceptr va = 0;
        uint64_t reserved = 0, mapped = 0;
        int dev = 0;
        std::vector<std::pair<CUmemGenericAllocationHandle, uint64_t>> chunks;   // (handle, bytes) in VA order
    };
    struct AllocRec {
        int dev;
        uint64_t off;
        uint64_t bytes;
        Box box;
        uint32_t es;
        uint64_t iid;
        uint32_t buffer = 0;
        int64_t absorbed_into = 0;                // in-place growth: memory now owned by this aid
        Token use;                                // local work that read / wrote it (in-place growth)
        std::shared_ptr<VmmRegion> vmm;           // VMM allocation (else arena range [off, off + bytes))
    };
    struct Prof {
        int kind;
        cudaEvent_t a, b;
        int dev;
        uint64_t iid = 0;
        int stream = 0;
        uint64_t issue_ns = 0;
    };
    struct TraceRec {
        uint64_t iid;
        int dev, stream, kind;
        double start_us, end_us, issue_us;
    };
    struct CopyInfo {
        int64_t src_aid, dst_aid;
        Box bb;
        Region region;
    };
    struct Parts {                                 // a kernel launched as shell + interior
        Token shell;
        Box interior;
        int64_t write_aid;
        std::vector<int64_t> bound;                // every allocation the kernel touches
    };
    struct Readback {
        char* dst;
        Box box;
        uint32_t es;
    };

    int owner_rank(int dev) const { return cfg_.world > 1 ? dev : 0; }
    int instr_owner(const Instr& ins) const;        // device that executes it, -1 = all
    cudaEvent_t get_event(int dev);
    void put_event(int dev, cudaEvent_t e);
    void poll(bool prune);
    Token dep_token(uint64_t j) const;
    bool owner_lookup(uint64_t j, int* o) const;
    void check_owner_known(const Instr& ins);
    const Instr* cur_ins_ = nullptr;              // instruction being processed (dep_owner lookups)
    void merge(Token& into, const Token& t) const;
    void wait_token(int sidx, const Token& t);
    Token record(int sidx);
    void set_dev(int dev);
    void check(cudaError_t e, const char* what);
    void checkd(CUresult e, const char* what);
    void signal_deps(const Instr& ins, int owner_dev);
    Token local_part(const std::vector<uint64_t>& deps) const;
    Token multi_local_part(const std::vector<uint64_t>& deps) const;
    char* alloc_ptr(int64_t aid);
    void exec_copy(const Instr& ins);
    bool exec_copy_tma(const Instr& ins, const AllocRec& S, const AllocRec& D, uint32_t es, int sidx, int dev);
    void exec_kernel(const Instr& ins);
    void build_kargs(const Instr& ins, KArgs& a);
    void exec_epoch(const Instr& ins);
    void throttle();
    void prune_tokens(uint64_t below);
    void note_use(const Instr& ins);
    void exec_transfer(const Instr& ins);
    // accessor bounds checking (§4.4): per-launch device records, copied to
    // pinned host memory after the kernel and inspected once it has exited
    struct OobRec {
        int dev;
        int slot;
        cudaEvent_t ev;
        uint64_t iid;
        int64_t task;
        int n_acc;
        uint32_t buf[kMaxAcc];
        Box range[kMaxAcc];
    };
    long long* oob_begin(int dev, int sidx, int n_acc);   // device record of the next launch
    void oob_end(int dev, int sidx, const Instr& ins, const TaskDesc& d, int n_acc);
    void oob_check(bool wait);
    std::vector<long long*> oob_dev_, oob_host_;
    std::vector<int> oob_next_;
    std::deque<OobRec> oob_pending_;
    static constexpr int kOobSlots = 1024;
    void exec_host_copy(const Instr& ins, const Token& deps);
    Arena& arena(int dev) { return dev < 0 ? host_arena_ : arenas_[dev]; }
    char* base_of(const AllocRec& r) {
        if (r.vmm) return reinterpret_cast<char*>(r.vmm->va);
        return (r.dev < 0 ? host_arena_.base : arenas_[r.dev].base) + r.off;
    }
    // NVLS multicast all-gather (exec_mc.cu)
    struct McGroup {
        CUmemGenericAllocationHandle h = 0;       // multicast object bound to the set's G allocations
        CUdeviceptr va = 0;
        uint64_t size = 0;
        std::vector<std::shared_ptr<VmmRegion>> regions;
        uint64_t slot = 0;                        // flag word of this group
        uint64_t expected = 0;                    // flag value once every round so far has landed
    };
    bool mc_enabled_ = false;                     // CEL_COLL_MC=1 (single process, distinct GPUs, VMM)
    uint64_t coll_min_bytes_ = 1ull << 20;        // smallest per-source set for NCCL (CEL_COLL_MIN_BYTES)
    int mc_state_ = 0;                            // 0 not set up, 1 ready, -1 unavailable
    uint64_t mc_gran_ = 0;
    CUmemGenericAllocationHandle mc_flag_h_ = 0;
    CUdeviceptr mc_flag_va_ = 0;
    std::vector<std::shared_ptr<VmmRegion>> mc_flag_dev_;
    std::vector<void*> mc_ctr_;
    std::map<std::vector<int64_t>, McGroup> mc_groups_;
    uint64_t mc_next_slot_ = 0;
    bool mc_setup();
    bool mc_map(CUmemGenericAllocationHandle h, uint64_t size, CUdeviceptr* va);
    void mc_group_destroy(McGroup& g);
    void mc_teardown();
    void mc_forget(const VmmRegion* r);
    bool exec_coll_mc(const std::vector<Instr>& m);
    bool exec_coll_p2p(const std::vector<Instr>& m);
    // RSim rows fused with their gathers (exec_fuse.cu)
    bool fuse_rows_ = false;                      // CEL_FUSE_ROWS=0: off
    bool flushing_ = false;
    std::vector<Instr> parked_;                   // instructions held back, in order
    std::unordered_set<uint64_t> parked_iids_;
    std::vector<std::pair<uint64_t, int>> deferred_signals_;   // (iid, rank): signal once it has run
    bool depends_on_parked(const Instr& ins) const;
    bool park_candidate(const Instr& ins);
    void park(const Instr& ins);
    void flush_parked();
    bool try_fuse(const std::vector<Instr>& m);
    void signal_one(uint64_t j, int jo, int o);
    void flush_deferred_signals();
    // WaveSim halo exchange fused into the stencil launches (exec_halo.cu)
    bool fuse_halo_ = false;                      // CEL_FUSE_HALO: multi-process, distinct GPUs
    bool halo_parked_ = false, halo_flushing_ = false;
    Instr halo_kernel_;                           // the held-back stencil instruction
    std::vector<Instr> halo_pushes_;              // its outgoing coherence copies
    std::vector<Instr> halo_deferred_;            // horizons that arrived in between
    std::unordered_set<uint64_t> halo_iids_;
    std::vector<std::array<unsigned, kHaloMax>> halo_ctr_;   // per device: CTA counters' host copies
    struct RsimChain {                            // per device: fused RSim rows (exec_halo.cu)
        unsigned ctr = 0, done = 0;               // the device counters' values after the last launch
        uint64_t seq = ~0ull, waits = ~0ull;      // compute stream state right after it
    };
    std::vector<RsimChain> rsim_chain_;
    bool halo_candidate(const Instr& ins);
    bool halo_attach(const Instr& ins);
    bool halo_depends(const Instr& ins) const;
    bool halo_launch(const Instr& k, const std::vector<Instr>& pushes);
    bool halo_launch_rsim(const Instr& k, const std::vector<Instr>& pushes);
    void halo_flush();
    bool p2p_gather_ = false;                     // gather sets as P2P gather kernels (CEL_COLL_P2P=0: off)
    uint64_t gather_off_ = 0;                     // per device arena: gather counter word (+64: CTA counter)
    std::vector<uint64_t> gather_exp_;            // per device: chunks received by P2P gathers so far
    void sync_streams();
    // VMM (single process): reserve / map / grow / release
    bool vmm_ = false;
    uint64_t vmm_gran_ = 2ull << 20;
    std::vector<std::pair<std::shared_ptr<VmmRegion>, Token>> vmm_free_;   // released once the token completes
    bool vmm_map_more(VmmRegion& v, uint64_t bytes);
    std::shared_ptr<VmmRegion> vmm_create(int dev, uint64_t bytes, uint64_t reserve);
    void vmm_release(VmmRegion& v);
    void vmm_reap(bool all);
    void exec_coll(const std::vector<Instr>& members);
    bool coll_init();
    Token materialize(int dev, const Token& t);
    cudaEvent_t prof_event(int dev);
    uint64_t* sig_slot(int dev, int from_rank, uint64_t iid);

    ExecConfig cfg_;
    Scheduler* sched_;
    int G_ = 0;
    std::vector<Stream> streams_;                  // dev*5 + {0 compute, 1 copy, 2 push, 3 sync, 4 halo}
    std::vector<std::vector<cudaEvent_t>> pool_;
    std::vector<std::vector<cudaEvent_t>> prof_pool_;  // timing-enabled events for the profile
    std::vector<cudaEvent_t> trace_ref_;              // per device: time origin of the trace
    uint64_t trace_ref_ns_ = 0;                       // host clock at the same point
    std::vector<TraceRec> trace_recs_;
    std::vector<Arena> arenas_;
    std::unordered_map<uint64_t, Token> tok_;
    std::unordered_map<uint64_t, Token> ltok_;     // local part of horizons / epochs
    std::unordered_map<uint64_t, int> kind_of_;    // iid -> owner device for event-only instrs (-1 all)
    std::unordered_map<int64_t, AllocRec> allocs_;
    std::unordered_map<uint32_t, std::pair<char*, size_t>> host_init_;
    std::unordered_map<int64_t, Readback> readbacks_;
    std::unordered_set<uint64_t> signalled_;       // (iid * world + target) already signalled
    std::vector<Prof> prof_pending_;
    double prof_ms_[kProfSlots] = {};    // kernel kinds, K_NUM = local copy, +1 peer copy, +2 shell, +3 collective
    uint64_t prof_n_[kProfSlots] = {};
    int prof_stride_ = 1;
    uint64_t prof_ctr_[kProfSlots] = {};
    bool prof_sample(int kind) { return prof_ctr_[kind]++ % uint64_t(prof_stride_) == 0; }
    std::vector<int> phys_;
    bool memops64_ = false;
    std::atomic<int> err_{0};
    // executor thread and its queue
    struct Item {
        int kind = 0;                              // 0 instruction, 1 function, 2 drain mark
        Instr ins;
        std::function<void()> fn;
        uint64_t mark = 0;
    };
    void push(Item&& it);
    void thread_main();
    void pin_thread();
    int pinned_core_ = -1;
    std::thread thr_;
    bool threaded_ = false;
    std::deque<Item> q_;
    std::mutex qm_;
    std::condition_variable qcv_, qfull_cv_, done_cv_;
    std::atomic<size_t> qsize_{0};
    bool sleeping_ = false, stop_ = false;
    uint64_t marks_posted_ = 0;
    uint64_t marks_done_ = 0;
    std::mutex dm_;
    struct BufInfo {
        Box extent;
        uint32_t es;
    };
    std::unordered_map<uint32_t, BufInfo> bufinfo_;   // executor-side copy of buffer shapes
    std::string errmsg_;
    ExecStats st_;
    ExecStats pub_;                               // published copy of st_ (stats())
    std::mutex smu_;
    void publish_stats() {
        std::lock_guard<std::mutex> l(smu_);
        pub_ = st_;
    }
    uint64_t since_poll_ = 0;
    uint64_t since_publish_ = 0;
    uint64_t prev_horizon_ = 0;
    uint64_t prune_floor_ = 0;                    // tokens below it were pruned (complete)
    std::unordered_set<uint64_t> live_alloc_iid_;
    std::vector<uint32_t> host_drop_;
    bool trace_ = false;
    bool split_ = true;
    bool peer_dma_ = true;                        // small contiguous pushes on a copy engine (CEL_PEER_DMA=0: off)
    uint64_t peer_dma_max_ = 4ull << 20;
    int kernel_variant_ = 0;                      // KArgs::variant (CEL_JACOBI=l, CEL_RSIM=0 for A/B)
    bool tma_copy_ = false;                       // strided local boxes by TMA tensor maps (CEL_COPY=tma)
    bool force_peer_ = false;                     // CEL_FORCE_PEER=1: virtual devices of one GPU use the peer path
    size_t max_pitch_ = size_t(1) << 31;          // cudaDevAttrMaxPitch (2-D DMA limit)
    bool no_grow_ = false;                      // CEL_NO_GROW=1: disable in-place growth (A/B)
    bool no_pad_ = false;                       // CEL_NO_PAD=1: allocations exactly as the IDAG's boxes
    uint32_t row_align_ = 16;                   // bytes the innermost dimension's rows are padded to (CEL_ROW_ALIGN)
    Box padded_box(const Box& b, uint32_t buffer, uint32_t es) const;
    bool grown_ = true;                           // track allocation uses for in-place growth
    std::unordered_map<uint64_t, CopyInfo> copy_info_;
    // §8 a7 all-gather as a collective: members are held until the whole set
    // has arrived (they are consecutive within one task's coherence copies)
    bool coll_ = false;                           // NCCL loaded and the devices qualify
    int coll_state_ = 0;                          // 0 communicators not built, 1 ready, -1 failed
    std::vector<void*> comms_;                    // ncclComm_t per local device
    unsigned char nccl_id_[128] = {};
    bool nccl_id_set_ = false;
    std::unordered_map<uint64_t, std::vector<Instr>> coll_pending_;
    // virtual-node mode: M1 staging arena and the flags sends / receives wait on
    Arena host_arena_;
    std::unordered_map<uint64_t, std::vector<uint64_t>> pending_send_;   // iid -> messages whose pulls complete it
    std::unordered_map<uint64_t, Token> msg_tok_;              // message -> its pull's completion (resolved once)
    // device-direct sends (P:L785 RDMA future work): a staging
    // copy device -> M1 whose data only leaves through sends is not executed;
    // the sends publish the device allocation itself and the receiver pulls
    // from it over NVLink.  Materialised (executed late) if anything else needs
    // the M1 bytes, or before its source allocation is freed.
    struct Staged {
        Instr ins;                                 // the elided copy
        Token deps;                                // its dependencies' completion
        bool consumed = false;                     // a send published its source
    };
    std::map<uint64_t, Staged> staged_;
    std::unordered_set<uint64_t> elided_iids_;     // every staging copy elided (pruned at epochs)
    bool direct_sends_ = false;                    // virtual-node mode; CEL_DIRECT_SENDS=0 stages through M1
    bool materializing_ = false;                   // exec_copy of an elided copy that is needed after all
    int64_t direct_src_ = -1;                      // settle_staged -> exec_transfer: device source of this send
    uint64_t direct_staged_ = 0;                   // ... and the elided copy that staged it
    Token settle_tok_;                             // copies materialised before this instruction
    void settle_staged(const Instr& ins);
    void materialize_staged(uint64_t iid);
    std::unordered_map<int64_t, Communicator::Mem> recv_dst_; // transfer tid * 2^32 + buffer -> split receive destination
    void resolve_sends(const Instr& ins);
    std::unordered_map<uint64_t, Parts> parts_;
    // flag slots per (sender rank) in each GPU's signal area: slot iid % kRing.
    // Waits are GEQ, so two iids sharing a slot must never be in flight
    // together: the window of in-flight iids is bounded by the executor queue
    // (16384 relayed instructions) and the per-stream event cap (2048) times the
    // G ranks' interleaving, far below 2^20
    static constexpr uint64_t kRing = 1u << 20;
};

}  // namespace cel
