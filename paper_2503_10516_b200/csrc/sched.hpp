// Host scheduler: task tracking + horizons, lookahead, instruction-graph (IDAG)
// generation.  One node, G local devices ("manage all devices of a
// multi-GPU node within a single process").  Rules R0-R14 of DESIGN.md.
#pragma once

#include <cstdint>
#include <cstdio>
#include <functional>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <tuple>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "geom.hpp"

namespace cel {

// ---- error codes (mirror include/cel.h)
enum : int {
    E_OK = 0,
    W_UNINIT_READ = 1,
    E_INVALID = -1,
    E_OUT_OF_BOUNDS = -2,
    E_OVERLAPPING_WRITE = -3,
    E_OOM = -4,
    E_CUDA = -5,
    E_NCCL = -6,
    E_STATE = -7,
};

// NeighborhoodAxes: the axis-only neighbourhood (a stencil reading no corners,
// SURVEY NEXT-3); its box is the cross's bounding box, mapper_region the cross
enum class MapKind : int { OneToOne = 0, Neighborhood = 1, All = 2, Fixed = 3, Remap = 4, NeighborhoodAxes = 5 };

struct Mapper {
    MapKind kind = MapKind::OneToOne;
    int64_t border[3] = {0, 0, 0};
    Box fixed;                        // Fixed / Remap (not normalised for Remap)
    int from_kernel_dim[3] = {-1, -1, -1};
};

enum Mode : int { MODE_READ = 1, MODE_WRITE = 2, MODE_READ_WRITE = 3 };

struct Access {
    uint32_t buf = 0;
    int mode = MODE_READ;
    Mapper map;
};

struct KParams {                      // workload kernel parameters (see include/cel.h)
    uint64_t seed = 0;
    float value = 0.f;
    uint32_t t = 0;
    uint32_t salt = 0;
};

using KernelFn = void (*)(void* user, int device, const void* chunk, const void* acc, int n_acc, void* stream);

struct TaskDesc {
    int dims = 1;
    Box range;
    int split = 0;                    // 0 = 1D, 1 = 2D
    int kernel = 0;
    KParams params;
    KernelFn fn = nullptr;
    void* fn_user = nullptr;
    std::vector<Access> acc;
};

using IdSet = SmallVec<int64_t, 6>;      // a set of instruction / task ids, sorted

// Readers since the last write, as append-only records (id, region): a read
// appends, a write removes its region from every record it overlaps, a
// horizon renames ids older than it and merges equal ids.  The set of ids
// overlapping any region equals that of a region map of id sets (R12), at
// O(1) cost per read.
struct ReaderList {
    struct Rec {
        int64_t id;
        Region r;
        Box bb;
    };
    std::vector<Rec> recs;

    void add(int64_t id, const Region& r) {
        if (r.empty()) return;
        if (!recs.empty() && recs.back().id == id) {
            recs.back().r = runion(recs.back().r, r);
            recs.back().bb = bbox(recs.back().bb, rbbox(r));
            return;
        }
        recs.push_back(Rec{id, r, rbbox(r)});
    }
    template <class F>
    void ids_in(const Region& w, F fn) const {
        if (w.empty()) return;
        const Box wb = rbbox(w);
        for (const Rec& x : recs) {
            if (!overlaps(x.bb, wb)) continue;
            bool hit = false;
            for (const Box& a : x.r) {
                for (const Box& b : w)
                    if (overlaps(a, b)) {
                        hit = true;
                        break;
                    }
                if (hit) break;
            }
            if (hit) fn(x.id);
        }
    }
    void remove(const Region& w) {
        if (w.empty()) return;
        const Box wb = rbbox(w);
        size_t k = 0;
        for (size_t i = 0; i < recs.size(); ++i) {
            Rec& x = recs[i];
            if (overlaps(x.bb, wb)) {
                Region rest = rdiff_nobb(x.r, w);
                if (rest.empty()) continue;
                if (!(rest == x.r)) {
                    x.bb = rbbox(rest);
                    x.r = std::move(rest);
                }
            }
            if (k != i) recs[k] = std::move(x);
            ++k;
        }
        recs.resize(k);
    }
    void subsume(int64_t h) {
        bool any = false;
        for (Rec& x : recs)
            if (x.id < h) {
                x.id = h;
                any = true;
            }
        if (!any) return;
        // merge records of equal id (keeps the list bounded across horizons):
        // the boxes of every record of an id gathered, one canon per merged id
        std::vector<Rec> out;
        std::vector<Region> extra;        // boxes to add to out[i]
        for (Rec& x : recs) {
            size_t k = 0;
            while (k < out.size() && out[k].id != x.id) ++k;
            if (k == out.size()) {
                out.push_back(std::move(x));
                extra.emplace_back();
            } else {
                extra[k].insert(extra[k].end(), x.r.begin(), x.r.end());
                out[k].bb = bbox(out[k].bb, x.bb);
            }
        }
        for (size_t k = 0; k < out.size(); ++k)
            if (!extra[k].empty()) {
                extra[k].insert(extra[k].end(), out[k].r.begin(), out[k].r.end());
                out[k].r = canon(std::move(extra[k]));
            }
        recs.swap(out);
    }
    template <class F>
    void all_ids(F fn) const {
        for (const Rec& x : recs) fn(x.id);
    }
};

// Table 1.  Send .. AwaitReceive occur only in virtual-node mode
// (cluster.hpp).
enum class IKind : uint8_t { Alloc, Free, Copy, Kernel, Horizon, Epoch, Send, Receive, SplitReceive, AwaitReceive };
constexpr int kNumIKinds = 10;
enum CopyReason : int { REASON_RESIZE = 0, REASON_COHERENCE = 1, REASON_READBACK = 2 };

constexpr int64_t NONE = -1;          // no writer (uninitialised)
constexpr int64_t HOST_AID = -1;      // implicit M0 allocation of a host-initialised buffer
constexpr int64_t USER_AID = -2;      // user pointer of a readback

struct Instr {
    uint64_t iid = 0;
    IKind kind = IKind::Epoch;
    int64_t task = -1;                // -1 = none
    uint32_t buffer = 0;
    // alloc / free
    int64_t aid = 0;
    int mem = 0;
    Box box;
    // copy
    int reason = 0;
    int64_t src_aid = 0, dst_aid = 0;
    int src_mem = 0, dst_mem = 0;
    Region region;
    int64_t readback = -1;
    // send (box, src_aid/src_mem = the node's M1 staging allocation) / receive /
    // split receive (region, dst_aid/dst_mem) / await receive (region):
    // transfer id = (transfer, buffer)
    int target = -1;
    uint64_t msg = 0;
    int64_t transfer = -1;
    // §8 a7: member of an all-gather copy set (not part of the instruction log):
    // group id (0 = none) and the number of copies in the group
    uint64_t coll = 0;
    uint32_t coll_n = 0;
    // kernel
    int device = -1;
    Box chunk;
    std::vector<int64_t> bindings;
    std::shared_ptr<const TaskDesc> desc;
    // all
    std::vector<uint64_t> deps;
    // multi-process rank filter (world > 1): owner device of each dependency as
    // the scheduler knew it when it emitted this instruction (-1 = every rank,
    // -2 = unknown: older than the scheduler's owner ring), so the executor
    // thread never reads the scheduler's ring, which the API thread overwrites
    std::vector<int8_t> dep_owner;
};

struct InstrSink {
    virtual ~InstrSink() = default;
    virtual void on_instr(const Instr& ins) = 0;   // called in iid (topological) order
};

// a send's pilot message, "transmitted to the receiver ahead of
// execution time"
struct Pilot {
    int sender = 0;
    uint64_t msg = 0;
    int receiver = 0;
    int64_t transfer = 0;      // transfer id (transfer, buffer)
    uint32_t buffer = 0;
    Box box;
};

using Push = std::tuple<int, uint32_t, Region>;   // (target node, buffer, region)

struct SchedStats {
    uint64_t n_by_kind[16] = {};
    uint64_t copies_by_reason[3] = {};
    uint64_t bytes_by_reason[3] = {};
    uint64_t bytes_d2d_peer = 0;
    uint64_t alloc_bytes_live = 0, alloc_bytes_peak = 0;
    uint64_t flushes = 0;
    uint64_t gather_sets = 0;                          // coherence copy sets that are all-gathers (§8 a7)
};

class Scheduler {
public:
    Scheduler(int n_devices, int lookahead, int horizon_step, bool checks, InstrSink* sink, FILE* log);
    ~Scheduler();

    int buffer_create(int dims, const int64_t extent[3], uint32_t elem_size, bool host_init, uint32_t* out);
    int task_submit(const TaskDesc& desc, uint64_t* tid_out, std::string* err);
    // Virtual-node mode (cluster.cpp): this node's share of a task -- the
    // command chunk `node_range` split over the local devices -- with the
    // transfers the replicated command-graph generation derived for it; the
    // task graph sees the whole task (`reads` / `writes` over all nodes).
    int task_submit_node(const TaskDesc& desc, const Box& node_range, const std::map<uint32_t, Region>& reads,
                         const std::map<uint32_t, Region>& writes, const std::vector<Push>& pushes,
                         const std::map<uint32_t, Region>& awaits, const std::map<uint32_t, Region>& remote_writes,
                         uint64_t* tid_out, std::string* err);
    // Virtual-node mode readback epoch: node 0 (rb >= 0) gathers, the others push.
    void epoch_node(int64_t rb, uint32_t rb_buf, const Box& rb_box, const std::vector<Push>& pushes,
                    const std::map<uint32_t, Region>& awaits);
    void set_node(int n) { node_ = n; }
    // Multi-process mode (one process per GPU, every rank replays the node's
    // IDAG): hand this rank's executor only the instructions it executes or
    // must take part in (allocs, frees, horizons, epochs, collectives, copies
    // into its memory, and instructions with a dependency it executes or
    // co-owns, which it must signal); record every instruction's owner device
    // for the executor (owner_of).
    void set_rank_filter(int rank, int world);
    // owner device of instruction `iid` (-1: every rank), false if unknown
    bool owner_of(uint64_t iid, int* owner) const;
    // the same from the recent-instruction ring only: safe to call from the
    // executor thread for instructions emitted before the one it processes
    bool ring_owner(uint64_t iid, int* owner) const {
        if (ring_iid_.empty()) return false;
        const uint64_t k = iid & (kOwnerRing - 1);
        if (ring_iid_[k] != iid) return false;
        *owner = ring_owner_[k];
        return true;
    }
    int node() const { return node_; }
    // pilots go to `fn` as they are produced ("transmitted ... ahead of execution time");
    // without a sink (execute=0) they are dropped: the send instruction in the log carries them
    void set_pilot_sink(std::function<void(const Pilot&)> fn) { pilot_sink_ = std::move(fn); }
    int64_t alloc_readback_id() { return next_rb_++; }
    void wait();
    int readback(uint32_t bid, const Box& box, int64_t* rb_out, std::string* err);
    int destroy(uint32_t bid, std::string* err);
    void shutdown();

    uint32_t elem_size(uint32_t bid) const;
    Box extent(uint32_t bid) const;
    bool has_buffer(uint32_t bid) const;
    const SchedStats& stats() const { return st_; }
    int64_t next_readback_id() const { return next_rb_; }
    uint64_t next_iid() const { return next_iid_; }
    void debug_dump(FILE* f) const;

private:
    struct PrepMemo;                                  // sched_memo.cpp
    struct CompileMemo;
    struct Alloc {
        int64_t aid;
        uint32_t buffer;
        int mem;
        Box box;
        int64_t iid;                                  // alloc instruction, -1 for HOST_AID
        RegionMap<int64_t> last_writer;
        ReaderList readers;
    };
    struct Buf {
        uint32_t bid;
        int dims;
        Box extent;
        uint32_t elem_size;
        bool host_init;
        RegionMap<int64_t> orig_writer;               // P:L372 "original producer"
        RegionMap<uint32_t> uptodate;                 // P:L371 bit m = memory Mm
        std::map<int, std::vector<Alloc*>> live;      // non-overlapping per memory
        std::unique_ptr<Alloc> host;
    };
    struct TBuf {                                     // task-graph tracking
        RegionMap<int64_t> last_writer;
        ReaderList readers;
        Region initialized;
    };
    using Key = std::pair<int, uint32_t>;             // (device, buffer)
    struct Cmd {
        int kind = 0;                                 // 0 task, 1 horizon, 2 epoch, 3 destroy
        int64_t tid = -1;
        std::shared_ptr<const TaskDesc> desc;
        std::vector<Box> chunks;
        std::map<Key, Region> reads, writes;
        std::map<Key, Box> req;
        int64_t rb = -1;
        uint32_t rb_buf = 0;
        Box rb_box;
        std::vector<uint32_t> destroy;
        // virtual-node mode
        std::vector<Push> pushes;                     // sorted by (target, buffer)
        std::map<uint32_t, Region> awaits, remote_writes;
        std::shared_ptr<PrepMemo> memo;               // set when its shape was submitted before (sched_memo.cpp)
    };

    // task graph (R7)
    int64_t tdag_submit(const std::map<uint32_t, Region>& reads, const std::map<uint32_t, Region>& writes);
    int64_t tdag_horizon();
    int64_t tdag_epoch();
    void tdag_subsume(int64_t h);
    // lookahead (R8)
    void push(Cmd&& c);
    void flush();
    bool is_allocating(const Cmd& c) const;
    std::map<std::pair<uint32_t, int>, Box> anticipated(const std::vector<Cmd>& q) const;
    void epoch_cmd(Cmd&& c);
    // IDAG (R9-R14)
    void compile(Cmd& c, const std::map<std::pair<uint32_t, int>, Box>& ant);
    void compile_task(Cmd& c, const std::map<std::pair<uint32_t, int>, Box>& ant);
    std::map<Key, Alloc*> allocate(Cmd& c, const std::map<std::pair<uint32_t, int>, Box>& ant);
    void transfers(Cmd& c, std::map<Key, Alloc*>& binding, bool readback_consumer);
    void transfer_req(Cmd& c) const;
    int submit_cmd(Cmd&& c, const std::map<uint32_t, Region>& reads, const std::map<uint32_t, Region>& writes,
                   uint64_t* tid_out);
    void compile_horizon(Cmd& c);
    void compile_epoch(Cmd& c);
    uint64_t emit(Instr& ins, std::vector<uint64_t>& deps);
    Alloc* new_alloc(uint32_t bid, int mem, const Box& box, int64_t tid);
    void free_alloc(Alloc* a, int64_t tid);
    uint64_t copy(int64_t tid, uint32_t bid, int reason, Alloc* src, Alloc* dst, const Region& reg, int64_t rb,
                  uint64_t coll = 0, uint32_t coll_n = 0);
    std::map<std::tuple<int64_t, int, int64_t>, Region> source_parts(Buf& buf, const Region& need, int m_dst);
    std::map<std::tuple<int64_t, int, int64_t>, Region> source_parts_q(
        Buf& buf, const std::vector<std::pair<Region, uint32_t>>& need_by_mask, int m_dst);
    std::map<uint32_t, uint32_t> all_gathers(
        const Cmd& c,
        const std::vector<std::pair<Key, std::vector<std::pair<std::tuple<int64_t, int, int64_t>, Region>>>>& pend,
        const std::map<Key, Alloc*>& binding) const;
    void subsume(int64_t h);
    void log_instr(const Instr& ins);
    int prepare(const TaskDesc& d, Cmd& c, std::string* err, const Box* node_range = nullptr) const;

    int G_;
    int mode_;
    bool checks_;
    InstrSink* sink_;
    FILE* log_;
    SchedStats st_;

    // task graph
    int64_t next_tid_ = 1;
    std::unordered_map<int64_t, int64_t> cp_;
    int64_t t_fallback_ = 0, t_pending_h_ = -1, max_cp_ = 0, cp_ref_ = 0;
    int horizon_step_;
    std::map<uint32_t, TBuf> tbufs_;

    // lookahead
    std::vector<Cmd> queue_;
    std::map<std::pair<uint32_t, int>, Box> queue_ant_;   // P:L589 requirements observed while queued
    int counter_ = 0;

    // IDAG
    std::map<uint32_t, std::unique_ptr<Buf>> bufs_;
    std::unordered_map<int64_t, std::unique_ptr<Alloc>> allocs_;
    std::vector<uint64_t> front_;                     // sorted
    std::vector<uint64_t> front_scratch_;
    std::vector<int64_t> sig_scratch_;                // compile memo signature (sched_memo.cpp)
    uint64_t next_iid_ = 1;
    int64_t fallback_ = 0, pending_h_ = -1;
    int64_t next_aid_ = 1;
    int64_t next_rb_ = 0;
    uint64_t next_coll_ = 1;
    int node_ = 0;                                    // virtual-node mode: this node's id
    int filter_rank_ = -1, filter_world_ = 1;
    static constexpr uint64_t kOwnerRing = 1ull << 20;
    std::vector<uint64_t> ring_iid_;                  // iid -> owner device, recent instructions
    std::vector<int8_t> ring_owner_;
    std::unordered_map<int64_t, int> alloc_owner_;    // live allocation iid -> device (old, still referenced)
    static int instr_owner(const Instr& ins);
    uint64_t next_msg_ = 0;                           // P:L400 "locally unique message id"
    std::function<void(const Pilot&)> pilot_sink_;
    uint64_t coll_min_bytes_ = 1ull << 20;            // CEL_COLL_MIN_BYTES: smallest per-source gather run as NCCL
public:
    // the executor runs gathers of any size as a collective (multicast): flag them all
    void set_coll_min_bytes(uint64_t b) { coll_min_bytes_ = b; }
private:
    uint32_t next_bid_ = 0;
    bool shut_ = false;

    // Steady-state fast path (sched_memo.cpp; DESIGN.md §2 "compile memo").
    // prepare() results per task shape, and compile_task() results per (task
    // shape, state of the accessed buffers with instruction ids taken relative
    // to the next iid): a hit re-emits the recorded instructions with ids
    // shifted and installs the recorded end state, shifted the same way.
    std::unordered_map<uint64_t, std::shared_ptr<PrepMemo>> prep_memo_;   // by hash of the shape key
    std::unordered_set<uint64_t> prep_seen_;                               // shape hashes submitted once
    bool memo_on_ = true;
    std::vector<Instr>* recording_ = nullptr;        // emit() copies instructions here while set
    uint64_t memo_hits_ = 0, memo_misses_ = 0;
    static void shape_key(const TaskDesc& d, std::vector<int64_t>& key);
    bool prep_lookup(const std::vector<int64_t>& key, uint64_t h, Cmd& c, std::map<uint32_t, Region>& reads,
                     std::map<uint32_t, Region>& writes);
    void prep_store(std::vector<int64_t>&& key, uint64_t h, const Cmd& c, const std::map<uint32_t, Region>& reads,
                    const std::map<uint32_t, Region>& writes);
    void state_sig(const Cmd& c, uint64_t base, std::vector<int64_t>& sig) const;
    static const CompileMemo* compile_lookup(const PrepMemo& p, const std::vector<int64_t>& sig);
    void compile_replay(const CompileMemo& m, Cmd& c, uint64_t base);
    void compile_store(std::vector<int64_t>&& sig, const Cmd& c, uint64_t base, std::vector<Instr>&& out,
                       const SchedStats& before, uint64_t coll_before);

public:
    uint64_t memo_hits() const { return memo_hits_; }
    uint64_t memo_misses() const { return memo_misses_; }
    void set_memo(bool on) { memo_on_ = on; }
};

// Virtual-node mode (§3.4; mirrors
// oracle/cluster.py): N nodes of D devices, one Scheduler each.  The
// command-graph decisions -- which node pushes what to whom, what each node
// awaits -- come from replicated bookkeeping kept once here: per buffer the
// node that last wrote each element (owner) and the set of nodes holding an
// up-to-date copy (holders).  Readings R17.
class Cluster {
public:
    Cluster(int n_nodes, int devices_per_node, int lookahead, int horizon_step, bool checks,
            const std::vector<InstrSink*>& sinks, const std::vector<FILE*>& logs);
    int buffer_create(int dims, const int64_t extent[3], uint32_t elem_size, bool host_init, uint32_t* out);
    int task_submit(const TaskDesc& desc, uint64_t* tid_out, std::string* err);
    void wait();
    // node 0 gathers `box` of `bid` (owners push what it lacks); returns the readback id
    int readback(uint32_t bid, const Box& box, int64_t* rb_out, std::string* err);
    int destroy(uint32_t bid, std::string* err);
    void shutdown();
    int nodes() const { return N_; }
    Scheduler& node(int k) { return *s_[k]; }
    const Scheduler& node(int k) const { return *s_[k]; }

private:
    struct Track {
        RegionMap<int64_t> owner;     // -1 never written, -2 host data (every node)
        RegionMap<uint32_t> holders;  // bit n: node n holds an up-to-date copy
    };
    void transfers(const std::vector<std::map<uint32_t, Region>>& need, std::vector<std::vector<Push>>& pushes,
                   std::vector<std::map<uint32_t, Region>>& awaits) const;
    int N_, D_;
    std::vector<std::unique_ptr<Scheduler>> s_;
    std::map<uint32_t, Track> t_;
};

}  // namespace cel
