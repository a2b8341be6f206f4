// Host scheduler implementation.  Rules: DESIGN.md R0-R14.  Paper passages
// are cited at each step; this is an independent implementation of the same
// readings the CPU oracle (oracle/scheduler.py) follows, and the two
// instruction logs are compared record for record by the tests.
#include "sched_impl.hpp"

#include <cstdlib>

#include <algorithm>
#include <cinttypes>
#include <cstring>

namespace cel {

namespace detail {

void split_1d(const Box& rng, int n, int dim, std::vector<Box>& out) {
    const int64_t lo = rng.lo[dim], hi = rng.hi[dim];
    const int64_t len = std::max<int64_t>(0, hi - lo);
    const int64_t q = len / n, r = len % n;
    int64_t start = lo;
    for (int k = 0; k < n; ++k) {
        const int64_t size = q + (k < r ? 1 : 0);
        out.push_back(rng.with_dim(dim, start, start + size).normalized());
        start += size;
    }
}

// R4: G = a*b, a >= b, a-b minimal
void factor_2d(int n, int* a, int* b) {
    int bb = 1;
    for (int c = 1; c * c <= n; ++c)
        if (n % c == 0) bb = c;
    *b = bb;
    *a = n / bb;
}

// P:L319-326 (§3.1): static split of the kernel index space over the devices.
std::vector<Box> split(const Box& rng, int n, int kind) {
    std::vector<Box> out;
    if (rng.empty()) {
        out.assign(n, Box{});
        return out;
    }
    if (kind == 0) {
        split_1d(rng, n, 0, out);
        return out;
    }
    int a, b;
    factor_2d(n, &a, &b);
    std::vector<Box> rows;
    split_1d(rng, a, 0, rows);
    for (int i = 0; i < a; ++i) {
        if (rows[i].empty()) {
            for (int j = 0; j < b; ++j) out.push_back(Box{});
            continue;
        }
        split_1d(rows[i], b, 1, out);
    }
    return out;
}

// R5: range mappers (remap is the RSim extension).
int apply_mapper(const Mapper& m, const Box& chunk, const Box& ext, Box* out) {
    if (chunk.empty()) {
        *out = Box{};
        return E_OK;
    }
    switch (m.kind) {
    case MapKind::OneToOne:
        if (!ext.contains(chunk)) return E_OUT_OF_BOUNDS;
        *out = chunk;
        return E_OK;
    case MapKind::Neighborhood:
    case MapKind::NeighborhoodAxes: {
        Box b;
        for (int d = 0; d < 3; ++d) {
            b.lo[d] = chunk.lo[d] - m.border[d];
            b.hi[d] = chunk.hi[d] + m.border[d];
        }
        *out = intersect(b, ext);
        return E_OK;
    }
    case MapKind::All:
        *out = ext;
        return E_OK;
    case MapKind::Fixed: {
        Box b = m.fixed.normalized();
        if (!ext.contains(b)) return E_OUT_OF_BOUNDS;
        *out = b;
        return E_OK;
    }
    case MapKind::Remap: {
        Box b;
        for (int k = 0; k < 3; ++k) {
            const int src = m.from_kernel_dim[k];
            if (src >= 0) {
                b.lo[k] = chunk.lo[src];
                b.hi[k] = chunk.hi[src];
            } else {
                b.lo[k] = m.fixed.lo[k];
                b.hi[k] = m.fixed.hi[k];
            }
        }
        if (b.empty()) {
            *out = Box{};
            return E_OK;
        }
        if (!ext.contains(b)) return E_OUT_OF_BOUNDS;
        *out = b;
        return E_OK;
    }
    }
    return E_INVALID;
}

int mapper_region(const Mapper& m, const Box& chunk, const Box& ext, Region* out) {
    Box bx;
    const int rc = apply_mapper(m, chunk, ext, &bx);
    if (rc != E_OK) return rc;
    out->clear();
    if (bx.empty()) return E_OK;
    if (m.kind != MapKind::NeighborhoodAxes) {
        *out = Region{bx};
        return E_OK;
    }
    // union over dims d of the chunk inflated by border[d] in dim d alone
    Region r{intersect(chunk, ext)};
    for (int d = 0; d < 3; ++d) {
        if (m.border[d] <= 0) continue;
        Box b = chunk;
        b.lo[d] -= m.border[d];
        b.hi[d] += m.border[d];
        b = intersect(b, ext);
        if (!b.empty()) r = runion(r, Region{b});
    }
    *out = std::move(r);
    return E_OK;
}

bool is_read(int mode) { return mode == MODE_READ || mode == MODE_READ_WRITE; }
bool is_write(int mode) { return mode == MODE_WRITE || mode == MODE_READ_WRITE; }

}  // namespace detail
using namespace detail;

Box map_access(const Mapper& m, const Box& chunk, const Box& ext) {
    Box b;
    if (apply_mapper(m, chunk, ext, &b) != E_OK) return Box{};
    return b;
}

Scheduler::~Scheduler() = default;

Scheduler::Scheduler(int n_devices, int lookahead, int horizon_step, bool checks, InstrSink* sink, FILE* log)
    : G_(n_devices), mode_(lookahead), checks_(checks), sink_(sink), log_(log), horizon_step_(horizon_step) {
    const char* cm = getenv("CEL_COLL_MIN_BYTES");
    if (cm && cm[0]) coll_min_bytes_ = strtoull(cm, nullptr, 10);
    const char* mm = getenv("CEL_SCHED_MEMO");
    if (mm && mm[0] == '0') memo_on_ = false;
    cp_[0] = 0;
    // init epoch: tid 0 / iid 0
    Instr e;
    e.iid = 0;
    e.kind = IKind::Epoch;
    e.task = 0;
    front_.push_back(0);
    st_.n_by_kind[int(IKind::Epoch)]++;
    log_instr(e);
    if (sink_) sink_->on_instr(e);
}


uint32_t Scheduler::elem_size(uint32_t bid) const { return bufs_.at(bid)->elem_size; }
Box Scheduler::extent(uint32_t bid) const { return bufs_.at(bid)->extent; }
bool Scheduler::has_buffer(uint32_t bid) const { return bufs_.count(bid) != 0; }

int Scheduler::buffer_create(int dims, const int64_t extent[3], uint32_t elem_size, bool host_init, uint32_t* out) {
    if (shut_) return E_STATE;
    if (dims < 1 || dims > 3 || elem_size == 0) return E_INVALID;
    int64_t lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
    for (int d = 0; d < dims; ++d) {
        if (extent[d] <= 0) return E_INVALID;
        hi[d] = extent[d];
    }
    const uint32_t bid = next_bid_++;
    auto b = std::make_unique<Buf>();
    b->bid = bid;
    b->dims = dims;
    b->extent = Box::make(lo, hi);
    b->elem_size = elem_size;
    b->host_init = host_init;
    // R6: host-initialised data is up-to-date on M0, produced by the current epoch/horizon
    b->orig_writer = RegionMap<int64_t>(b->extent, host_init ? fallback_ : NONE);
    b->uptodate = RegionMap<uint32_t>(b->extent, host_init ? 1u : 0u);
    if (host_init) {
        b->host.reset(new Alloc{HOST_AID, bid, 0, b->extent, -1, RegionMap<int64_t>(b->extent, fallback_), ReaderList{}});
    }
    TBuf& t = tbufs_[bid];
    t.last_writer = RegionMap<int64_t>(b->extent, host_init ? t_fallback_ : NONE);
    t.readers = ReaderList{};
    t.initialized = host_init ? Region{b->extent} : Region{};
    bufs_[bid] = std::move(b);
    *out = bid;
    return E_OK;
}

// ------------------------------------------------------------ task graph (R7)
int64_t Scheduler::tdag_submit(const std::map<uint32_t, Region>& reads, const std::map<uint32_t, Region>& writes) {
    // RAW / WAR / WAW at element granularity
    std::vector<int64_t> deps;
    for (auto& kv : reads)
        tbufs_[kv.first].last_writer.for_values_in(kv.second, [&](int64_t v) {
            if (v >= 0) deps.push_back(v);
        });
    for (auto& kv : writes) {
        TBuf& t = tbufs_[kv.first];
        t.readers.ids_in(kv.second, [&](int64_t r) { deps.push_back(r); });
        t.last_writer.for_values_in(kv.second, [&](int64_t v) {
            if (v >= 0) deps.push_back(v);
        });
    }
    if (deps.empty()) deps.push_back(t_fallback_);
    const int64_t tid = next_tid_++;
    int64_t cp = 0;
    for (int64_t d : deps) cp = std::max(cp, cp_[d]);
    cp_[tid] = cp + 1;
    for (auto& kv : reads) tbufs_[kv.first].readers.add(tid, kv.second);
    for (auto& kv : writes) {
        TBuf& t = tbufs_[kv.first];
        t.last_writer.update(kv.second, tid);
        t.readers.remove(kv.second);
        t.initialized = runion(t.initialized, kv.second);
    }
    max_cp_ = std::max(max_cp_, cp_[tid]);
    return tid;
}

void Scheduler::tdag_subsume(int64_t h) {
    for (auto& kv : tbufs_) {
        kv.second.last_writer.map_values([h](int64_t v) { return (v >= 0 && v < h) ? h : v; });
        kv.second.readers.subsume(h);
    }
}

int64_t Scheduler::tdag_horizon() {
    // horizon; the previous one is applied (R7)
    const int64_t tid = next_tid_++;
    cp_[tid] = max_cp_;
    cp_ref_ = max_cp_;
    if (t_pending_h_ >= 0) {
        tdag_subsume(t_pending_h_);
        t_fallback_ = t_pending_h_;
        // cp of tasks older than the applied horizon is never read again
        for (auto it = cp_.begin(); it != cp_.end();) {
            if (it->first < t_fallback_)
                it = cp_.erase(it);
            else
                ++it;
        }
    }
    t_pending_h_ = tid;
    return tid;
}

int64_t Scheduler::tdag_epoch() {
    const int64_t tid = next_tid_++;
    cp_[tid] = 0;
    tdag_subsume(tid);
    t_fallback_ = tid;
    t_pending_h_ = -1;
    max_cp_ = 0;
    cp_ref_ = 0;
    // bounded bookkeeping: cp of tasks older than the epoch is never read again
    for (auto it = cp_.begin(); it != cp_.end();) {
        if (it->first < tid)
            it = cp_.erase(it);
        else
            ++it;
    }
    return tid;
}

// ------------------------------------------------------------ submit
int Scheduler::prepare(const TaskDesc& d, Cmd& c, std::string* err, const Box* node_range) const {
    if (d.dims < 1 || d.dims > 3) {
        if (err) *err = "task dims must be 1..3";
        return E_INVALID;
    }
    for (const Access& a : d.acc) {
        if (!bufs_.count(a.buf)) {
            if (err) *err = "access to an unknown or destroyed buffer";
            return E_INVALID;
        }
        if (a.mode != MODE_READ && a.mode != MODE_WRITE && a.mode != MODE_READ_WRITE) {
            if (err) *err = "bad access mode";
            return E_INVALID;
        }
        if (int(a.map.kind) < 0 || int(a.map.kind) > 5) {
            if (err) *err = "bad range mapper";
            return E_INVALID;
        }
    }
    c.chunks = split(node_range ? *node_range : d.range, G_, d.split);
    for (int dev = 0; dev < G_; ++dev) {
        const Box& ch = c.chunks[dev];
        if (ch.empty()) continue;
        for (const Access& a : d.acc) {
            Region reg;
            const int rc = mapper_region(a.map, ch, bufs_.at(a.buf)->extent, &reg);
            if (rc != E_OK) {
                if (err) *err = "range mapper result outside the buffer extent";
                return rc;
            }
            if (reg.empty()) continue;
            const Key k{dev, a.buf};
            if (is_read(a.mode)) c.reads[k] = runion(c.reads[k], reg);
            if (is_write(a.mode)) c.writes[k] = runion(c.writes[k], reg);
        }
    }
    // §4.4 overlapping-write detection
    std::map<uint32_t, std::vector<std::pair<int, const Region*>>> wb;
    for (auto& kv : c.writes) wb[kv.first.second].push_back({kv.first.first, &kv.second});
    for (auto& kv : wb) {
        auto& v = kv.second;
        for (size_t i = 0; i < v.size(); ++i)
            for (size_t j = i + 1; j < v.size(); ++j)
                if (!rinter(*v[i].second, *v[j].second).empty()) {
                    if (err) {
                        char buf[160];
                        snprintf(buf, sizeof buf, "devices %d and %d write overlapping regions of buffer %u",
                                 v[i].first, v[j].first, kv.first);
                        *err = buf;
                    }
                    return E_OVERLAPPING_WRITE;
                }
    }
    for (auto& kv : c.reads) c.req[kv.first] = bbox(c.req[kv.first], rbbox(kv.second));
    for (auto& kv : c.writes) c.req[kv.first] = bbox(c.req[kv.first], rbbox(kv.second));
    return E_OK;
}

int Scheduler::task_submit(const TaskDesc& desc, uint64_t* tid_out, std::string* err) {
    if (shut_) return E_STATE;
    Cmd c;
    c.kind = 0;
    std::map<uint32_t, Region> reads, writes;
    std::vector<int64_t> key;
    uint64_t h = 0;
    if (memo_on_) {   // sched_memo.cpp: a shape seen before reuses its prepare() result
        shape_key(desc, key);
        h = memo_hash(key);
        bool live = true;
        for (const Access& a : desc.acc) live = live && bufs_.count(a.buf) != 0;
        if (live) prep_lookup(key, h, c, reads, writes);
    }
    if (!c.memo) {
        const int rc = prepare(desc, c, err);
        if (rc != E_OK) return rc;
        for (auto& kv : c.reads) reads[kv.first.second] = runion(reads[kv.first.second], kv.second);
        for (auto& kv : c.writes) writes[kv.first.second] = runion(writes[kv.first.second], kv.second);
        // a shape's second submission stores its prepare() result (most
        // programs repeat shapes; RSim's never do, and pays only a hash)
        if (memo_on_ && !prep_seen_.insert(h).second) prep_store(std::move(key), h, c, reads, writes);
        if (prep_seen_.size() > 4096) prep_seen_.clear();
    }
    c.desc = std::make_shared<const TaskDesc>(desc);
    return submit_cmd(std::move(c), reads, writes, tid_out);
}

int Scheduler::task_submit_node(const TaskDesc& desc, const Box& node_range, const std::map<uint32_t, Region>& reads,
                                const std::map<uint32_t, Region>& writes, const std::vector<Push>& pushes,
                                const std::map<uint32_t, Region>& awaits,
                                const std::map<uint32_t, Region>& remote_writes, uint64_t* tid_out,
                                std::string* err) {
    if (shut_) return E_STATE;
    Cmd c;
    c.kind = 0;
    const int rc = prepare(desc, c, err, &node_range);
    if (rc != E_OK) return rc;
    c.pushes = pushes;
    c.awaits = awaits;
    c.remote_writes = remote_writes;
    transfer_req(c);
    c.desc = std::make_shared<const TaskDesc>(desc);
    return submit_cmd(std::move(c), reads, writes, tid_out);
}

void Scheduler::transfer_req(Cmd& c) const {
    // P:L398 / P:L417: pushed data is staged in, and awaited data received into,
    // one contiguous M1 allocation per buffer (requirement key device -1 -> M1)
    std::map<uint32_t, Box> boxes;
    for (auto& p : c.pushes) {
        Box& b = boxes[std::get<1>(p)];
        b = bbox(b, rbbox(std::get<2>(p)));
    }
    for (auto& kv : c.awaits) {
        Box& b = boxes[kv.first];
        b = bbox(b, rbbox(kv.second));
    }
    for (auto& kv : boxes) c.req[{-1, kv.first}] = kv.second;
}

void Scheduler::epoch_node(int64_t rb, uint32_t rb_buf, const Box& rb_box, const std::vector<Push>& pushes,
                           const std::map<uint32_t, Region>& awaits) {
    if (shut_) return;
    Cmd e;
    e.kind = 2;
    e.rb = rb;
    e.rb_buf = rb_buf;
    e.rb_box = rb_box.normalized();
    e.pushes = pushes;
    e.awaits = awaits;
    transfer_req(e);
    epoch_cmd(std::move(e));
}

int Scheduler::submit_cmd(Cmd&& c, const std::map<uint32_t, Region>& reads, const std::map<uint32_t, Region>& writes,
                          uint64_t* tid_out) {
    int status = E_OK;
    if (checks_) {  // §4.4 uninitialised-read detection: warning
        for (auto& kv : reads)
            if (!rdiff(kv.second, tbufs_[kv.first].initialized).empty()) status = W_UNINIT_READ;
    }
    c.tid = tdag_submit(reads, writes);
    if (tid_out) *tid_out = uint64_t(c.tid);
    push(std::move(c));
    if (max_cp_ - cp_ref_ >= horizon_step_) {
        Cmd h;
        h.kind = 1;
        h.tid = tdag_horizon();
        push(std::move(h));
    }
    return status;
}

void Scheduler::wait() {
    if (shut_) return;
    Cmd e;
    e.kind = 2;
    epoch_cmd(std::move(e));
}

int Scheduler::readback(uint32_t bid, const Box& box, int64_t* rb_out, std::string* err) {
    if (shut_) return E_STATE;
    if (!bufs_.count(bid)) {
        if (err) *err = "unknown buffer";
        return E_INVALID;
    }
    if (!bufs_[bid]->extent.contains(box)) {
        if (err) *err = "readback box outside the buffer extent";
        return E_OUT_OF_BOUNDS;
    }
    Cmd e;
    e.kind = 2;
    e.rb = next_rb_++;
    e.rb_buf = bid;
    e.rb_box = box.normalized();
    if (rb_out) *rb_out = e.rb;
    epoch_cmd(std::move(e));
    return E_OK;
}

int Scheduler::destroy(uint32_t bid, std::string* err) {
    if (shut_) return E_STATE;
    if (!bufs_.count(bid)) {
        if (err) *err = "unknown buffer";
        return E_INVALID;
    }
    flush();
    Cmd c;
    c.kind = 3;
    c.destroy.push_back(bid);
    compile(c, {});
    tbufs_.erase(bid);
    return E_OK;
}

void Scheduler::shutdown() {
    if (shut_) return;
    flush();
    if (!bufs_.empty()) {
        Cmd c;
        c.kind = 3;
        for (auto& kv : bufs_) c.destroy.push_back(kv.first);
        compile(c, {});
        tbufs_.clear();
    }
    Cmd e;
    e.kind = 2;
    epoch_cmd(std::move(e));
    shut_ = true;
}

void Scheduler::epoch_cmd(Cmd&& c) {
    flush();
    c.tid = tdag_epoch();
    compile(c, {});
}

// ------------------------------------------------------------ lookahead (R8, §4.3)
std::map<std::pair<uint32_t, int>, Box> Scheduler::anticipated(const std::vector<Cmd>& q) const {
    // all requirements observed while queued, per (buffer, memory)
    std::map<std::pair<uint32_t, int>, Box> ant;
    for (const Cmd& c : q)
        for (auto& kv : c.req) {
            Box& b = ant[{kv.first.second, 2 + kv.first.first}];
            b = bbox(b, kv.second);
        }
    return ant;
}

bool Scheduler::is_allocating(const Cmd& c) const {
    // "whether compiling it right away would emit any alloc instructions"
    const auto& ant = queue_ant_;     // bbox of the queued commands' requirements (incremental)
    for (auto& kv : c.req) {
        const int m = 2 + kv.first.first;
        const Buf& b = *bufs_.at(kv.first.second);
        bool ok = false;
        auto it = b.live.find(m);
        if (it != b.live.end())
            for (const Alloc* a : it->second)
                if (a->box.contains(kv.second)) {
                    ok = true;
                    break;
                }
        if (!ok) {
            auto at = ant.find({kv.first.second, m});
            if (at != ant.end() && at->second.contains(kv.second)) ok = true;
        }
        if (!ok) return true;
    }
    return false;
}

void Scheduler::push(Cmd&& c) {
    if (mode_ == 0) {  // lookahead none
        compile(c, {});
        return;
    }
    if (c.kind == 1) {  // horizon
        if (queue_.empty()) {
            compile(c, {});
            return;
        }
        queue_.push_back(std::move(c));   // horizons carry no requirements
        ++counter_;
        if (mode_ == 1 && counter_ >= 2) flush();  // P:L584 "two horizons after the last allocating command"
        return;
    }
    const bool alloc = is_allocating(c);
    if (mode_ == 1 && queue_.empty() && !alloc) {
        compile(c, {});
        return;
    }
    for (auto& kv : c.req) {
        Box& b = queue_ant_[{kv.first.second, 2 + kv.first.first}];
        b = bbox(b, kv.second);
    }
    queue_.push_back(std::move(c));
    if (alloc) counter_ = 0;
}

void Scheduler::flush() {
    if (queue_.empty()) return;
    std::vector<Cmd> q;
    q.swap(queue_);
    std::map<std::pair<uint32_t, int>, Box> ant;
    ant.swap(queue_ant_);
    counter_ = 0;
    st_.flushes++;
    for (Cmd& c : q) compile(c, ant);
}

// ------------------------------------------------------------ IDAG emission
void Scheduler::log_instr(const Instr& ins) {
    if (!log_) return;
    auto pbox = [&](const Box& b) {
        fprintf(log_, "[[%" PRId64 ",%" PRId64 ",%" PRId64 "],[%" PRId64 ",%" PRId64 ",%" PRId64 "]]", b.lo[0],
                b.lo[1], b.lo[2], b.hi[0], b.hi[1], b.hi[2]);
    };
    static const char* kinds[] = {"alloc", "free",  "copy",    "kernel",        "horizon",
                                  "epoch", "send", "receive", "split_receive", "await_receive"};
    static const char* reasons[] = {"resize", "coherence", "readback"};
    fprintf(log_, "{\"iid\":%" PRIu64 ",\"kind\":\"%s\",\"task\":", ins.iid, kinds[int(ins.kind)]);
    if (ins.task < 0)
        fprintf(log_, "null");
    else
        fprintf(log_, "%" PRId64, ins.task);
    switch (ins.kind) {
    case IKind::Alloc:
        fprintf(log_, ",\"buffer\":%u,\"aid\":%" PRId64 ",\"mem\":%d,\"box\":", ins.buffer, ins.aid, ins.mem);
        pbox(ins.box);
        break;
    case IKind::Free:
        fprintf(log_, ",\"buffer\":%u,\"aid\":%" PRId64 ",\"mem\":%d", ins.buffer, ins.aid, ins.mem);
        break;
    case IKind::Copy:
        fprintf(log_,
                ",\"buffer\":%u,\"reason\":\"%s\",\"src_aid\":%" PRId64 ",\"src_mem\":%d,\"dst_aid\":%" PRId64
                ",\"dst_mem\":%d,\"region\":[",
                ins.buffer, reasons[ins.reason], ins.src_aid, ins.src_mem, ins.dst_aid, ins.dst_mem);
        for (size_t i = 0; i < ins.region.size(); ++i) {
            if (i) fputc(',', log_);
            pbox(ins.region[i]);
        }
        fputc(']', log_);
        if (ins.readback >= 0) fprintf(log_, ",\"readback\":%" PRId64, ins.readback);
        break;
    case IKind::Kernel:
        fprintf(log_, ",\"device\":%d,\"chunk\":", ins.device);
        pbox(ins.chunk);
        fprintf(log_, ",\"bindings\":[");
        for (size_t i = 0; i < ins.bindings.size(); ++i) fprintf(log_, i ? ",%" PRId64 : "%" PRId64, ins.bindings[i]);
        fputc(']', log_);
        break;
    case IKind::Send:
        fprintf(log_, ",\"buffer\":%u,\"target\":%d,\"msg\":%" PRIu64 ",\"src_aid\":%" PRId64 ",\"src_mem\":%d,\"box\":",
                ins.buffer, ins.target, ins.msg, ins.src_aid, ins.src_mem);
        pbox(ins.box);
        break;
    case IKind::Receive:
    case IKind::SplitReceive:
    case IKind::AwaitReceive:
        fprintf(log_, ",\"buffer\":%u,\"transfer\":[%" PRId64 ",%u]", ins.buffer, ins.transfer, ins.buffer);
        if (ins.kind != IKind::AwaitReceive)
            fprintf(log_, ",\"dst_aid\":%" PRId64 ",\"dst_mem\":%d", ins.dst_aid, ins.dst_mem);
        fprintf(log_, ",\"region\":[");
        for (size_t i = 0; i < ins.region.size(); ++i) {
            if (i) fputc(',', log_);
            pbox(ins.region[i]);
        }
        fputc(']', log_);
        break;
    default:
        break;
    }
    fprintf(log_, ",\"deps\":[");
    for (size_t i = 0; i < ins.deps.size(); ++i) fprintf(log_, i ? ",%" PRIu64 : "%" PRIu64, ins.deps[i]);
    fprintf(log_, "]}\n");
}

int Scheduler::instr_owner(const Instr& ins) {
    switch (ins.kind) {
    case IKind::Alloc:
    case IKind::Free:
        return ins.mem >= 2 ? ins.mem - 2 : -1;
    case IKind::Kernel:
        return ins.device;
    case IKind::Copy:
        return ins.src_mem >= 2 ? ins.src_mem - 2 : (ins.dst_mem >= 2 ? ins.dst_mem - 2 : -1);
    default:
        return -1;
    }
}

void Scheduler::set_rank_filter(int rank, int world) {
    filter_rank_ = rank;
    filter_world_ = world;
    if (world > 1) {
        ring_iid_.assign(kOwnerRing, ~0ull);
        ring_owner_.assign(kOwnerRing, -1);
    }
}

bool Scheduler::owner_of(uint64_t iid, int* owner) const {
    if (ring_iid_.empty()) return false;
    const uint64_t k = iid & (kOwnerRing - 1);
    if (ring_iid_[k] == iid) {
        *owner = ring_owner_[k];
        return true;
    }
    auto it = alloc_owner_.find(int64_t(iid));
    if (it == alloc_owner_.end()) return false;
    *owner = it->second;
    return true;
}

uint64_t Scheduler::emit(Instr& ins, std::vector<uint64_t>& deps) {
    std::sort(deps.begin(), deps.end());
    deps.erase(std::unique(deps.begin(), deps.end()), deps.end());
    if (deps.empty()) deps.push_back(uint64_t(fallback_));  // R12 fallback edge
    ins.iid = next_iid_++;
    ins.deps = deps;
    // execution front: drop deps, add self
    std::vector<uint64_t>& nf = front_scratch_;
    nf.clear();
    std::set_difference(front_.begin(), front_.end(), deps.begin(), deps.end(), std::back_inserter(nf));
    nf.push_back(ins.iid);
    front_.swap(nf);
    st_.n_by_kind[int(ins.kind)]++;
    log_instr(ins);
    if (recording_) recording_->push_back(ins);
    if (filter_world_ > 1) {
        // all-gather members may run as a collective that every rank takes part
        // in (§8 a7): co-owned, like horizons, so their dependents reach everyone
        const int own = ins.coll_n ? -1 : instr_owner(ins);
        const uint64_t k = ins.iid & (kOwnerRing - 1);
        ring_owner_[k] = int8_t(own);
        ring_iid_[k] = ins.iid;
        if (ins.kind == IKind::Alloc) alloc_owner_[int64_t(ins.iid)] = own;
        bool rel = (ins.kind != IKind::Copy && ins.kind != IKind::Kernel) || own < 0 || own == filter_rank_ ||
                   ins.coll_n != 0 || (ins.kind == IKind::Copy && ins.dst_mem - 2 == filter_rank_);
        ins.dep_owner.resize(ins.deps.size());
        for (size_t i = 0; i < ins.deps.size(); ++i) {
            int o = 0;
            const bool known = owner_of(ins.deps[i], &o);
            ins.dep_owner[i] = known ? int8_t(o) : int8_t(-2);
            // a dependency this rank executes or co-owns (horizons, epochs): it must signal it
            if (!known || o < 0 || o == filter_rank_) rel = true;
        }
        if (!rel) return ins.iid;                 // other ranks' business: the executor never sees it
    }
    if (sink_) sink_->on_instr(ins);
    return ins.iid;
}

Scheduler::Alloc* Scheduler::new_alloc(uint32_t bid, int mem, const Box& box, int64_t tid) {
    Instr ins;
    ins.kind = IKind::Alloc;
    ins.task = tid;
    ins.buffer = bid;
    ins.aid = next_aid_++;
    ins.mem = mem;
    ins.box = box;
    std::vector<uint64_t> deps;
    const uint64_t iid = emit(ins, deps);
    auto a = std::unique_ptr<Alloc>(new Alloc{ins.aid, bid, mem, box, int64_t(iid), RegionMap<int64_t>(box, NONE),
                                              ReaderList{}});
    Alloc* p = a.get();
    allocs_[ins.aid] = std::move(a);
    bufs_[bid]->live[mem].push_back(p);
    st_.alloc_bytes_live += box.volume() * bufs_[bid]->elem_size;
    st_.alloc_bytes_peak = std::max(st_.alloc_bytes_peak, st_.alloc_bytes_live);
    return p;
}

void Scheduler::free_alloc(Alloc* a, int64_t tid) {
    if (filter_world_ > 1) alloc_owner_.erase(a->iid);
    std::vector<uint64_t> deps{uint64_t(a->iid)};
    for (auto& p : a->last_writer.e)
        if (p.first >= 0) deps.push_back(uint64_t(p.first));
    a->readers.all_ids([&](int64_t r) { deps.push_back(uint64_t(r)); });
    Instr ins;
    ins.kind = IKind::Free;
    ins.task = tid;
    ins.buffer = a->buffer;
    ins.aid = a->aid;
    ins.mem = a->mem;
    ins.box = a->box;
    emit(ins, deps);
    Buf& b = *bufs_[a->buffer];
    auto& v = b.live[a->mem];
    v.erase(std::find(v.begin(), v.end(), a));
    st_.alloc_bytes_live -= a->box.volume() * b.elem_size;
    allocs_.erase(a->aid);
}

uint64_t Scheduler::copy(int64_t tid, uint32_t bid, int reason, Alloc* src, Alloc* dst, const Region& reg,
                         int64_t rb, uint64_t coll, uint32_t coll_n) {
    // Table 1 `copy` with R12 dependencies
    std::vector<uint64_t> deps;
    auto add = [&](int64_t v) {
        if (v >= 0) deps.push_back(uint64_t(v));
    };
    if (src->iid >= 0) deps.push_back(uint64_t(src->iid));
    src->last_writer.for_values_in(reg, add);
    if (dst) {
        deps.push_back(uint64_t(dst->iid));
        dst->readers.ids_in(reg, [&](int64_t r) { deps.push_back(uint64_t(r)); });
        dst->last_writer.for_values_in(reg, add);
    }
    Instr ins;
    ins.kind = IKind::Copy;
    ins.task = tid;
    ins.buffer = bid;
    ins.reason = reason;
    ins.src_aid = src->aid;
    ins.src_mem = src->mem;
    ins.dst_aid = dst ? dst->aid : USER_AID;
    ins.dst_mem = dst ? dst->mem : 0;
    ins.region = reg;
    ins.readback = rb;
    ins.coll = coll;
    ins.coll_n = coll_n;
    const uint64_t iid = emit(ins, deps);
    const int64_t me = int64_t(iid);
    src->readers.add(me, reg);
    if (dst) {
        dst->last_writer.update(reg, me);
        dst->readers.remove(reg);
    }
    const uint64_t bytes = rvolume(reg) * bufs_[bid]->elem_size;
    st_.copies_by_reason[reason]++;
    st_.bytes_by_reason[reason] += bytes;
    if (ins.src_mem >= 2 && ins.dst_mem >= 2 && ins.src_mem != ins.dst_mem) st_.bytes_d2d_peer += bytes;
    return iid;
}

std::map<std::tuple<int64_t, int, int64_t>, Region> Scheduler::source_parts(Buf& buf, const Region& need, int m_dst) {
    return source_parts_q(buf, buf.uptodate.query(need), m_dst);
}

std::map<std::tuple<int64_t, int, int64_t>, Region> Scheduler::source_parts_q(
    Buf& buf, const std::vector<std::pair<Region, uint32_t>>& need_by_mask, int m_dst) {
    // producer split x source memory (R10) x source allocation
    std::map<std::tuple<int64_t, int, int64_t>, Region> parts;
    for (auto& q : need_by_mask) {
        const uint32_t mask = q.second;
        int s = -1;
        for (int m = 2; m < 32; ++m)
            if (((mask >> m) & 1u) && m != m_dst) {
                s = m;
                break;
            }
        if (s < 0) s = (mask & 2u) ? 1 : ((mask & 1u) ? 0 : -1);
        if (s < 0) continue;
        std::vector<Alloc*> srcs;
        if (s == 0) {
            srcs.push_back(buf.host.get());
        } else {
            auto it = buf.live.find(s);
            if (it != buf.live.end()) srcs = it->second;
            std::sort(srcs.begin(), srcs.end(), [](const Alloc* a, const Alloc* b) { return a->aid < b->aid; });
        }
        for (Alloc* a : srcs) {
            Region part = rinter(q.first, a->box);
            if (part.empty()) continue;
            for (auto& w : buf.orig_writer.query(part)) {
                Region& r = parts[std::make_tuple(w.second, s, a->aid)];
                r = runion(r, w.first);
            }
        }
    }
    return parts;
}

namespace {
// a box is one contiguous byte run of a row-major allocation over `a`
bool contiguous_in(const Box& b, const Box& a) {
    int d = 2;
    while (d > 0 && b.lo[d] == a.lo[d] && b.hi[d] == a.hi[d]) --d;
    for (int o = 0; o < d; ++o)
        if (b.extent(o) != 1) return false;
    return true;
}
}  // namespace

// §8 a7: a buffer read through chunk-independent mappers (`all`,
// `fixed`) whose coherence copies are, for every source device s, one
// contiguous box copied to each of the other G-1 devices is an all-gather
// (P:L161-163).  Returns buffer -> number of copies for each such
// buffer.  The copies stay as they are in the instruction graph; the executor
// may run the set as one collective.
std::map<uint32_t, uint32_t> Scheduler::all_gathers(
    const Cmd& c, const std::vector<std::pair<Key, std::vector<std::pair<std::tuple<int64_t, int, int64_t>, Region>>>>& pend,
    const std::map<Key, Alloc*>& binding) const {
    std::map<uint32_t, uint32_t> out;
    if (G_ < 2) return out;
    std::map<uint32_t, bool> eligible;
    for (const Access& a : c.desc->acc) {
        if (!is_read(a.mode)) continue;
        const bool ci = a.map.kind == MapKind::All || a.map.kind == MapKind::Fixed;
        auto it = eligible.find(a.buf);
        eligible[a.buf] = (it == eligible.end() ? true : it->second) && ci;
    }
    for (auto& e : eligible) {
        if (!e.second) continue;
        const uint32_t bid = e.first;
        // per source device: region and the set of receivers
        std::map<int, std::pair<Box, std::vector<int>>> roots;
        bool ok = true;
        uint32_t n = 0;
        for (auto& pk : pend) {
            if (pk.first.second != bid) continue;
            const int d = pk.first.first;
            auto bit = binding.find(pk.first);
            for (auto& p : pk.second) {
                const int ms = std::get<1>(p.first);
                if (ms < 2 || p.second.size() != 1 || bit == binding.end()) {
                    ok = false;
                    break;
                }
                const int s = ms - 2;
                const Box& b = p.second[0];
                const Alloc* src = allocs_.at(std::get<2>(p.first)).get();
                // one contiguous byte run in both allocations, robust to the
                // executor padding the innermost dimension of multi-dimensional
                // allocations: 1-D buffers, or a single row segment
                const Box& ext = bufs_.at(bid)->extent;
                int inner = 2;
                while (inner > 0 && ext.extent(inner) <= 1) --inner;
                bool row = true;
                for (int k = 0; k < inner; ++k)
                    if (b.extent(k) != 1) row = false;
                if (!contiguous_in(b, src->box) || !contiguous_in(b, bit->second->box) || !row) {
                    ok = false;
                    break;
                }
                auto rit = roots.find(s);
                if (rit == roots.end()) {
                    roots[s] = {b, {d}};
                } else {
                    if (!(rit->second.first == b) ||
                        std::find(rit->second.second.begin(), rit->second.second.end(), d) != rit->second.second.end()) {
                        ok = false;
                        break;
                    }
                    rit->second.second.push_back(d);
                }
                ++n;
            }
            if (!ok) break;
        }
        if (!ok || roots.empty()) continue;
        uint64_t min_bytes = ~0ull;
        for (auto& r : roots) {
            if (int(r.second.second.size()) != G_ - 1) ok = false;
            min_bytes = std::min<uint64_t>(min_bytes, r.second.first.volume() * bufs_.at(bid)->elem_size);
        }
        // small gathers (RSim's row, 84 KB per source at G = 4) are latency
        // bound: NCCL's group launch and rendezvous cost ~1 ms per set there,
        // against ~30 us for the peer pushes, so only sets whose
        // every source sends >= coll_min_bytes_ qualify
        if (ok && min_bytes >= coll_min_bytes_) out[bid] = n;
    }
    return out;
}

void Scheduler::compile(Cmd& c, const std::map<std::pair<uint32_t, int>, Box>& ant) {
    switch (c.kind) {
    case 0:
        compile_task(c, ant);
        break;
    case 1:
        compile_horizon(c);
        break;
    case 2:
        compile_epoch(c);
        break;
    case 3:  // R14 destroy
        for (uint32_t bid : c.destroy) {
            Buf& b = *bufs_[bid];
            std::vector<Alloc*> all;
            for (auto& kv : b.live) all.insert(all.end(), kv.second.begin(), kv.second.end());
            std::sort(all.begin(), all.end(), [](const Alloc* x, const Alloc* y) { return x->aid < y->aid; });
            for (Alloc* a : all) free_alloc(a, -1);
            bufs_.erase(bid);
        }
        break;
    }
}

std::map<Scheduler::Key, Scheduler::Alloc*> Scheduler::allocate(Cmd& c,
                                                                 const std::map<std::pair<uint32_t, int>, Box>& ant) {
    const int64_t tid = c.tid;
    std::map<Key, Alloc*> binding;
    // R9 allocation (Fig. 3): resize chain alloc -> copy -> free;
    // M1 requirements (device -1, virtual-node transfers) come first
    for (auto& kv : c.req) {
        const int m = 2 + kv.first.first;
        const uint32_t bid = kv.first.second;
        const Box& req = kv.second;
        Buf& buf = *bufs_[bid];
        std::vector<Alloc*>& live = buf.live[m];
        Alloc* hit = nullptr;
        for (Alloc* a : live)
            if (a->box.contains(req)) {
                hit = a;
                break;
            }
        if (hit) {
            binding[kv.first] = hit;
            continue;
        }
        Box bx = req;
        auto at = ant.find({bid, m});
        if (at != ant.end()) bx = bbox(bx, at->second);  // P:L589 widening
        std::vector<Alloc*> merged;
        for (;;) {
            merged.clear();
            Box nb = bx;
            for (Alloc* a : live)
                if (!intersect(a->box, bx).empty()) {
                    merged.push_back(a);
                    nb = bbox(nb, a->box);
                }
            if (nb == bx) break;
            bx = nb;
        }
        Alloc* na = new_alloc(bid, m, bx, tid);
        const Region utd = buf.uptodate.where([m](uint32_t mask) { return ((mask >> m) & 1u) != 0; });
        std::sort(merged.begin(), merged.end(), [](const Alloc* x, const Alloc* y) { return x->aid < y->aid; });
        for (Alloc* a : merged) {
            const Region src_reg = rinter(utd, a->box);
            for (auto& q : buf.orig_writer.query(src_reg)) copy(tid, bid, REASON_RESIZE, a, na, q.first, -1);
            free_alloc(a, tid);
        }
        binding[kv.first] = na;
    }
    return binding;
}

// Virtual-node mode, §3.4 Peer-to-Peer Communication (mirrors
// oracle/scheduler.py Runtime._transfers).  Outbound: the pushed
// region is made coherent in M1, then one send per rectangle of each
// original-producer fragment, each with a locally unique message id and a
// pilot.  Inbound: one receive into M1 when every consumer reads
// the same part of the awaited region, else a split receive plus one await
// receive per consumer-split fragment (R17).
void Scheduler::transfers(Cmd& c, std::map<Key, Alloc*>& binding, bool readback_consumer) {
    const int64_t tid = c.tid;
    for (auto& p : c.pushes) {
        const int target = std::get<0>(p);
        const uint32_t bid = std::get<1>(p);
        const Region& reg = std::get<2>(p);
        Buf& buf = *bufs_.at(bid);
        Alloc* m1 = binding.at({-1, bid});
        std::vector<std::pair<Region, uint32_t>> need;
        for (auto& q : buf.uptodate.query(reg))
            if (q.second != 0 && ((q.second >> 1) & 1u) == 0) need.push_back(std::move(q));
        if (!need.empty()) {
            auto parts = source_parts_q(buf, need, 1);
            for (auto& pp : parts) {
                const int64_t aid = std::get<2>(pp.first);
                Alloc* src = aid == HOST_AID ? buf.host.get() : allocs_.at(aid).get();
                copy(tid, bid, REASON_COHERENCE, src, m1, pp.second, -1);
            }
            for (auto& pp : parts) buf.uptodate.apply(pp.second, [](uint32_t mask) { return mask | 2u; });
        }
        for (auto& q : buf.orig_writer.query(reg)) {
            for (const Box& bx : q.first) {
                std::vector<uint64_t> deps{uint64_t(m1->iid)};
                m1->last_writer.for_values_in(Region{bx}, [&](int64_t v) {
                    if (v >= 0) deps.push_back(uint64_t(v));
                });
                Instr ins;
                ins.kind = IKind::Send;
                ins.task = tid;
                ins.buffer = bid;
                ins.target = target;
                ins.msg = next_msg_++;
                ins.src_aid = m1->aid;
                ins.src_mem = 1;
                ins.box = bx;
                const Pilot pl{node_, ins.msg, target, tid, bid, bx};
                if (pilot_sink_) pilot_sink_(pl);
                const uint64_t iid = emit(ins, deps);
                m1->readers.add(int64_t(iid), Region{bx});
            }
        }
    }
    for (auto& kv : c.awaits) {
        const uint32_t bid = kv.first;
        const Region& reg = kv.second;
        Buf& buf = *bufs_.at(bid);
        Alloc* m1 = binding.at({-1, bid});
        std::vector<Region> consumers;
        if (readback_consumer) {
            consumers.push_back(reg);
        } else {
            for (int d = 0; d < G_; ++d) {
                auto rit = c.reads.find({d, bid});
                if (rit == c.reads.end()) continue;
                Region x = rinter(rit->second, reg);
                if (!x.empty()) consumers.push_back(std::move(x));
            }
        }
        bool same = true;
        for (size_t i = 1; i < consumers.size(); ++i)
            if (!(consumers[i] == consumers[0])) same = false;
        std::vector<uint64_t> deps{uint64_t(m1->iid)};
        m1->readers.ids_in(reg, [&](int64_t r) { deps.push_back(uint64_t(r)); });
        m1->last_writer.for_values_in(reg, [&](int64_t v) {
            if (v >= 0) deps.push_back(uint64_t(v));
        });
        Instr ins;
        ins.kind = same ? IKind::Receive : IKind::SplitReceive;
        ins.task = tid;
        ins.buffer = bid;
        ins.transfer = tid;
        ins.dst_aid = m1->aid;
        ins.dst_mem = 1;
        ins.region = reg;
        const uint64_t r_iid = emit(ins, deps);
        std::vector<std::pair<Region, uint64_t>> frags;
        if (same) {
            frags.push_back({reg, r_iid});
        } else {
            std::vector<Region> atoms{reg};
            for (const Region& cr : consumers) {
                std::vector<Region> nxt;
                for (const Region& a : atoms) {
                    Region i = rinter(a, cr);
                    Region o = rdiff(a, cr);
                    if (!i.empty()) nxt.push_back(std::move(i));
                    if (!o.empty()) nxt.push_back(std::move(o));
                }
                atoms.swap(nxt);
            }
            for (const Region& a : atoms) {
                Instr aw;
                aw.kind = IKind::AwaitReceive;
                aw.task = tid;
                aw.buffer = bid;
                aw.transfer = tid;
                aw.region = a;
                std::vector<uint64_t> ad{r_iid};
                frags.push_back({a, emit(aw, ad)});
            }
        }
        for (auto& f : frags) {
            m1->last_writer.update(f.first, int64_t(f.second));
            m1->readers.remove(f.first);
            buf.orig_writer.update(f.first, int64_t(f.second));
        }
        buf.uptodate.update(reg, 2u);
    }
}

void Scheduler::compile_task(Cmd& c, const std::map<std::pair<uint32_t, int>, Box>& ant) {
    const int64_t tid = c.tid;
    const uint64_t base = next_iid_;
    // steady-state fast path (sched_memo.cpp): a recorded compile from the same
    // state (which fixes the live allocations, so it allocates nothing either)
    bool memo = memo_on_ && c.memo && c.pushes.empty() && c.awaits.empty() && c.remote_writes.empty();
    std::vector<int64_t>& sig = sig_scratch_;
    if (memo) {
        state_sig(c, base, sig);
        if (const CompileMemo* m = compile_lookup(*c.memo, sig)) {
            ++memo_hits_;
            compile_replay(*m, c, base);
            return;
        }
        ++memo_misses_;
    }
    std::map<Key, Alloc*> binding = allocate(c, ant);
    memo = memo && next_iid_ == base;   // record only compiles that allocate nothing
    std::vector<Instr> rec;
    SchedStats before;
    const uint64_t coll_before = next_coll_;
    if (memo) {
        before = st_;
        recording_ = &rec;
    }
    if (!c.pushes.empty() || !c.awaits.empty()) transfers(c, binding, false);
    // R10 coherence copies; masks as they stood before this task
    std::vector<std::tuple<uint32_t, Region, int>> updates;
    using Part = std::pair<std::tuple<int64_t, int, int64_t>, Region>;
    std::vector<std::pair<Key, std::vector<Part>>> pend;
    for (auto& kv : c.req) {
        auto rit = c.reads.find(kv.first);
        if (rit == c.reads.end() || rit->second.empty()) continue;
        const int m = 2 + kv.first.first;
        const uint32_t bid = kv.first.second;
        Buf& buf = *bufs_[bid];
        // need = reads - uptodate(M_d) - uninitialised, partitioned by mask in one query
        std::vector<std::pair<Region, uint32_t>> need;
        for (auto& q : buf.uptodate.query(rit->second))
            if (q.second != 0 && ((q.second >> m) & 1u) == 0) need.push_back(std::move(q));
        if (need.empty()) continue;
        auto parts = source_parts_q(buf, need, m);
        pend.emplace_back(kv.first, std::vector<Part>(parts.begin(), parts.end()));
    }
    const std::map<uint32_t, uint32_t> gathers = all_gathers(c, pend, binding);
    std::map<uint32_t, uint64_t> group;
    for (auto& g : gathers) group[g.first] = next_coll_++;
    st_.gather_sets += gathers.size();
    for (auto& pk : pend) {
        const uint32_t bid = pk.first.second;
        Buf& buf = *bufs_[bid];
        auto git = group.find(bid);
        for (auto& p : pk.second) {
            const int64_t aid = std::get<2>(p.first);
            Alloc* src = aid == HOST_AID ? buf.host.get() : allocs_.at(aid).get();
            if (git != group.end())
                copy(tid, bid, REASON_COHERENCE, src, binding[pk.first], p.second, -1, git->second, gathers.at(bid));
            else
                copy(tid, bid, REASON_COHERENCE, src, binding[pk.first], p.second, -1);
            updates.emplace_back(bid, p.second, 2 + pk.first.first);
        }
    }
    for (auto& u : updates) {
        const uint32_t bit = 1u << std::get<2>(u);
        bufs_[std::get<0>(u)]->uptodate.apply(std::get<1>(u), [bit](uint32_t mask) { return mask | bit; });
    }
    // R11 device kernels, device ascending
    std::map<int, uint64_t> kernels;
    for (int d = 0; d < G_; ++d) {
        const Box& ch = c.chunks[d];
        if (ch.empty()) continue;
        std::vector<uint64_t> deps;
        for (auto it = c.req.lower_bound({d, 0}); it != c.req.end() && it->first.first == d; ++it) {
            Alloc* a = binding[it->first];
            deps.push_back(uint64_t(a->iid));
            auto add = [&](int64_t v) {
                if (v >= 0) deps.push_back(uint64_t(v));
            };
            auto rit = c.reads.find(it->first);
            if (rit != c.reads.end()) a->last_writer.for_values_in(rit->second, add);
            auto wit = c.writes.find(it->first);
            if (wit != c.writes.end()) {
                a->readers.ids_in(wit->second, [&](int64_t r) { deps.push_back(uint64_t(r)); });
                a->last_writer.for_values_in(wit->second, add);
            }
        }
        Instr ins;
        ins.kind = IKind::Kernel;
        ins.task = tid;
        ins.device = d;
        ins.chunk = ch;
        ins.desc = c.desc;
        for (const Access& acc : c.desc->acc) {
            auto b = binding.find({d, acc.buf});
            ins.bindings.push_back(b != binding.end() ? b->second->aid : 0);
        }
        const uint64_t k = emit(ins, deps);
        const int64_t me = int64_t(k);
        for (auto it = c.req.lower_bound({d, 0}); it != c.req.end() && it->first.first == d; ++it) {
            Alloc* a = binding[it->first];
            auto rit = c.reads.find(it->first);
            if (rit != c.reads.end()) a->readers.add(me, rit->second);
            auto wit = c.writes.find(it->first);
            if (wit != c.writes.end()) {
                a->last_writer.update(wit->second, me);
                a->readers.remove(wit->second);
            }
        }
        kernels[d] = k;
    }
    for (auto& kv : c.writes) {
        Buf& buf = *bufs_[kv.first.second];
        buf.orig_writer.update(kv.second, int64_t(kernels[kv.first.first]));
        buf.uptodate.update(kv.second, 1u << (2 + kv.first.first));
    }
    // virtual-node mode: what other nodes wrote in this task is stale here
    for (auto& kv : c.remote_writes) {
        Buf& buf = *bufs_.at(kv.first);
        buf.uptodate.update(kv.second, 0u);
        buf.orig_writer.update(kv.second, NONE);
    }
    if (memo) {
        recording_ = nullptr;
        compile_store(std::vector<int64_t>(sig), c, base, std::move(rec), before, coll_before);
    }
}

void Scheduler::subsume(int64_t h) {
    // horizon / epoch application (R7)
    auto f = [h](int64_t v) { return (v >= 0 && v < h) ? h : v; };
    for (auto& kv : bufs_) {
        Buf& b = *kv.second;
        b.orig_writer.map_values(f);
        for (auto& lv : b.live)
            for (Alloc* a : lv.second) {
                a->last_writer.map_values(f);
                a->readers.subsume(h);
            }
        if (b.host) {
            b.host->last_writer.map_values(f);
            b.host->readers.subsume(h);
        }
    }
}

void Scheduler::compile_horizon(Cmd& c) {
    // depends on every instruction of the execution front
    Instr ins;
    ins.kind = IKind::Horizon;
    ins.task = c.tid;
    std::vector<uint64_t> deps(front_);
    const uint64_t h = emit(ins, deps);
    if (pending_h_ >= 0) {
        subsume(pending_h_);
        fallback_ = pending_h_;
    }
    pending_h_ = int64_t(h);
}

void Scheduler::compile_epoch(Cmd& c) {
    if (!c.pushes.empty() || !c.awaits.empty()) {   // virtual-node readback gather
        std::map<Key, Alloc*> binding = allocate(c, {});
        transfers(c, binding, true);
    }
    if (c.rb >= 0) {  // R13 readback into the user pointer
        Buf& buf = *bufs_[c.rb_buf];
        Region need = rinter(buf.uptodate.where([](uint32_t mask) { return mask != 0; }), c.rb_box);
        if (!need.empty()) {
            auto parts = source_parts(buf, need, 0);
            for (auto& p : parts) {
                const int64_t aid = std::get<2>(p.first);
                Alloc* src = aid == HOST_AID ? buf.host.get() : allocs_.at(aid).get();
                copy(c.tid, c.rb_buf, REASON_READBACK, src, nullptr, p.second, c.rb);
            }
        }
    }
    Instr ins;
    ins.kind = IKind::Epoch;
    ins.task = c.tid;
    std::vector<uint64_t> deps(front_);
    const uint64_t e = emit(ins, deps);
    subsume(int64_t(e));
    fallback_ = int64_t(e);
    pending_h_ = -1;
}

}  // namespace cel

namespace cel {
void Scheduler::debug_dump(FILE* f) const {
    for (auto& kv : bufs_) {
        const Buf& b = *kv.second;
        size_t ob = 0, ub = 0;
        for (auto& e : b.orig_writer.e) ob += e.second.size();
        for (auto& e : b.uptodate.e) ub += e.second.size();
        fprintf(f, "buffer %u: orig_writer %zu entries / %zu boxes, uptodate %zu entries / %zu boxes\n", kv.first,
                b.orig_writer.e.size(), ob, b.uptodate.e.size(), ub);
        for (auto& lv : b.live)
            for (const Alloc* a : lv.second) {
                size_t lb = 0, rb = 0;
                for (auto& e : a->last_writer.e) lb += e.second.size();
                for (auto& e : a->readers.recs) rb += e.r.size();
                fprintf(f, "  alloc %lld mem %d: last_writer %zu/%zu readers %zu/%zu\n", (long long)a->aid, a->mem,
                        a->last_writer.e.size(), lb, a->readers.recs.size(), rb);
            }
    }
    fprintf(f, "tdag cp entries %zu, front %zu\n", cp_.size(), front_.size());
}
}  // namespace cel
