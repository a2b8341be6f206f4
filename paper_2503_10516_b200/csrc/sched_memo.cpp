// Steady-state fast path of the IDAG generator (DESIGN.md §2 "compile memo";
// SURVEY NEXT-2, PAPER.md L526 / L754-759: the scheduler must stay ahead of
// sub-100 us device steps).
//
// compile_task() is a deterministic function of (a) the task's shape -- range,
// split, accessors -- and (b) the state of the buffers it accesses: the
// up-to-date masks, the original producers, every live allocation with its
// last writers and readers, and the fallback edge.  Instruction ids enter
// that state only through differences from the next id to be emitted: shifting
// every id in the state by d shifts every id compile_task emits and every id
// it leaves in the state by d.  So once a shape has been compiled from a state
// that, with ids taken relative to the next iid, equals a recorded one, the
// recorded instructions and end state are replayed shifted by d -- the same
// instructions (R9-R12) the full compile would emit, at the cost of a state
// signature and the emits.  An iterative program reaches such a periodic state
// after a few horizons (WaveSim: two shapes, period = the horizon step).
//
// Not memoised: compiles that allocate (R9 resize chains), virtual-node
// transfers, and a shape's first submission.
#include "sched_impl.hpp"

#include <cstring>

namespace cel {

uint64_t detail::memo_hash(const std::vector<int64_t>& v) {
    uint64_t h = v.size();
    for (int64_t x : v) h ^= uint64_t(x) + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    return h;
}

namespace {
void put_box(std::vector<int64_t>& s, const Box& b) {
    s.insert(s.end(), b.lo, b.lo + 3);
    s.insert(s.end(), b.hi, b.hi + 3);
}
void put_region(std::vector<int64_t>& s, const Region& r) {
    s.push_back(int64_t(r.size()));
    for (const Box& b : r) put_box(s, b);
}
// an instruction id relative to the next iid; specials (NONE, HOST_AID) apart
inline int64_t rel(int64_t v, uint64_t base) { return v >= 0 ? int64_t(base) - v : v - (int64_t(1) << 62); }
inline int64_t shift(int64_t v, int64_t d) { return v >= 0 ? v + d : v; }
constexpr size_t kMaxPrep = 64, kMaxCompile = 16;   // shapes; recorded compiles per shape
}  // namespace

struct Scheduler::CompileMemo {
    struct AllocPost {
        int64_t aid;
        RegionMap<int64_t> last_writer;
        ReaderList readers;
    };
    struct BufPost {
        uint32_t bid;
        RegionMap<uint32_t> uptodate;
        RegionMap<int64_t> orig_writer;
        std::vector<AllocPost> allocs;   // b.live in map order, then the host allocation
    };
    std::vector<int64_t> sig;
    uint64_t base = 0;                   // next iid when recorded
    std::vector<uint64_t> alloc_iids;    // sorted: dependencies on these stay as they are
    std::vector<Instr> out;              // emitted instructions, as recorded
    std::vector<BufPost> bufs;           // end state, ids as recorded
    uint64_t copies_by_reason[3] = {}, bytes_by_reason[3] = {}, bytes_d2d_peer = 0, gather_sets = 0;
    uint64_t coll_base = 0, coll_n = 0;
};

struct Scheduler::PrepMemo {
    std::vector<int64_t> key;
    std::vector<Box> chunks;
    std::map<Key, Region> reads, writes;
    std::map<Key, Box> req;
    std::map<uint32_t, Region> breads, bwrites;
    std::vector<std::unique_ptr<CompileMemo>> compiled;   // the states this shape was compiled from
    size_t next_slot = 0;
};


void Scheduler::shape_key(const TaskDesc& d, std::vector<int64_t>& k) {
    k.clear();
    k.push_back(d.dims);
    put_box(k, d.range);
    k.push_back(d.split);
    k.push_back(int64_t(d.acc.size()));
    for (const Access& a : d.acc) {
        k.push_back(a.buf);
        k.push_back(a.mode);
        k.push_back(int64_t(a.map.kind));
        k.insert(k.end(), a.map.border, a.map.border + 3);
        put_box(k, a.map.fixed);
        k.insert(k.end(), a.map.from_kernel_dim, a.map.from_kernel_dim + 3);
    }
}

bool Scheduler::prep_lookup(const std::vector<int64_t>& key, uint64_t h, Cmd& c, std::map<uint32_t, Region>& reads,
                            std::map<uint32_t, Region>& writes) {
    auto it = prep_memo_.find(h);
    if (it == prep_memo_.end() || it->second->key != key) return false;
    const PrepMemo& m = *it->second;
    c.memo = it->second;
    c.chunks = m.chunks;
    c.reads = m.reads;
    c.writes = m.writes;
    c.req = m.req;
    reads = m.breads;
    writes = m.bwrites;
    return true;
}

void Scheduler::prep_store(std::vector<int64_t>&& key, uint64_t h, const Cmd& c, const std::map<uint32_t, Region>& reads,
                           const std::map<uint32_t, Region>& writes) {
    if (prep_memo_.size() >= kMaxPrep) prep_memo_.clear();
    auto m = std::make_shared<PrepMemo>();
    m->key = std::move(key);
    m->chunks = c.chunks;
    m->reads = c.reads;
    m->writes = c.writes;
    m->req = c.req;
    m->breads = reads;
    m->bwrites = writes;
    prep_memo_[h] = std::move(m);
}

void Scheduler::state_sig(const Cmd& c, uint64_t base, std::vector<int64_t>& s) const {
    s.clear();
    s.push_back(G_);
    s.push_back(rel(fallback_, base));
    s.push_back(int64_t(coll_min_bytes_));
    std::vector<uint32_t> bids;
    for (const Access& a : c.desc->acc) bids.push_back(a.buf);
    std::sort(bids.begin(), bids.end());
    bids.erase(std::unique(bids.begin(), bids.end()), bids.end());
    auto put_alloc = [&](const Alloc& a) {
        s.push_back(a.aid);
        put_box(s, a.box);
        s.push_back(a.iid);   // absolute: kernels and copies depend on the alloc instruction itself
        s.push_back(int64_t(a.last_writer.e.size()));
        for (auto& e : a.last_writer.e) {
            s.push_back(rel(e.first, base));
            put_region(s, e.second);
        }
        s.push_back(int64_t(a.readers.recs.size()));
        for (auto& r : a.readers.recs) {
            s.push_back(rel(r.id, base));
            put_region(s, r.r);
        }
    };
    for (uint32_t bid : bids) {
        const Buf& b = *bufs_.at(bid);
        s.push_back(bid);
        s.push_back(int64_t(b.uptodate.e.size()));
        for (auto& e : b.uptodate.e) {
            s.push_back(e.first);
            put_region(s, e.second);
        }
        s.push_back(int64_t(b.orig_writer.e.size()));
        for (auto& e : b.orig_writer.e) {
            s.push_back(rel(e.first, base));
            put_region(s, e.second);
        }
        s.push_back(int64_t(b.live.size()));
        for (auto& lv : b.live) {
            s.push_back(lv.first);
            s.push_back(int64_t(lv.second.size()));
            for (const Alloc* a : lv.second) put_alloc(*a);
        }
        s.push_back(b.host ? 1 : 0);
        if (b.host) put_alloc(*b.host);
    }
}

const Scheduler::CompileMemo* Scheduler::compile_lookup(const PrepMemo& p, const std::vector<int64_t>& sig) {
    for (const auto& m : p.compiled)
        if (m->sig.size() == sig.size() && std::memcmp(m->sig.data(), sig.data(), sig.size() * sizeof(int64_t)) == 0)
            return m.get();
    return nullptr;
}

void Scheduler::compile_store(std::vector<int64_t>&& sig, const Cmd& c, uint64_t base, std::vector<Instr>&& out,
                              const SchedStats& before, uint64_t coll_before) {
    auto m = std::unique_ptr<CompileMemo>(new CompileMemo);
    m->sig = std::move(sig);
    m->base = base;
    m->out = std::move(out);
    std::vector<uint32_t> bids;
    for (const Access& a : c.desc->acc) bids.push_back(a.buf);
    std::sort(bids.begin(), bids.end());
    bids.erase(std::unique(bids.begin(), bids.end()), bids.end());
    for (uint32_t bid : bids) {
        const Buf& b = *bufs_.at(bid);
        CompileMemo::BufPost bp;
        bp.bid = bid;
        bp.uptodate = b.uptodate;
        bp.orig_writer = b.orig_writer;
        for (auto& lv : b.live)
            for (const Alloc* a : lv.second) {
                bp.allocs.push_back({a->aid, a->last_writer, a->readers});
                if (a->iid >= 0) m->alloc_iids.push_back(uint64_t(a->iid));
            }
        if (b.host) bp.allocs.push_back({b.host->aid, b.host->last_writer, b.host->readers});
        m->bufs.push_back(std::move(bp));
    }
    for (int r = 0; r < 3; ++r) {
        m->copies_by_reason[r] = st_.copies_by_reason[r] - before.copies_by_reason[r];
        m->bytes_by_reason[r] = st_.bytes_by_reason[r] - before.bytes_by_reason[r];
    }
    std::sort(m->alloc_iids.begin(), m->alloc_iids.end());
    m->bytes_d2d_peer = st_.bytes_d2d_peer - before.bytes_d2d_peer;
    m->gather_sets = st_.gather_sets - before.gather_sets;
    m->coll_base = coll_before;
    m->coll_n = next_coll_ - coll_before;
    PrepMemo& p = *c.memo;
    if (p.compiled.size() < kMaxCompile) {
        p.compiled.push_back(std::move(m));
    } else {
        p.compiled[p.next_slot] = std::move(m);
        p.next_slot = (p.next_slot + 1) % kMaxCompile;
    }
}

void Scheduler::compile_replay(const CompileMemo& m, Cmd& c, uint64_t base) {
    const int64_t d = int64_t(base) - int64_t(m.base);
    const uint64_t coll_shift = next_coll_ - m.coll_base;
    std::vector<uint64_t> deps;
    for (const Instr& r : m.out) {
        Instr ins = r;
        ins.task = c.tid;
        if (ins.kind == IKind::Kernel) ins.desc = c.desc;
        if (ins.coll) ins.coll += coll_shift;
        deps.resize(r.deps.size());
        for (size_t i = 0; i < r.deps.size(); ++i)
            deps[i] = std::binary_search(m.alloc_iids.begin(), m.alloc_iids.end(), r.deps[i])
                          ? r.deps[i]
                          : uint64_t(int64_t(r.deps[i]) + d);
        ins.deps.clear();
        ins.dep_owner.clear();
        emit(ins, deps);
    }
    next_coll_ += m.coll_n;
    auto install = [d](Alloc& a, const CompileMemo::AllocPost& p) {
        a.last_writer = p.last_writer;
        for (auto& e : a.last_writer.e) e.first = shift(e.first, d);
        a.readers = p.readers;
        for (auto& r : a.readers.recs) r.id = shift(r.id, d);
    };
    for (const CompileMemo::BufPost& bp : m.bufs) {
        Buf& b = *bufs_.at(bp.bid);
        b.uptodate = bp.uptodate;
        b.orig_writer = bp.orig_writer;
        for (auto& e : b.orig_writer.e) e.first = shift(e.first, d);
        size_t i = 0;
        for (auto& lv : b.live)
            for (Alloc* a : lv.second) install(*a, bp.allocs[i++]);
        if (b.host) install(*b.host, bp.allocs[i++]);
    }
    for (int r = 0; r < 3; ++r) {
        st_.copies_by_reason[r] += m.copies_by_reason[r];
        st_.bytes_by_reason[r] += m.bytes_by_reason[r];
    }
    st_.bytes_d2d_peer += m.bytes_d2d_peer;
    st_.gather_sets += m.gather_sets;
}

}  // namespace cel
