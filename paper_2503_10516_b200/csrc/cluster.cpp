// Virtual-node mode: N node schedulers and the replicated
// push / await-push bookkeeping between them (mirrors oracle/cluster.py, R17).
#include <cstdio>

#include "sched_impl.hpp"

namespace cel {
using namespace detail;

Cluster::Cluster(int n_nodes, int devices_per_node, int lookahead, int horizon_step, bool checks,
                 const std::vector<InstrSink*>& sinks, const std::vector<FILE*>& logs)
    : N_(n_nodes), D_(devices_per_node) {
    for (int k = 0; k < N_; ++k) {
        s_.emplace_back(new Scheduler(D_, lookahead, horizon_step, checks, sinks[k], logs[k]));
        s_.back()->set_node(k);
    }
}

int Cluster::buffer_create(int dims, const int64_t extent[3], uint32_t elem_size, bool host_init, uint32_t* out) {
    uint32_t bid = 0;
    for (int k = 0; k < N_; ++k) {
        const int rc = s_[k]->buffer_create(dims, extent, elem_size, host_init, &bid);
        if (rc != E_OK) return rc;
    }
    const Box ext = s_[0]->extent(bid);
    t_.emplace(bid, Track{RegionMap<int64_t>(ext, host_init ? -2 : -1),
                          RegionMap<uint32_t>(ext, host_init ? uint32_t((1ull << N_) - 1) : 0u)});
    *out = bid;
    return E_OK;
}

// For each receiving node m and buffer b: the elements of need[m][b] that m
// does not hold come from their owner (never-written elements: nothing).
// Pushes are coalesced per (owner, receiver, buffer); the await
// region of m is the union.
void Cluster::transfers(const std::vector<std::map<uint32_t, Region>>& need, std::vector<std::vector<Push>>& pushes,
                        std::vector<std::map<uint32_t, Region>>& awaits) const {
    std::vector<std::map<std::pair<int, uint32_t>, Region>> pm(N_);
    awaits.assign(N_, {});
    for (int m = 0; m < N_; ++m) {
        for (auto& kv : need[m]) {
            const Track& tr = t_.at(kv.first);
            const Region held = tr.holders.where([m](uint32_t mask) { return ((mask >> m) & 1u) != 0; });
            const Region miss = rdiff(kv.second, held);
            for (auto& q : tr.owner.query(miss)) {
                const int64_t n = q.second;
                if (n < 0 || n == m) continue;
                Region& r = pm[n][{m, kv.first}];
                r = runion(r, q.first);
                Region& a = awaits[m][kv.first];
                a = runion(a, q.first);
            }
        }
    }
    pushes.assign(N_, {});
    for (int n = 0; n < N_; ++n)
        for (auto& kv : pm[n]) pushes[n].push_back(Push{kv.first.first, kv.first.second, kv.second});
}

int Cluster::task_submit(const TaskDesc& desc, uint64_t* tid_out, std::string* err) {
    for (const Access& a : desc.acc)
        if (!s_[0]->has_buffer(a.buf)) {
            if (err) *err = "access to an unknown or destroyed buffer";
            return E_INVALID;
        }
    if (desc.dims < 1 || desc.dims > 3) {
        if (err) *err = "task dims must be 1..3";
        return E_INVALID;
    }
    // R17: command chunks, 1-D over the nodes; the task's split applies inside a node
    const std::vector<Box> chunks = split(desc.range, N_, 0);
    std::vector<std::map<uint32_t, Region>> rd(N_), wr(N_);
    for (int n = 0; n < N_; ++n) {
        if (chunks[n].empty()) continue;
        for (const Access& a : desc.acc) {
            Region reg;
            const int rc = mapper_region(a.map, chunks[n], s_[0]->extent(a.buf), &reg);
            if (rc != E_OK) {
                if (err) *err = "range mapper result outside the buffer extent";
                return rc;
            }
            if (reg.empty()) continue;
            if (is_read(a.mode)) rd[n][a.buf] = runion(rd[n][a.buf], reg);
            if (is_write(a.mode)) wr[n][a.buf] = runion(wr[n][a.buf], reg);
        }
    }
    // §4.4 overlapping writes across nodes
    for (int i = 0; i < N_; ++i)
        for (int j = i + 1; j < N_; ++j)
            for (auto& kv : wr[i]) {
                auto it = wr[j].find(kv.first);
                if (it != wr[j].end() && !rinter(kv.second, it->second).empty()) {
                    if (err) {
                        char buf[160];
                        snprintf(buf, sizeof buf, "nodes %d and %d write overlapping regions of buffer %u", i, j,
                                 kv.first);
                        *err = buf;
                    }
                    return E_OVERLAPPING_WRITE;
                }
            }
    std::map<uint32_t, Region> reads, writes;
    for (int n = 0; n < N_; ++n) {
        for (auto& kv : rd[n]) reads[kv.first] = runion(reads[kv.first], kv.second);
        for (auto& kv : wr[n]) writes[kv.first] = runion(writes[kv.first], kv.second);
    }
    std::vector<std::vector<Push>> pushes;
    std::vector<std::map<uint32_t, Region>> awaits;
    transfers(rd, pushes, awaits);
    int status = E_OK;
    for (int n = 0; n < N_; ++n) {
        std::map<uint32_t, Region> remote;
        for (int k = 0; k < N_; ++k) {
            if (k == n) continue;
            for (auto& kv : wr[k]) remote[kv.first] = runion(remote[kv.first], kv.second);
        }
        uint64_t tid = 0;
        const int rc = s_[n]->task_submit_node(desc, chunks[n], reads, writes, pushes[n], awaits[n], remote, &tid,
                                               err);
        if (rc < 0) return rc;   // a node rejected a chunk: only node-local validation can fail here
        if (n == 0) {
            status = rc;
            if (tid_out) *tid_out = tid;
        }
    }
    for (int m = 0; m < N_; ++m)
        for (auto& kv : awaits[m])
            t_.at(kv.first).holders.apply(kv.second, [m](uint32_t mask) { return mask | (1u << m); });
    for (int n = 0; n < N_; ++n)
        for (auto& kv : wr[n]) {
            Track& tr = t_.at(kv.first);
            tr.owner.update(kv.second, int64_t(n));
            tr.holders.update(kv.second, 1u << n);
        }
    return status;
}

void Cluster::wait() {
    for (auto& s : s_) s->wait();
}

int Cluster::readback(uint32_t bid, const Box& box, int64_t* rb_out, std::string* err) {
    if (!s_[0]->has_buffer(bid)) {
        if (err) *err = "unknown buffer";
        return E_INVALID;
    }
    if (!s_[0]->extent(bid).contains(box)) {
        if (err) *err = "readback box outside the buffer extent";
        return E_OUT_OF_BOUNDS;
    }
    std::vector<std::map<uint32_t, Region>> need(N_);
    need[0][bid] = Region{box.normalized()};
    std::vector<std::vector<Push>> pushes;
    std::vector<std::map<uint32_t, Region>> awaits;
    transfers(need, pushes, awaits);
    const int64_t rb = s_[0]->alloc_readback_id();
    for (int n = 0; n < N_; ++n) s_[n]->epoch_node(n == 0 ? rb : -1, bid, box, pushes[n], awaits[n]);
    for (auto& kv : awaits[0]) t_.at(kv.first).holders.apply(kv.second, [](uint32_t mask) { return mask | 1u; });
    if (rb_out) *rb_out = rb;
    return E_OK;
}

int Cluster::destroy(uint32_t bid, std::string* err) {
    for (auto& s : s_) {
        const int rc = s->destroy(bid, err);
        if (rc != E_OK) return rc;
    }
    t_.erase(bid);
    return E_OK;
}

void Cluster::shutdown() {
    for (auto& s : s_) s->shutdown();
}

}  // namespace cel
