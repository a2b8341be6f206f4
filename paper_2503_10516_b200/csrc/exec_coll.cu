// Executor: the `all` gather as an NCCL collective.
#include "exec_impl.hpp"

namespace cel {

bool Executor::coll_init() {
    if (coll_state_) return coll_state_ > 0;
    coll_state_ = -1;
    if (cfg_.world > 1) {
        if (!nccl_id_set_) return false;
        ncclUniqueId id;
        memcpy(&id, nccl_id_, sizeof id);
        ncclComm_t c = nullptr;
        set_dev(cfg_.rank);
        // collective over all ranks; every rank reaches the same first group
        if (trace_) fprintf(stderr, "[cel r%d] ncclCommInitRank ...\n", cfg_.rank);
        if (g_nccl.init_rank(&c, cfg_.world, id, cfg_.rank) != ncclSuccess) return false;
        if (trace_) fprintf(stderr, "[cel r%d] ncclCommInitRank done\n", cfg_.rank);
        comms_.assign(1, c);
    } else {
        std::vector<ncclComm_t> cs(G_, nullptr);
        if (g_nccl.init_all(cs.data(), G_, phys_.data()) != ncclSuccess) return false;
        comms_.assign(cs.begin(), cs.end());
    }
    coll_state_ = 1;
    return true;
}

// §8 a7: an all-gather copy set (Scheduler::all_gathers) executed as
// one group of NCCL broadcasts, one per source device, in place in every
// device's allocation (the `all` mapper; NVLink / NVSwitch
// collectives instead of G(G-1) separate pushes).
// §8 a7 / §8(e) as a hand-written kernel: each source device stores its chunk
// into every receiver's allocation (P2P stores over NVLink / NVSwitch, into
// IPC-mapped arenas across processes) and bumps each receiver's gather
// counter; each receiver's stream waits until its counter has counted every
// chunk sent to it so far (cuStreamWaitValue64 GEQ, no host round trip).  One
// launch and one wait per device per set, instead of G - 1 pushes with their
// events and flags each, or an NCCL group.  Every rank keeps the same
// expected counts: they follow from the replicated instruction graph.
bool Executor::exec_coll_p2p(const std::vector<Instr>& m) {
    if (!p2p_gather_) return false;
    const uint32_t es = bufinfo_.at(m[0].buffer).es;
    if (es % 4) return false;
    std::map<int, std::vector<const Instr*>> roots;
    for (const Instr& x : m) {
        if (x.region.size() != 1 || x.src_mem < 2 || x.dst_mem < 2) return false;
        roots[x.src_mem - 2].push_back(&x);
    }
    for (auto& rt : roots) {
        if (int(rt.second.size()) > kMaxGatherDst) return false;
        for (const Instr* x : rt.second)
            if (!(x->region[0] == rt.second[0]->region[0])) return false;   // one box per source
    }
    auto lin = [](const Box& b, const Box& a) {
        return uint64_t(((b.lo[0] - a.lo[0]) * a.extent(1) + (b.lo[1] - a.lo[1])) * a.extent(2) + (b.lo[2] - a.lo[2]));
    };
    std::vector<int> locals;
    if (cfg_.world > 1) locals.push_back(cfg_.rank);
    else
        for (int v = 0; v < G_; ++v) locals.push_back(v);
    // wait for the dependencies of every member a local device sends or receives
    for (int v : locals) {
        Token t;
        for (const Instr& x : m)
            if (x.src_mem - 2 == v || x.dst_mem - 2 == v) {
                cur_ins_ = &x;
                merge(t, local_part(x.deps));
            }
        set_dev(v);
        wait_token(v * kStreamsPerDev + S_PUSH, t);
    }
    uint64_t bytes_total = 0;
    std::vector<Token> src_done(G_);
    for (auto& rt : roots) {
        const int s = rt.first;
        const Box& b = rt.second[0]->region[0];
        bytes_total += b.volume() * es * rt.second.size();
        if (owner_rank(s) != cfg_.rank) continue;
        P2PGatherArgs a;
        memset(&a, 0, sizeof a);
        const AllocRec& S = allocs_.at(rt.second[0]->src_aid);
        a.src = base_of(S) + lin(b, S.box) * es;
        a.bytes = b.volume() * es;
        uintptr_t al = reinterpret_cast<uintptr_t>(a.src) | uintptr_t(a.bytes);
        for (const Instr* x : rt.second) {
            const AllocRec& D = allocs_.at(x->dst_aid);
            const int dd = x->dst_mem - 2;
            a.dst[a.ndst] = base_of(D) + lin(b, D.box) * es;
            a.counter[a.ndst] = reinterpret_cast<unsigned long long*>(arenas_[dd].base + gather_off_);
            al |= reinterpret_cast<uintptr_t>(a.dst[a.ndst]);
            a.ndst++;
        }
        a.vec4 = (al & 15) == 0;
        a.ctr = reinterpret_cast<unsigned*>(arenas_[s].base + gather_off_ + 64);
        const int sidx = s * kStreamsPerDev + S_PUSH;
        set_dev(s);
        if (cfg_.profile && prof_sample(K_NUM + 3)) {
            Prof p{K_NUM + 3, prof_event(s), prof_event(s), s, m[0].iid, sidx, now_ns()};
            cudaEventRecord(p.a, streams_[sidx].s);
            st_.kernel_launches += launch_p2p_gather(a, streams_[sidx].s);
            cudaEventRecord(p.b, streams_[sidx].s);
            prof_pending_.push_back(p);
        } else {
            st_.kernel_launches += launch_p2p_gather(a, streams_[sidx].s);
        }
        check(cudaGetLastError(), "P2P gather launch");
        if (cfg_.world > 1) src_done[s] = record(sidx);
    }
    for (const Instr& x : m) gather_exp_[x.dst_mem - 2]++;
    std::vector<Token> tv(G_);
    for (int v : locals) {
        const int sidx = v * kStreamsPerDev + S_PUSH;
        set_dev(v);
        checkd(g_drv.wait64(reinterpret_cast<CUstream>(streams_[sidx].s),
                            reinterpret_cast<CUdeviceptr>(arenas_[v].base + gather_off_), gather_exp_[v],
                            CU_STREAM_WAIT_VALUE_GEQ),
               "cuStreamWaitValue64 (gather counter)");
        tv[v] = record(sidx);
    }
    // a member is complete once its receiver's counter has counted it: that
    // wait also implies the source kernel's reads and stores are done, so
    // the receiver's event alone stands for the copy (no cross-device waits
    // for the next row's kernel); a source rank that is not the receiver
    // holds the source kernel's completion as its part
    for (const Instr& x : m) {
        const int sd = x.src_mem - 2, dd = x.dst_mem - 2;
        Token lt;
        if (owner_rank(dd) == cfg_.rank) merge(lt, tv[dd]);
        else if (owner_rank(sd) == cfg_.rank) merge(lt, src_done[sd]);
        if (cfg_.world > 1) {
            ltok_[x.iid] = lt;
            for (int rk : {owner_rank(sd), owner_rank(dd)})
                if (rk != cfg_.rank) lt.remote.push_back({rk, x.iid});
        }
        tok_[x.iid] = lt;
    }
    st_.coll_groups++;
    st_.coll_copies += m.size();
    st_.coll_p2p++;
    st_.bytes_copy[2] += bytes_total;
    return true;
}

void Executor::exec_coll(const std::vector<Instr>& m) {
    const uint32_t es = bufinfo_.at(m[0].buffer).es;
    if (!parked_.empty()) {
        if (try_fuse(m)) return;                  // the producing row kernels carry the gather (exec_fuse.cu)
        flush_parked();                           // the members depend on them: launch them plainly first
    }
    if (exec_coll_mc(m)) return;                  // NVLS multicast stores (exec_mc.cu)
    if (exec_coll_p2p(m)) return;                 // P2P gather kernels
    uint64_t min_bytes = ~0ull;
    for (const Instr& x : m) min_bytes = std::min<uint64_t>(min_bytes, rvolume(x.region) * es);
    if (cfg_.world == 1 && (!coll_ || min_bytes < coll_min_bytes_)) {
        // one process, and no NCCL or a set too small for it (flagged for the
        // multicast path, which did not apply): the members run as the peer
        // pushes they are.  (Multi-process runs only flag sets the scheduler's
        // identical threshold admits, so every rank joins the same groups.)
        for (const Instr& x : m) {
            cur_ins_ = &x;
            exec_copy(x);
            if (grown_) note_use(x);
        }
        return;
    }
    if (!coll_init()) {
        errmsg_ = "NCCL communicator setup failed (set collective = 0 to use peer pushes)";
        err_ = E_NCCL;
        return;
    }
    // local devices taking part: all G (one process) or this rank's device
    std::vector<int> locals;
    if (cfg_.world > 1) locals.push_back(cfg_.rank);
    else
        for (int v = 0; v < G_; ++v) locals.push_back(v);
    auto lin = [](const Box& b, const Box& a) {          // element offset of b.lo in a row-major over a
        return uint64_t(((b.lo[0] - a.lo[0]) * a.extent(1) + (b.lo[1] - a.lo[1])) * a.extent(2) + (b.lo[2] - a.lo[2]));
    };
    std::vector<Token> tv(G_);
    for (int v : locals) {
        Token t;
        for (const Instr& x : m)
            if (x.src_mem - 2 == v || x.dst_mem - 2 == v) {
                cur_ins_ = &x;
                merge(t, local_part(x.deps));
            }
        const int sidx = v * kStreamsPerDev + S_PUSH;
        set_dev(v);
        wait_token(sidx, t);
    }
    // roots in ascending device order; a root's region is the same box for all receivers
    std::map<int, std::vector<const Instr*>> roots;
    for (const Instr& x : m) roots[x.src_mem - 2].push_back(&x);
    std::vector<Prof> profs;
    if (cfg_.profile)
        for (int v : locals) {
            const int sidx = v * kStreamsPerDev + S_PUSH;
            set_dev(v);                  // profile events belong to the device's stream
            Prof p{K_NUM + 3, prof_event(v), prof_event(v), v, m[0].iid, sidx, now_ns()};
            cudaEventRecord(p.a, streams_[sidx].s);
            profs.push_back(p);
        }
    uint64_t bytes_total = 0;
    // address of root s's box in local device v's memory
    auto addr = [&](int s, int v) -> char* {
        const std::vector<const Instr*>& xs = roots.at(s);
        const Box& b = xs[0]->region[0];
        if (v == s) {
            const AllocRec& S = allocs_.at(xs[0]->src_aid);
            return base_of(S) + lin(b, S.box) * es;
        }
        for (const Instr* x : xs)
            if (x->dst_mem - 2 == v) {
                const AllocRec& D = allocs_.at(x->dst_aid);
                return base_of(D) + lin(b, D.box) * es;
            }
        return nullptr;
    };
    // every device a root with an equal-size box at offset root x count of one
    // contiguous layout (N-body's P): one in-place ncclAllGather per device,
    // which NCCL may run over NVLink SHARP (NVLS) multicast
    static const char* agenv = getenv("CEL_COLL_AG");
    bool ag = g_nccl.allgather && !(agenv && agenv[0] == '0') && int(roots.size()) == G_;
    size_t count = 0;
    if (ag) {
        count = size_t(roots.begin()->second[0]->region[0].volume()) * es;
        for (auto& rt : roots)
            if (size_t(rt.second[0]->region[0].volume()) * es != count) ag = false;
        for (size_t k = 0; k < locals.size() && ag; ++k) {
            char* b0 = addr(0, locals[k]);
            for (int sr = 0; sr < G_ && ag; ++sr)
                if (!b0 || addr(sr, locals[k]) != b0 + size_t(sr) * count) ag = false;
        }
    }
    ncclResult_t r = g_nccl.group_start();
    if (ag) {
        for (size_t k = 0; k < locals.size() && r == ncclSuccess; ++k) {
            const int v = locals[k];
            char* b0 = addr(0, v);
            const int sidx = v * kStreamsPerDev + S_PUSH;
            r = g_nccl.allgather(b0 + size_t(v) * count, b0, count, ncclUint8, static_cast<ncclComm_t>(comms_[k]),
                                 streams_[sidx].s);
        }
        bytes_total = count * size_t(G_) * size_t(G_ - 1);
        st_.coll_allgathers++;
        roots.clear();                          // nothing left for broadcasts
    }
    for (auto& rt : roots) {
        const int s = rt.first;
        const Instr& x0 = *rt.second[0];
        const Box& b = x0.region[0];
        const AllocRec& S = allocs_.at(x0.src_aid);
        const size_t bytes = size_t(b.volume()) * es;
        bytes_total += bytes * rt.second.size();
        for (size_t k = 0; k < locals.size() && r == ncclSuccess; ++k) {
            const int v = locals[k];
            char* buf = nullptr;
            if (v == s) {
                buf = base_of(S) + lin(b, S.box) * es;
            } else {
                for (const Instr* x : rt.second)
                    if (x->dst_mem - 2 == v) {
                        const AllocRec& D = allocs_.at(x->dst_aid);
                        buf = base_of(D) + lin(b, D.box) * es;
                    }
            }
            if (!buf) {
                errmsg_ = "all-gather set without a receiver on a device";
                err_ = E_STATE;
                g_nccl.group_end();
                return;
            }
            const int sidx = v * kStreamsPerDev + S_PUSH;
            r = g_nccl.bcast(buf, buf, bytes, ncclUint8, s, static_cast<ncclComm_t>(comms_[k]), streams_[sidx].s);
        }
    }
    const ncclResult_t r2 = g_nccl.group_end();
    if (trace_) fprintf(stderr, "[cel r%d] broadcast group of %zu copies issued\n", cfg_.rank, m.size());
    if (r != ncclSuccess || r2 != ncclSuccess) {
        errmsg_ = std::string("ncclBroadcast: ") + g_nccl.errstr(r != ncclSuccess ? r : r2);
        err_ = E_NCCL;
        return;
    }
    for (auto& p : profs) {
        set_dev(p.dev);
        cudaEventRecord(p.b, streams_[p.stream].s);
        prof_pending_.push_back(p);
    }
    for (int v : locals) {
        set_dev(v);                  // events come from the device's pool
        tv[v] = record(v * kStreamsPerDev + S_PUSH);
    }
    for (const Instr& x : m) {
        const int sd = x.src_mem - 2, dd = x.dst_mem - 2;
        Token lt;
        for (int v : locals)
            if (v == sd || v == dd) merge(lt, tv[v]);
        if (cfg_.world > 1) {
            // the source's rank (sendbuff reusable) and the destination's rank
            // (data arrived) each hold part of the completion
            ltok_[x.iid] = lt;
            for (int rk : {owner_rank(sd), owner_rank(dd)})
                if (rk != cfg_.rank) lt.remote.push_back({rk, x.iid});
        }
        tok_[x.iid] = lt;
    }
    st_.coll_groups++;
    st_.coll_copies += m.size();
    st_.bytes_copy[2] += bytes_total;   // NCCL's kernels are library launches: not in kernel_launches
}

}  // namespace cel
