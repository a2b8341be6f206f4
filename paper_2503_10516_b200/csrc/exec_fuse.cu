// Executor: an RSim row's all-gather fused into the row kernel (SURVEY §8 a7
// and §8(e); "RSim puts more pressure on the communication
// logic").
//
// The gather of row t is the coherence copy set of task t + 1 (every device
// reads all rows), so it reaches the executor after the kernel that writes
// row t.  The executor therefore parks that kernel instruction (and anything
// that depends on it) until the next all-gather set arrives: if the set's
// copies read exactly the rows the parked kernels write, each kernel is
// launched with a peer epilogue (`launch_rsim_fused`): every thread also
// stores its element into every receiving device's allocation, and the last
// CTA bumps the receivers' gather counters -- the same counters and expected
// counts as the P2P gather kernels (exec_coll.cu).  Receivers' compute
// streams wait for their counter, so the next row's kernel follows with no
// copy launch, event or flag in between.  Anything else that depends on a
// parked kernel (a horizon, an epoch, a drain) releases the parked
// instructions in order with the ordinary path.  The instruction graph and
// its log are unchanged: the set's copies complete when the fused kernels'
// stores have landed.
#include "exec_impl.hpp"

namespace cel {

bool Executor::depends_on_parked(const Instr& ins) const {
    for (uint64_t j : ins.deps)
        if (parked_iids_.count(j)) return true;
    return false;
}

// A row kernel this rank launches, fusable as a gather source.
bool Executor::park_candidate(const Instr& ins) {
    if (!fuse_rows_ || flushing_ || ins.kind != IKind::Kernel || !ins.desc || ins.desc->kernel != K_RSIM_ROW) return false;
    if (owner_rank(ins.device) != cfg_.rank) return false;
    KArgs a;
    build_kargs(ins, a);
    return rsim_fusable(a);
}

void Executor::park(const Instr& ins) {
    parked_.push_back(ins);
    parked_iids_.insert(ins.iid);
}

// Release every parked instruction, in order, through the ordinary path.
void Executor::flush_parked() {
    if (parked_.empty()) return;
    std::vector<Instr> q;
    q.swap(parked_);
    parked_iids_.clear();
    flushing_ = true;
    for (const Instr& x : q) {
        on_instr_impl(x);
        cur_ins_ = nullptr;
    }
    flushing_ = false;
}

// The set `m` (complete, about to execute): fuse it into the parked row
// kernels that produce it.  True: done (kernels launched, members' tokens
// set, the rest of the parked instructions released).
bool Executor::try_fuse(const std::vector<Instr>& m) {
    if (parked_.empty()) return false;
    const uint32_t es = bufinfo_.at(m[0].buffer).es;
    if (es != 4) return false;
    std::map<int, std::vector<const Instr*>> roots;
    for (const Instr& x : m) {
        if (x.region.size() != 1 || x.src_mem < 2 || x.dst_mem < 2) return false;
        roots[x.src_mem - 2].push_back(&x);
    }
    // every local source's members: one box, written by a parked row kernel of
    // that device through its write accessor, into allocations of rows x cols
    std::map<int, const Instr*> kernel_of;
    for (auto& rt : roots) {
        const int s = rt.first;
        if (int(rt.second.size()) > kMaxGatherDst) return false;
        const Box& b = rt.second[0]->region[0];
        for (const Instr* x : rt.second)
            if (!(x->region[0] == b) || allocs_.at(x->dst_aid).box.extent(2) != 1) return false;
        if (owner_rank(s) != cfg_.rank) continue;
        const Instr* k = nullptr;
        for (const Instr& p : parked_)
            if (p.kind == IKind::Kernel && p.device == s && p.desc && p.desc->kernel == K_RSIM_ROW &&
                std::find(rt.second[0]->deps.begin(), rt.second[0]->deps.end(), p.iid) != rt.second[0]->deps.end()) {
                const Box w = map_access(p.desc->acc[1].map, p.chunk, bufinfo_.at(p.desc->acc[1].buf).extent);
                if (w == b && p.bindings[1] == rt.second[0]->src_aid) k = &p;
            }
        if (!k) return false;
        kernel_of[s] = k;
    }
    std::vector<int> locals;
    if (cfg_.world > 1) locals.push_back(cfg_.rank);
    else
        for (int v = 0; v < G_; ++v) locals.push_back(v);
    // launch: each local source's kernel after its own dependencies and those
    // of its members (readers of the receivers' rows), on its compute stream
    std::vector<Token> src_done(G_);
    for (auto& ks : kernel_of) {
        const int s = ks.first;
        const Instr& k = *ks.second;
        const int sidx = s * kStreamsPerDev + S_COMPUTE;
        set_dev(s);
        Token t;
        cur_ins_ = &k;
        for (uint64_t j : k.deps) merge(t, dep_token(j));
        for (const Instr* x : roots.at(s)) {
            cur_ins_ = x;
            for (uint64_t j : x->deps)
                if (j != k.iid) merge(t, dep_token(j));
        }
        wait_token(sidx, t);
        KArgs a;
        build_kargs(k, a);
        PeerOut po;
        memset(&po, 0, sizeof po);
        for (const Instr* x : roots.at(s)) {
            const AllocRec& D = allocs_.at(x->dst_aid);
            const int dd = x->dst_mem - 2;
            po.base[po.n] = base_of(D);
            po.lo0[po.n] = D.box.lo[0];
            po.lo1[po.n] = D.box.lo[1];
            po.n1[po.n] = D.box.extent(1);
            po.counter[po.n] = reinterpret_cast<unsigned long long*>(arenas_[dd].base + gather_off_);
            po.n++;
        }
        po.ctr = reinterpret_cast<unsigned*>(arenas_[s].base + gather_off_ + 64);
        int n = 0;
        if (cfg_.profile && prof_sample(K_RSIM_ROW)) {
            Prof p{K_RSIM_ROW, prof_event(s), prof_event(s), s, k.iid, sidx, now_ns()};
            cudaEventRecord(p.a, streams_[sidx].s);
            n = launch_rsim_fused(a, po, streams_[sidx].s);
            cudaEventRecord(p.b, streams_[sidx].s);
            prof_pending_.push_back(p);
        } else {
            n = launch_rsim_fused(a, po, streams_[sidx].s);
        }
        check(cudaGetLastError(), "fused RSim row launch");
        if (n != 1 && !err_) {
            errmsg_ = "fused RSim row: kernel no longer applicable";
            err_ = E_STATE;
            return true;
        }
        st_.kernel_launches += n;
        st_.workload_launches += n;
        tok_[k.iid] = record(sidx);
        src_done[s] = tok_[k.iid];
        if (cfg_.world > 1) kind_of_[k.iid] = k.device;
        if (grown_) note_use(k);
    }
    // the parked kernels ran: release them from the park (their dependents
    // stay parked until below)
    std::vector<Instr> rest;
    for (const Instr& p : parked_) {
        bool launched = false;
        for (auto& ks : kernel_of) launched = launched || ks.second->iid == p.iid;
        if (!launched) rest.push_back(p);
    }
    for (const Instr& x : m) gather_exp_[x.dst_mem - 2]++;
    std::vector<Token> tv(G_);
    for (int v : locals) {
        const int sidx = v * kStreamsPerDev + S_COMPUTE;
        set_dev(v);
        checkd(g_drv.wait64(reinterpret_cast<CUstream>(streams_[sidx].s),
                            reinterpret_cast<CUdeviceptr>(arenas_[v].base + gather_off_), gather_exp_[v],
                            CU_STREAM_WAIT_VALUE_GEQ),
               "cuStreamWaitValue64 (fused gather counter)");
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
    st_.coll_fused++;
    // what else was parked (dependents of the kernels) now runs in order
    parked_.clear();
    parked_iids_.clear();
    for (const Instr& p : rest) park(p);
    if (!deferred_signals_.empty()) flush_deferred_signals();
    flush_parked();
    return true;
}

}  // namespace cel
