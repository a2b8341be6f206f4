// Executor: WaveSim's halo exchange fused into the stencil launches (SURVEY §7
// step 6 and NEXT-2; §5 WaveSim strong scaling, L490 §3.6: the
// coherence copies between neighbouring devices are the per-step overhead).
//
// Multi-process runs on distinct GPUs.  A wave5 kernel instruction this rank
// executes is held back until the next instruction that depends on it: the
// coherence copies that push its boundary rows to the neighbours (emitted at
// the start of the next task's compilation) attach to it, horizons in between
// wait with it.  The launch (`launch_wave5_halo`) then
//   - stores each attached copy's rows from the CTAs that compute them
//     straight into the receiver's allocation (IPC-mapped peer memory over
//     NVLink), after the copy's remote dependencies -- readers of the
//     receiver's rows, whose flags arrive in this GPU's slots -- and the last
//     such CTA writes the receiver's flag slot with the copy's id: exactly
//     what the copy and its signal would have done;
//   - awaits each incoming copy (a neighbour's push into rows this launch
//     reads) in the CTAs that read those rows, not on the stream: interior
//     CTAs never wait, and consecutive steps follow each other on the compute
//     stream with programmatic dependent launch.
// Same instructions, same dependencies, same flags; the instruction graph and
// its log are unchanged.  Anything else that depends on the held-back work
// releases it first; anything the fused launch cannot express (a copy that is
// not a whole-row band of the chunk, too many flags) runs the ordinary way.
#include "exec_impl.hpp"

namespace cel {

bool Executor::halo_depends(const Instr& ins) const {
    for (uint64_t j : ins.deps)
        if (halo_iids_.count(j)) return true;
    return false;
}

// A wave5 instruction this rank launches whose vector kernel applies, or an
// RSim row whose TMA kernel applies (its row goes to every other rank).
bool Executor::halo_candidate(const Instr& ins) {
    if (!fuse_halo_ || halo_flushing_ || ins.kind != IKind::Kernel || !ins.desc) return false;
    if (ins.desc->kernel != K_WAVE5 && ins.desc->kernel != K_RSIM_ROW) return false;
    if (owner_rank(ins.device) != cfg_.rank || cfg_.bounds_check) return false;
    KArgs a;
    build_kargs(ins, a);
    if (ins.desc->kernel == K_RSIM_ROW) return rsim_fusable(a);
    // row bands only (the 1-D split): with 2-D tiles the column halos stay
    // copies, and awaiting them in the kernel holds every strip of the tile
    // (3441 vs 4422 steps/s at 4 B200 with the shell / interior path)
    const Box& ext = bufinfo_.at(ins.desc->acc[0].buf).extent;
    if (ins.chunk.lo[1] != ext.lo[1] || ins.chunk.hi[1] != ext.hi[1]) return false;
    unsigned gx = 0, gy = 0;
    return wave5_strip(a, &gx, &gy) > 0;
}

// A coherence copy of rows the held-back kernel writes, into another GPU.
bool Executor::halo_attach(const Instr& ins) {
    const Instr& k = halo_kernel_;
    static int mode = -1;                          // CEL_HALO_MODE bit 1 off: pushes stay copies (A/B)
    if (mode < 0) {
        const char* e = getenv("CEL_HALO_MODE");
        mode = e ? atoi(e) : 3;
    }
    if (!(mode & 1)) return false;
    if (ins.kind != IKind::Copy || ins.coll_n) return false;
    if (k.desc->kernel == K_WAVE5 && int(halo_pushes_.size()) >= kHaloMax) return false;
    if (ins.src_mem - 2 != k.device || ins.dst_mem < 2 || owner_rank(ins.dst_mem - 2) == cfg_.rank) return false;
    if (phys_[ins.dst_mem - 2] == phys_[k.device] || ins.src_aid != k.bindings[1] || ins.region.size() != 1) return false;
    if (std::find(ins.deps.begin(), ins.deps.end(), k.iid) == ins.deps.end()) return false;
    for (uint64_t j : ins.deps)
        if (j != k.iid && halo_iids_.count(j)) return false;
    const Box& b = ins.region[0];
    if (k.desc->kernel == K_RSIM_ROW) {
        // the row the kernel writes, to another rank's allocation of whole rows
        const Box w = map_access(k.desc->acc[1].map, k.chunk, bufinfo_.at(k.desc->acc[1].buf).extent);
        auto d = allocs_.find(ins.dst_aid);
        if (!(b == w) || int(halo_pushes_.size()) >= kMaxGatherDst || d == allocs_.end() || d->second.es != 4 ||
            d->second.box.extent(2) != 1)
            return false;
        halo_pushes_.push_back(ins);
        halo_iids_.insert(ins.iid);
        return true;
    }
    if (b.lo[1] != k.chunk.lo[1] || b.hi[1] != k.chunk.hi[1] || b.lo[0] < k.chunk.lo[0] || b.hi[0] > k.chunk.hi[0] ||
        b.extent(2) != 1)
        return false;
    auto d = allocs_.find(ins.dst_aid);
    if (d == allocs_.end() || d->second.es != 4 || d->second.box.extent(2) != 1 || d->second.box.extent(1) % 4 ||
        (b.lo[1] - d->second.box.lo[1]) % 4 || (reinterpret_cast<uintptr_t>(base_of(d->second)) & 15))
        return false;
    halo_pushes_.push_back(ins);
    halo_iids_.insert(ins.iid);
    return true;
}

// An RSim row with its pushes to the other ranks (`rsim_row_tma_t<true>` in
// flag mode): every thread stores its element into each receiver's
// allocation, the last CTA writes the receivers' flag slots; the incoming
// copies of the rows the kernel reads are awaited by the kernel.  One launch
// per row instead of a launch, G - 1 copies, G - 1 flag writes and G - 1
// stream waits.
bool Executor::halo_launch_rsim(const Instr& k, const std::vector<Instr>& pushes) {
    const int dev = k.device;
    const int sidx = dev * kStreamsPerDev + S_COMPUTE;
    Stream& cs = streams_[sidx];
    KArgs a;
    build_kargs(k, a);
    if (!rsim_fusable(a)) return false;
    PeerOut po;
    memset(&po, 0, sizeof po);
    po.flags = 1;
    Token t;
    std::vector<uint64_t> newly;
    static int mode = -1;                          // CEL_HALO_MODE bit 2 off: incoming copies awaited by the stream
    if (mode < 0) {
        const char* e = getenv("CEL_HALO_MODE");
        mode = e ? atoi(e) : 3;
    }
    cur_ins_ = &k;
    for (uint64_t j : k.deps) {
        Token dt = dep_token(j);
        auto ci = copy_info_.find(j);
        if ((mode & 2) && dt.local.empty() && dt.remote.size() == 1 && ci != copy_info_.end() &&
            ci->second.dst_aid == k.bindings[0]) {
            // the flag is the remote entry's (an elided copy's token is its
            // own dependencies': the id to wait for is not always j)
            const uint64_t rj = dt.remote[0].second;
            const uint64_t key = (uint64_t(dt.remote[0].first) << 56) ^ rj;
            if (cs.waited_remote.count(key)) continue;     // an earlier launch on this stream waited for it
            if (po.n_in == kMaxGatherDst) return false;
            po.in_flag[po.n_in] = reinterpret_cast<const unsigned long long*>(sig_slot(dev, dt.remote[0].first, rj));
            po.in_value[po.n_in] = rj;
            // rows the awaited copy may have written: its own region, or -- an
            // elided copy standing for its dependencies -- any row
            const int64_t r0 = (rj == j) ? ci->second.bb.lo[0] : 0;
            po.in_row0 = po.n_in == 0 ? r0 : std::min(po.in_row0, r0);
            po.n_in++;
            newly.push_back(key);
        } else {
            merge(t, dt);
        }
    }
    for (const Instr& p : pushes) {
        cur_ins_ = &p;
        for (uint64_t j : p.deps) {
            if (j == k.iid) continue;
            Token dt = dep_token(j);
            merge(t, Token{dt.local, {}});
            for (auto& r : dt.remote) {
                const uint64_t key = (uint64_t(r.first) << 56) ^ r.second;
                if (cs.waited_remote.count(key)) continue;
                const unsigned long long* f = reinterpret_cast<const unsigned long long*>(sig_slot(dev, r.first, r.second));
                bool dup = false;
                for (int i = 0; i < po.n_wait; ++i) dup = dup || po.wait_flag[i] == f;
                if (dup) continue;
                if (po.n_wait == kMaxGatherDst) return false;
                po.wait_flag[po.n_wait] = f;
                po.wait_value[po.n_wait] = r.second;
                po.n_wait++;
                newly.push_back(key);
            }
        }
        const AllocRec& D = allocs_.at(p.dst_aid);
        po.base[po.n] = base_of(D);
        po.lo0[po.n] = D.box.lo[0];
        po.lo1[po.n] = D.box.lo[1];
        po.n1[po.n] = D.box.extent(1);
        po.flag[po.n] = reinterpret_cast<unsigned long long*>(sig_slot(p.dst_mem - 2, cfg_.rank, p.iid));
        po.value[po.n] = p.iid;
        po.n++;
    }
    po.ctr = reinterpret_cast<unsigned*>(arenas_[dev].base + gather_off_ + 128);
    po.done = reinterpret_cast<unsigned*>(arenas_[dev].base + gather_off_ + 192);
    if (trace_) {
        const AllocRec& R = allocs_.at(k.bindings[0]);
        const AllocRec& Wa = allocs_.at(k.bindings[1]);
        fprintf(stderr, "[cel r%d] rsim fused iid %llu t %u R aid %lld box [%lld,%lld)x[%lld,%lld) abs %lld W aid %lld abs %lld in %d war %d out %d\n",
                cfg_.rank, (unsigned long long)k.iid, a.t, (long long)k.bindings[0], (long long)R.box.lo[0], (long long)R.box.hi[0],
                (long long)R.box.lo[1], (long long)R.box.hi[1], (long long)R.absorbed_into, (long long)k.bindings[1],
                (long long)Wa.absorbed_into, po.n_in, po.n_wait, po.n);
        for (const Instr& p : pushes) {
            const AllocRec& D = allocs_.at(p.dst_aid);
            fprintf(stderr, "[cel r%d]   push iid %llu -> dev %d aid %lld box [%lld,%lld)x[%lld,%lld) abs %lld region [%lld,%lld)x[%lld,%lld)\n",
                    cfg_.rank, (unsigned long long)p.iid, p.dst_mem - 2, (long long)p.dst_aid, (long long)D.box.lo[0],
                    (long long)D.box.hi[0], (long long)D.box.lo[1], (long long)D.box.hi[1], (long long)D.absorbed_into,
                    (long long)p.region[0].lo[0], (long long)p.region[0].hi[0], (long long)p.region[0].lo[1],
                    (long long)p.region[0].hi[1]);
        }
    }
    cur_ins_ = &k;
    set_dev(dev);
    wait_token(sidx, t);
    // row chain: when the previous operation on the compute stream was a
    // fused row and this one needs no other wait, wait for the previous row's
    // local stores (its CTAs' count) instead of its grid, whose tail waits for
    // the NVLink stores' acknowledgements (CEL_RSIM_CHAIN=0: off)
    static int chain_env = -1;
    if (chain_env < 0) {
        const char* e = getenv("CEL_RSIM_CHAIN");
        chain_env = (e && e[0] == '0') ? 0 : 1;
    }
    if (rsim_chain_.empty()) rsim_chain_.resize(size_t(G_));
    RsimChain& rc = rsim_chain_[size_t(dev)];
    const unsigned grid = unsigned((k.chunk.volume() + 127) / 128);
    po.ctr_last = rc.ctr + grid - 1;
    po.done_wait = rc.done;
    po.chain = chain_env && rc.done > 0 && cs.seq == rc.seq && cs.waits == rc.waits ? 1 : 0;
    int n = 0;
    if (cfg_.profile && prof_sample(K_RSIM_ROW)) {
        Prof pr{K_RSIM_ROW, prof_event(dev), prof_event(dev), dev, k.iid, sidx, now_ns()};
        cudaEventRecord(pr.a, cs.s);
        n = launch_rsim_fused(a, po, cs.s);
        cudaEventRecord(pr.b, cs.s);
        prof_pending_.push_back(pr);
    } else {
        n = launch_rsim_fused(a, po, cs.s);
    }
    check(cudaGetLastError(), "fused RSim row launch (flags)");
    if (n != 1) {
        if (!err_) {
            errmsg_ = "fused RSim row: kernel no longer applicable";
            err_ = E_STATE;
        }
        return true;
    }
    for (uint64_t key : newly) cs.waited_remote.insert(key);
    rc.ctr += grid;
    rc.done += grid;
    st_.kernel_launches += 1;
    st_.workload_launches += 1;
    st_.halo_fused += pushes.size();
    st_.halo_in_waits += uint64_t(po.n_in);
    const Token done = record(sidx);
    rc.seq = cs.seq;
    rc.waits = cs.waits;
    st_.halo_chained += uint64_t(po.chain);
    tok_[k.iid] = done;
    kind_of_[k.iid] = dev;
    for (const Instr& p : pushes) {
        tok_[p.iid] = done;
        kind_of_[p.iid] = dev;
        copy_info_[p.iid] = CopyInfo{p.src_aid, p.dst_aid, rbbox(p.region), p.region};
        signalled_.insert(p.iid * uint64_t(cfg_.world) + uint64_t(owner_rank(p.dst_mem - 2)));
        st_.bytes_copy[2] += rvolume(p.region) * 4;
    }
    if (grown_) {
        note_use(k);
        for (const Instr& p : pushes) note_use(p);
    }
    return true;
}

// Launch the held-back kernel with its pushes, or say it cannot.
bool Executor::halo_launch(const Instr& k, const std::vector<Instr>& pushes) {
    if (k.desc->kernel == K_RSIM_ROW) return halo_launch_rsim(k, pushes);
    const int dev = k.device;
    const int sidx = dev * kStreamsPerDev + S_COMPUTE;
    KArgs a;
    build_kargs(k, a);
    unsigned gx = 0, gy = 0;
    const int64_t h = wave5_strip(a, &gx, &gy);
    if (h <= 0) return false;
    HaloArgs hx;
    memset(&hx, 0, sizeof hx);
    Token t;
    // incoming: the kernel's dependencies on other ranks' copies into the
    // allocation it reads u from (their rows), awaited by the reading CTAs
    // (CEL_HALO_MODE bit 2 off: by the stream, for A/B)
    static int mode = -1;
    if (mode < 0) {
        const char* e = getenv("CEL_HALO_MODE");
        mode = e ? atoi(e) : 3;
    }
    cur_ins_ = &k;
    for (uint64_t j : k.deps) {
        Token dt = dep_token(j);
        auto ci = copy_info_.find(j);
        if ((mode & 2) && dt.local.empty() && dt.remote.size() == 1 && ci != copy_info_.end() && ci->second.dst_aid == k.bindings[0] &&
            hx.n_in < kHaloMax) {
            const uint64_t rj = dt.remote[0].second;     // the remote entry's id (see halo_launch_rsim)
            hx.in_flag[hx.n_in] = reinterpret_cast<const unsigned long long*>(sig_slot(dev, dt.remote[0].first, rj));
            hx.in_value[hx.n_in] = rj;
            hx.in_r0[hx.n_in] = ci->second.bb.lo[0];
            hx.in_r1[hx.n_in] = ci->second.bb.hi[0];
            hx.n_in++;
        } else {
            merge(t, dt);
        }
    }
    // outgoing: each push's other dependencies -- local ones on the stream,
    // remote ones (the receivers' readers) awaited by the pushing CTAs
    if (halo_ctr_.empty()) halo_ctr_.assign(size_t(G_), std::array<unsigned, kHaloMax>{});
    std::array<unsigned, kHaloMax> ctr = halo_ctr_[size_t(dev)];
    for (const Instr& p : pushes) {
        cur_ins_ = &p;
        for (uint64_t j : p.deps) {
            if (j == k.iid) continue;
            Token dt = dep_token(j);
            merge(t, Token{dt.local, {}});
            for (auto& r : dt.remote) {
                const unsigned long long* f = reinterpret_cast<const unsigned long long*>(sig_slot(dev, r.first, r.second));
                bool dup = false;
                for (int i = 0; i < hx.n_war; ++i) dup = dup || (hx.war_flag[i] == f && hx.war_value[i] >= r.second);
                if (dup) continue;
                if (hx.n_war == kHaloMax) return false;
                hx.war_flag[hx.n_war] = f;
                hx.war_value[hx.n_war] = r.second;
                hx.n_war++;
            }
        }
        const int i = hx.n_out;
        const AllocRec& D = allocs_.at(p.dst_aid);
        const Box& b = p.region[0];
        hx.base[i] = base_of(D);
        hx.lo0[i] = D.box.lo[0];
        hx.lo1[i] = D.box.lo[1];
        hx.n1[i] = D.box.extent(1);
        hx.r0[i] = b.lo[0];
        hx.r1[i] = b.hi[0];
        hx.flag[i] = reinterpret_cast<unsigned long long*>(sig_slot(p.dst_mem - 2, cfg_.rank, p.iid));
        hx.value[i] = p.iid;
        // CTAs that compute the rows: every column block of each strip they touch
        const int64_t s0 = (b.lo[0] - k.chunk.lo[0]) / h, s1 = (b.hi[0] - 1 - k.chunk.lo[0]) / h;
        const unsigned n = unsigned(s1 - s0 + 1) * gx;
        hx.ctr[i] = reinterpret_cast<unsigned*>(arenas_[dev].base + gather_off_ + 256) + i;
        hx.ctr_last[i] = ctr[size_t(i)] + n - 1;
        ctr[size_t(i)] += n;
        hx.n_out++;
    }
    cur_ins_ = &k;
    set_dev(dev);
    wait_token(sidx, t);
    int n = 0;
    if (cfg_.profile && prof_sample(K_WAVE5)) {
        Prof pr{K_WAVE5, prof_event(dev), prof_event(dev), dev, k.iid, sidx, now_ns()};
        cudaEventRecord(pr.a, streams_[sidx].s);
        n = launch_wave5_halo(a, hx, streams_[sidx].s);
        cudaEventRecord(pr.b, streams_[sidx].s);
        prof_pending_.push_back(pr);
    } else {
        n = launch_wave5_halo(a, hx, streams_[sidx].s);
    }
    check(cudaGetLastError(), "fused wave5 halo launch");
    if (n != 1) {
        if (!err_) {
            errmsg_ = "fused wave5 halo launch: kernel no longer applicable";
            err_ = E_STATE;
        }
        return true;
    }
    halo_ctr_[size_t(dev)] = ctr;
    st_.kernel_launches += 1;
    st_.workload_launches += 1;
    st_.halo_fused += pushes.size();
    st_.halo_in_waits += uint64_t(hx.n_in);
    const Token done = record(sidx);
    tok_[k.iid] = done;
    kind_of_[k.iid] = dev;
    for (const Instr& p : pushes) {
        tok_[p.iid] = done;
        kind_of_[p.iid] = dev;
        copy_info_[p.iid] = CopyInfo{p.src_aid, p.dst_aid, rbbox(p.region), p.region};
        // the launch wrote the receiver's flag: no stream write for it later
        signalled_.insert(p.iid * uint64_t(cfg_.world) + uint64_t(owner_rank(p.dst_mem - 2)));
        st_.bytes_copy[2] += rvolume(p.region) * 4;
    }
    if (grown_) {
        note_use(k);
        for (const Instr& p : pushes) note_use(p);
    }
    return true;
}

// Release the held-back kernel: fused with its pushes when expressible, else
// the ordinary path; then the horizons that waited with it.
void Executor::halo_flush() {
    if (!halo_parked_) return;
    halo_parked_ = false;
    Instr k = std::move(halo_kernel_);
    std::vector<Instr> pushes, deferred;
    pushes.swap(halo_pushes_);
    deferred.swap(halo_deferred_);
    halo_iids_.clear();
    halo_flushing_ = true;
    if (!halo_launch(k, pushes)) {
        on_instr_impl(k);
        for (const Instr& p : pushes) on_instr_impl(p);
    }
    for (const Instr& x : deferred) on_instr_impl(x);
    halo_flushing_ = false;
    cur_ins_ = nullptr;
}

}  // namespace cel
