// Executor: device-kernel instructions, shell / interior split for
// halo overlap, accessor bounds-check records (§4.4).
#include "exec_impl.hpp"

namespace cel {

// The launch arguments of a built-in kernel instruction: chunk, parameters and
// one accessor per access (allocation base and box, the range mapper's box).
void Executor::build_kargs(const Instr& ins, KArgs& a) {
    const TaskDesc& d = *ins.desc;
    memset(&a, 0, sizeof a);
    a.kind = d.kernel;
    a.n_acc = int(std::min<size_t>(d.acc.size(), kMaxAcc));
    for (int k = 0; k < 3; ++k) {
        a.chunk.lo[k] = ins.chunk.lo[k];
        a.chunk.hi[k] = ins.chunk.hi[k];
    }
    a.seed = d.params.seed;
    a.value = d.params.value;
    a.t = d.params.t;
    a.salt = d.params.salt;
    a.fast = cfg_.fast_math ? 1 : 0;
    a.variant = kernel_variant_;
    for (int i = 0; i < a.n_acc; ++i) {
        const Access& ac = d.acc[i];
        DAcc& A = a.acc[i];
        const Box ext = bufinfo_.at(ac.buf).extent;
        for (int k = 0; k < 3; ++k) A.ext[k] = ext.hi[k];
        A.es = bufinfo_.at(ac.buf).es;
        A.mode = ac.mode;
        A.map = int(ac.map.kind);
        for (int k = 0; k < 3; ++k) {
            A.border[k] = ac.map.border[k];
            A.fixed.lo[k] = ac.map.fixed.lo[k];
            A.fixed.hi[k] = ac.map.fixed.hi[k];
        }
        const Box mb = map_access(ac.map, ins.chunk, ext);
        for (int k = 0; k < 3; ++k) {
            A.box.lo[k] = mb.lo[k];
            A.box.hi[k] = mb.hi[k];
        }
        auto it = allocs_.find(ins.bindings[i]);
        if (it != allocs_.end()) {
            A.base = base_of(it->second);
            for (int k = 0; k < 3; ++k) {
                A.lo[k] = it->second.box.lo[k];
                A.n[k] = it->second.box.extent(k);
            }
        }
    }
}

void Executor::exec_kernel(const Instr& ins) {
    const TaskDesc& d = *ins.desc;
    const int dev = ins.device;
    const int sidx = dev * kStreamsPerDev + S_COMPUTE;
    set_dev(dev);
    Token deps;
    for (uint64_t j : ins.deps) merge(deps, dep_token(j));
    wait_token(sidx, deps);
    if (d.kernel == K_CALLBACK) {
        std::vector<cel_accessor> acc(d.acc.size());
        for (size_t i = 0; i < d.acc.size(); ++i) {
            const int64_t aid = ins.bindings[i];
            auto it = allocs_.find(aid);
            memset(&acc[i], 0, sizeof acc[i]);
            if (it == allocs_.end()) continue;
            acc[i].base = base_of(it->second);
            for (int k = 0; k < 3; ++k) {
                acc[i].alloc_box.min[k] = uint64_t(it->second.box.lo[k]);
                acc[i].alloc_box.max[k] = uint64_t(it->second.box.hi[k]);
            }
            acc[i].elem_size = it->second.es;
            const Box rg = map_access(d.acc[i].map, ins.chunk, bufinfo_.at(d.acc[i].buf).extent);
            for (int k = 0; k < 3; ++k) {
                acc[i].range.min[k] = uint64_t(rg.lo[k]);
                acc[i].range.max[k] = uint64_t(rg.hi[k]);
            }
        }
        const int n_chk = int(std::min<size_t>(acc.size(), kMaxAcc));
        if (cfg_.bounds_check && n_chk) {
            long long* rec = oob_begin(dev, sidx, n_chk);
            for (int i = 0; i < n_chk; ++i) acc[i].oob = rec + 6 * i;
        }
        cel_box ch;
        for (int k = 0; k < 3; ++k) {
            ch.min[k] = uint64_t(ins.chunk.lo[k]);
            ch.max[k] = uint64_t(ins.chunk.hi[k]);
        }
        if (d.fn) d.fn(d.fn_user, dev, &ch, acc.data(), int(acc.size()), streams_[sidx].s);
        if (cfg_.bounds_check && n_chk) oob_end(dev, sidx, ins, d, n_chk);
        tok_[ins.iid] = record(sidx);
        return;
    }
    KArgs a;
    build_kargs(ins, a);
    // Shell / interior split of stencil launches: the boundary bands that
    // neighbouring devices read (halo rows) are computed first on a
    // high-priority stream, so their coherence copies leave while the interior
    // is still running.  Same instruction, same result; only the launch order
    // and the per-part completion events change.
    Box interior = ins.chunk;
    bool split = false;
    if (split_ && (d.kernel == K_WAVE5 || d.kernel == K_JACOBI7 || d.kernel == K_STENCIL3)) {
        for (const Access& ac : d.acc) {
            if ((ac.map.kind != MapKind::Neighborhood && ac.map.kind != MapKind::NeighborhoodAxes) ||
                (ac.mode != MODE_READ && ac.mode != MODE_READ_WRITE))
                continue;
            const Box& ext = bufinfo_.at(ac.buf).extent;
            const Box rb = map_access(ac.map, ins.chunk, ext);
            // bands along the innermost dimension are widened to 16 bytes, so
            // the interior keeps the chunk's alignment (vectorised kernels)
            int inner = 2;
            while (inner > 0 && ext.extent(inner) <= 1) --inner;
            const int64_t es = int64_t(bufinfo_.at(ac.buf).es);
            for (int k = 0; k < 3; ++k) {
                int64_t bw = ac.map.border[k];
                if (k == inner && k > 0 && (es == 4 || es == 8)) bw = (bw + 16 / es - 1) / (16 / es) * (16 / es);
                if (rb.lo[k] < ins.chunk.lo[k]) {
                    interior.lo[k] = std::max(interior.lo[k], ins.chunk.lo[k] + bw);
                    split = true;
                }
                if (rb.hi[k] > ins.chunk.hi[k]) {
                    interior.hi[k] = std::min(interior.hi[k], ins.chunk.hi[k] - bw);
                    split = true;
                }
            }
        }
        // only worth it when the interior is big enough to hide the halo
        // chain (a launch costs a few microseconds; tiny chunks are latency-bound)
        if (interior.empty() || interior.volume() < (uint64_t(1) << 18)) split = false;
    }
    long long* oob = nullptr;
    if (cfg_.bounds_check && a.n_acc) {
        split = false;                            // one record per instruction, one launch stream
        oob = oob_begin(dev, sidx, a.n_acc);
        a.checked = 1;
        for (int i = 0; i < a.n_acc; ++i) a.acc[i].oob = oob + 6 * i;
    }
    auto launch = [&](const Box& ch, int stream, bool shell_part) {
        KArgs b = a;
        for (int k = 0; k < 3; ++k) {
            b.chunk.lo[k] = ch.lo[k];
            b.chunk.hi[k] = ch.hi[k];
        }
        for (int i = 0; i < b.n_acc; ++i) {
            const Box mb = map_access(d.acc[i].map, ch, bufinfo_.at(d.acc[i].buf).extent);
            for (int k = 0; k < 3; ++k) {
                b.acc[i].box.lo[k] = mb.lo[k];
                b.acc[i].box.hi[k] = mb.hi[k];
            }
        }
        int n;
        if (cfg_.profile && prof_sample(shell_part ? K_NUM + 2 : d.kernel)) {
            Prof p{shell_part ? K_NUM + 2 : d.kernel, prof_event(dev), prof_event(dev), dev, ins.iid, stream, now_ns()};
            cudaEventRecord(p.a, streams_[stream].s);
            n = launch_workload(b, streams_[stream].s);
            cudaEventRecord(p.b, streams_[stream].s);
            prof_pending_.push_back(p);
        } else {
            n = launch_workload(b, streams_[stream].s);
        }
        check(cudaGetLastError(), "kernel launch");
        st_.kernel_launches += n;
        st_.workload_launches += n;
    };
    if (!split) {
        launch(ins.chunk, sidx, false);
        if (oob) oob_end(dev, sidx, ins, d, a.n_acc);
        tok_[ins.iid] = record(sidx);
        return;
    }
    // shell launches: every dependency (they read the incoming halos), on the
    // high-priority halo stream.  (Measured and rejected in round 2: shells
    // ahead of the interior on the compute stream -- no cross-stream wait for
    // the interior, but it then waits for the halos: 6.9k vs 7.5k steps/s at
    // 4 B200, 3.97k vs 4.04k at 2.)
    const int hidx = dev * kStreamsPerDev + S_HALO;
    wait_token(hidx, deps);
    std::vector<Box> shell;
    subtract_into(ins.chunk, interior, shell);
    for (const Box& b : shell) launch(b, hidx, true);
    Token tshell = record(hidx);
    // interior launch: only dependencies whose accesses conflict with the
    // interior's (copies into halo rows it never reads are skipped)
    Token ideps;
    for (uint64_t j : ins.deps) {
        auto ci = copy_info_.find(j);
        bool conflict = true;
        if (ci != copy_info_.end()) {
            conflict = false;
            for (size_t i = 0; i < d.acc.size() && !conflict; ++i) {
                const Access& ac = d.acc[i];
                const int64_t aid = ins.bindings[i];
                const Box ib = map_access(ac.map, interior, bufinfo_.at(ac.buf).extent);
                auto hits = [&](const CopyInfo& c) {
                    if (intersect(c.bb, ib).empty()) return false;
                    for (const Box& b : c.region)
                        if (!intersect(b, ib).empty()) return true;
                    return false;
                };
                if (ci->second.dst_aid == aid && hits(ci->second)) conflict = true;             // RAW / WAW
                if (ci->second.src_aid == aid && (ac.mode & MODE_WRITE) && hits(ci->second)) conflict = true;  // WAR
            }
        }
        if (conflict) merge(ideps, dep_token(j));
    }
    wait_token(sidx, ideps);
    // the interior must also follow the shell launches' own predecessors on
    // the halo stream only through real conflicts, which `ideps` carries
    launch(interior, sidx, false);
    Token tint = record(sidx);
    Token all = tint;
    merge(all, tshell);
    tok_[ins.iid] = all;
    int64_t waid = 0;
    for (size_t i = 0; i < d.acc.size(); ++i)
        if (d.acc[i].mode & MODE_WRITE) waid = ins.bindings[i];
    parts_[ins.iid] = Parts{tshell, interior, waid, ins.bindings};
}

}  // namespace cel
