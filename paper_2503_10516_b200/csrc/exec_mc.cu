// Executor: the `all` gather over NVLink SHARP multicast (the
// all-gather of §8 a7, "RSim puts more pressure on the
// communication logic").
//
// One process owning G distinct GPUs with VMM allocations: the G allocations
// that receive a gather set (one per device, the same box) are bound to one
// multicast object.  Each source device runs one kernel that reads its chunk
// and stores it once to the multicast address; NVSwitch replicates the stores
// into every bound allocation, so a source sends its bytes over NVLink once
// instead of G - 1 times.  The kernel's last CTA adds 1 to a multicast flag
// (release, system scope); every device's stream waits until its own copy of
// the flag has counted all sources of the round (cuStreamWaitValue64 GEQ).
// The instruction graph is unchanged: the members of the set are the paper's
// G (G - 1) producer-split copies; only their execution differs.
#include "exec_impl.hpp"

namespace cel {

// multicast objects need every device added before memory is bound, memory
// created by cuMemCreate on those devices, and sizes in multicast granules
bool Executor::mc_setup() {
    if (mc_state_) return mc_state_ > 0;
    mc_state_ = -1;
    if (cfg_.world != 1 || !vmm_ || G_ < 2 || !g_drv.multicast() || !g_drv.wait64) return false;
    for (int a = 0; a < G_; ++a)
        for (int b = a + 1; b < G_; ++b)
            if (phys_[a] == phys_[b]) return false;
    for (int p : phys_) {
        int v = 0;
        if (g_drv.devattr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, CUdevice(p)) != CUDA_SUCCESS || !v) return false;
    }
    CUmulticastObjectProp mp;
    memset(&mp, 0, sizeof mp);
    mp.numDevices = unsigned(G_);
    mp.size = vmm_gran_;
    size_t gr = 0;
    if (g_drv.mc_granularity(&gr, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || gr == 0) return false;
    if (vmm_gran_ % gr) return false;
    mc_gran_ = gr;
    // the flag object: one granule per device, bound to one multicast object;
    // the kernels add to the multicast address, each stream waits on its
    // device's own granule
    mp.size = round_up(vmm_gran_, gr);
    if (g_drv.mc_create(&mc_flag_h_, &mp) != CUDA_SUCCESS) return false;
    bool ok = true;
    for (int d = 0; d < G_ && ok; ++d) ok = g_drv.mc_add_device(mc_flag_h_, CUdevice(phys_[d])) == CUDA_SUCCESS;
    mc_flag_dev_.assign(G_, nullptr);
    for (int d = 0; d < G_ && ok; ++d) {
        auto v = vmm_create(d, mp.size, mp.size);
        if (!v) {
            ok = false;
            break;
        }
        mc_flag_dev_[d] = v;
        ok = g_drv.mc_bind_mem(mc_flag_h_, 0, v->chunks[0].first, 0, mp.size, 0) == CUDA_SUCCESS;
        set_dev(d);
        ok = ok && cudaMemset(reinterpret_cast<void*>(v->va), 0, mp.size) == cudaSuccess;
    }
    if (ok) ok = mc_map(mc_flag_h_, mp.size, &mc_flag_va_);
    mc_ctr_.assign(G_, nullptr);
    for (int d = 0; d < G_ && ok; ++d) {
        set_dev(d);
        ok = cudaMalloc(&mc_ctr_[d], 64) == cudaSuccess && cudaMemset(mc_ctr_[d], 0, 64) == cudaSuccess;
    }
    for (int d = 0; d < G_; ++d) {
        set_dev(d);
        cudaDeviceSynchronize();
    }
    if (!ok) {
        cudaGetLastError();
        mc_teardown();
        return false;
    }
    mc_state_ = 1;
    return true;
}

bool Executor::mc_map(CUmemGenericAllocationHandle h, uint64_t size, CUdeviceptr* va) {
    if (g_drv.reserve(va, size, mc_gran_, 0, 0) != CUDA_SUCCESS) return false;
    if (g_drv.map(*va, size, 0, h, 0) != CUDA_SUCCESS) {
        g_drv.addr_free(*va, size);
        *va = 0;
        return false;
    }
    std::vector<CUmemAccessDesc> acc;
    for (int p : phys_) {
        CUmemAccessDesc d;
        d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        d.location.id = p;
        d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        acc.push_back(d);
    }
    if (g_drv.set_access(*va, size, acc.data(), acc.size()) != CUDA_SUCCESS) {
        g_drv.unmap(*va, size);
        g_drv.addr_free(*va, size);
        *va = 0;
        return false;
    }
    return true;
}

void Executor::mc_group_destroy(McGroup& g) {
    if (g.va) {
        g_drv.unmap(g.va, g.size);
        g_drv.addr_free(g.va, g.size);
    }
    if (g.h) {
        for (int d = 0; d < G_; ++d) g_drv.mc_unbind(g.h, CUdevice(phys_[d]), 0, g.size);
        g_drv.release(g.h);
    }
    g.va = 0;
    g.h = 0;
}

void Executor::mc_teardown() {
    for (auto& kv : mc_groups_) mc_group_destroy(kv.second);
    mc_groups_.clear();
    if (mc_flag_va_) {
        g_drv.unmap(mc_flag_va_, mc_gran_ ? round_up(vmm_gran_, mc_gran_) : vmm_gran_);
        g_drv.addr_free(mc_flag_va_, mc_gran_ ? round_up(vmm_gran_, mc_gran_) : vmm_gran_);
        mc_flag_va_ = 0;
    }
    if (mc_flag_h_) {
        const uint64_t size = round_up(vmm_gran_, mc_gran_ ? mc_gran_ : vmm_gran_);
        for (int d = 0; d < G_; ++d) g_drv.mc_unbind(mc_flag_h_, CUdevice(phys_[d]), 0, size);
        g_drv.release(mc_flag_h_);
        mc_flag_h_ = 0;
    }
    for (auto& v : mc_flag_dev_)
        if (v) vmm_release(*v);
    mc_flag_dev_.clear();
    for (int d = 0; d < int(mc_ctr_.size()); ++d)
        if (mc_ctr_[d]) {
            set_dev(d);
            cudaFree(mc_ctr_[d]);
        }
    mc_ctr_.clear();
}

// Groups whose bound memory is about to be unmapped (free) must go first.
void Executor::mc_forget(const VmmRegion* r) {
    for (auto it = mc_groups_.begin(); it != mc_groups_.end();) {
        bool hit = false;
        for (auto& p : it->second.regions) hit = hit || p.get() == r;
        if (hit) {
            mc_group_destroy(it->second);
            it = mc_groups_.erase(it);
        } else {
            ++it;
        }
    }
}

// Runs the set as multicast stores if its allocations qualify; false: not
// applicable (the caller takes the NCCL or push path), nothing issued.
bool Executor::exec_coll_mc(const std::vector<Instr>& m) {
    if (!mc_enabled_ || !mc_setup()) return false;
    const uint32_t es = bufinfo_.at(m[0].buffer).es;
    if (es % 4) return false;
    // the receiving allocation of every device, and the roots' boxes
    std::vector<int64_t> aid(G_, -1);
    std::map<int, std::vector<const Instr*>> roots;
    auto bind = [&](int v, int64_t a) {
        if (aid[v] != -1 && aid[v] != a) return false;
        aid[v] = a;
        return true;
    };
    for (const Instr& x : m) {
        if (x.region.size() != 1) return false;
        const int s = x.src_mem - 2, d = x.dst_mem - 2;
        if (s < 0 || d < 0 || !bind(s, x.src_aid) || !bind(d, x.dst_aid)) return false;
        roots[s].push_back(&x);
    }
    const AllocRec* first = nullptr;
    std::vector<std::shared_ptr<VmmRegion>> regs;
    for (int v = 0; v < G_; ++v) {
        if (aid[v] < 0) return false;
        const AllocRec& A = allocs_.at(aid[v]);
        if (!A.vmm || A.absorbed_into || A.vmm->mapped % mc_gran_) return false;
        if (first && (!(A.box == first->box) || A.vmm->mapped != first->vmm->mapped)) return false;
        if (!first) first = &A;
        regs.push_back(A.vmm);
    }
    for (auto& rt : roots) {
        const Box& b = rt.second[0]->region[0];
        for (const Instr* x : rt.second)
            if (!(x->region[0] == b)) return false;
        const uint64_t off = uint64_t(((b.lo[0] - first->box.lo[0]) * first->box.extent(1) + (b.lo[1] - first->box.lo[1])) *
                                          first->box.extent(2) +
                                      (b.lo[2] - first->box.lo[2])) *
                             es;
        if (off % 16) return false;           // 16-byte multicast stores from the chunk's start
    }
    // the multicast object of this set of allocations (bound once, reused by
    // every round; rebuilt if an allocation grew)
    McGroup* g = nullptr;
    auto it = mc_groups_.find(aid);
    if (it != mc_groups_.end() && it->second.size == first->vmm->mapped) g = &it->second;
    if (!g) {
        if (it != mc_groups_.end()) {                 // stale binding: nothing may use it any more
            sync_streams();
            mc_group_destroy(it->second);
            mc_groups_.erase(it);
        }
        McGroup ng;
        ng.size = first->vmm->mapped;
        ng.regions = regs;
        ng.slot = mc_next_slot_++;
        CUmulticastObjectProp mp;
        memset(&mp, 0, sizeof mp);
        mp.numDevices = unsigned(G_);
        mp.size = ng.size;
        bool ok = ng.slot * 8 < round_up(vmm_gran_, mc_gran_) && g_drv.mc_create(&ng.h, &mp) == CUDA_SUCCESS;
        for (int d = 0; d < G_ && ok; ++d) ok = g_drv.mc_add_device(ng.h, CUdevice(phys_[d])) == CUDA_SUCCESS;
        for (int d = 0; d < G_ && ok; ++d) {
            uint64_t o = 0;
            for (auto& c : regs[d]->chunks) {
                ok = ok && g_drv.mc_bind_mem(ng.h, o, c.first, 0, c.second, 0) == CUDA_SUCCESS;
                o += c.second;
            }
        }
        ok = ok && mc_map(ng.h, ng.size, &ng.va);
        if (!ok) {
            mc_group_destroy(ng);
            return false;
        }
        g = &(mc_groups_[aid] = ng);
    }
    g->expected += roots.size();
    const uint64_t slot_off = g->slot * 8;
    // sources: wait for every member's dependencies (the readers of the
    // previous contents on every receiving device), store, release the flag
    for (auto& rt : roots) {
        const int s = rt.first;
        const int sidx = s * kStreamsPerDev + S_PUSH;
        set_dev(s);
        Token t;
        for (const Instr* x : rt.second) {
            cur_ins_ = x;
            merge(t, local_part(x->deps));
        }
        wait_token(sidx, t);
        const Box& b = rt.second[0]->region[0];
        const uint64_t off = uint64_t(((b.lo[0] - first->box.lo[0]) * first->box.extent(1) + (b.lo[1] - first->box.lo[1])) *
                                          first->box.extent(2) +
                                      (b.lo[2] - first->box.lo[2])) *
                             es;
        const uint64_t bytes = b.volume() * es;
        const char* src = base_of(allocs_.at(aid[s])) + off;
        char* dst = reinterpret_cast<char*>(g->va) + off;
        auto* flag = reinterpret_cast<unsigned long long*>(mc_flag_va_ + slot_off);
        if (cfg_.profile && prof_sample(K_NUM + 3)) {
            Prof p{K_NUM + 3, prof_event(s), prof_event(s), s, m[0].iid, sidx, now_ns()};
            cudaEventRecord(p.a, streams_[sidx].s);
            st_.kernel_launches += launch_mc_gather(src, dst, bytes, flag, static_cast<unsigned*>(mc_ctr_[s]),
                                                    streams_[sidx].s);
            cudaEventRecord(p.b, streams_[sidx].s);
            prof_pending_.push_back(p);
        } else {
            st_.kernel_launches += launch_mc_gather(src, dst, bytes, flag, static_cast<unsigned*>(mc_ctr_[s]),
                                                    streams_[sidx].s);
        }
        check(cudaGetLastError(), "multicast gather launch");
        st_.bytes_copy[2] += bytes;
    }
    // receivers (every device): the round is complete on a device once its own
    // copy of the flag counts every source of every round so far
    std::vector<Token> tv(G_);
    for (int v = 0; v < G_; ++v) {
        const int sidx = v * kStreamsPerDev + S_PUSH;
        set_dev(v);
        checkd(g_drv.wait64(reinterpret_cast<CUstream>(streams_[sidx].s), mc_flag_dev_[v]->va + slot_off, g->expected,
                            CU_STREAM_WAIT_VALUE_GEQ),
               "cuStreamWaitValue64 (multicast flag)");
        tv[v] = record(sidx);
    }
    for (const Instr& x : m) {
        Token lt = tv[x.src_mem - 2];
        merge(lt, tv[x.dst_mem - 2]);
        tok_[x.iid] = lt;
    }
    st_.coll_groups++;
    st_.coll_copies += m.size();
    st_.coll_multicast++;
    return true;
}

void Executor::sync_streams() {
    for (auto& s : streams_)
        if (s.s) cudaStreamSynchronize(s.s);
}

}  // namespace cel
