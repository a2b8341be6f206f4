// Executor implementation (see exec.hpp).  Paper: §4.1 out-of-order dispatch
// (P:L515-530), allocation instructions, copy instructions
// (P:L292), epochs, horizons.
#include "exec_impl.hpp"

namespace cel {

// ------------------------------------------------------------ arena (allocation manager)
// Deterministic first-fit sub-allocator over one pre-reserved device range per
// device.  Every process of a multi-process run replays the same alloc/free
// sequence for every device, so it knows every allocation's address without
// communication; a freed range carries the completion token of its free
// instruction, and a new allocation that reuses it inherits that token.
bool Executor::Arena::alloc(uint64_t bytes, uint64_t* off, Token* tok) {
    bytes = round_up(std::max<uint64_t>(bytes, 1), kAlign);
    for (auto it = free_.begin(); it != free_.end(); ++it) {
        if (it->second.len < bytes) continue;
        *off = it->first;
        *tok = it->second.tok;
        FreeRange rest{it->second.len - bytes, it->second.tok};
        const uint64_t o = it->first;
        free_.erase(it);
        if (rest.len) free_[o + bytes] = rest;
        return true;
    }
    return false;
}

bool Executor::Arena::extend(uint64_t off, uint64_t old_bytes, uint64_t new_bytes, Token* tok) {
    const uint64_t a = off + round_up(std::max<uint64_t>(old_bytes, 1), kAlign);
    const uint64_t b = off + round_up(std::max<uint64_t>(new_bytes, 1), kAlign);
    if (b <= a) return true;
    auto it = free_.find(a);
    if (it == free_.end() || it->second.len < b - a) return false;
    *tok = it->second.tok;
    FreeRange rest{it->second.len - (b - a), it->second.tok};
    free_.erase(it);
    if (rest.len) free_[b] = rest;
    return true;
}

Token& Executor::Arena::release(uint64_t off, uint64_t bytes, Token tok) {
    bytes = round_up(std::max<uint64_t>(bytes, 1), kAlign);
    auto nx = free_.lower_bound(off);
    // coalesce with the successor
    if (nx != free_.end() && off + bytes == nx->first) {
        bytes += nx->second.len;
        for (auto& e : nx->second.tok.local) tok.local.push_back(e);
        for (auto& e : nx->second.tok.remote) tok.remote.push_back(e);
        nx = free_.erase(nx);
    }
    // coalesce with the predecessor
    if (nx != free_.begin()) {
        auto pv = std::prev(nx);
        if (pv->first + pv->second.len == off) {
            pv->second.len += bytes;
            for (auto& e : tok.local) pv->second.tok.local.push_back(e);
            for (auto& e : tok.remote) pv->second.tok.remote.push_back(e);
            return pv->second.tok;
        }
    }
    FreeRange& fr = free_[off];
    fr = FreeRange{bytes, std::move(tok)};
    return fr.tok;
}

// ------------------------------------------------------------ VMM allocations
// SURVEY NEXT-3, P:L549-556 ("allocations are very slow ... resizing"): in a
// single process every allocation of at least one granule gets its own
// reserved virtual address range, sized for growth to the buffer's end along
// dim 0, with physical memory mapped as needed.  A resize that keeps the
// rows as a prefix (R9 growth at the end of dim 0) maps more granules behind
// the old ones: no copy, no matter what else was allocated since (the arena
// form of growth needs the range right after the allocation to be free).
std::shared_ptr<Executor::VmmRegion> Executor::vmm_create(int dev, uint64_t bytes, uint64_t reserve) {
    auto v = std::make_shared<VmmRegion>();
    v->dev = dev;
    v->reserved = round_up(std::max(reserve, bytes), vmm_gran_);
    if (g_drv.reserve(&v->va, v->reserved, vmm_gran_, 0, 0) != CUDA_SUCCESS) {
        v->reserved = round_up(bytes, vmm_gran_);             // no room to grow: reserve what is needed now
        if (g_drv.reserve(&v->va, v->reserved, vmm_gran_, 0, 0) != CUDA_SUCCESS) return nullptr;
    }
    if (!vmm_map_more(*v, bytes)) {
        vmm_release(*v);
        return nullptr;
    }
    return v;
}

bool Executor::vmm_map_more(VmmRegion& v, uint64_t bytes) {
    const uint64_t want = round_up(bytes, vmm_gran_);
    if (want <= v.mapped) return true;
    if (want > v.reserved) return false;
    const uint64_t add = want - v.mapped;
    CUmemAllocationProp prop;
    memset(&prop, 0, sizeof prop);
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = phys_[v.dev];
    CUmemGenericAllocationHandle h;
    if (g_drv.create(&h, add, &prop, 0) != CUDA_SUCCESS) return false;
    if (g_drv.map(v.va + v.mapped, add, 0, h, 0) != CUDA_SUCCESS) {
        g_drv.release(h);
        return false;
    }
    // every GPU of this process may read or push into it (peer access by mapping)
    std::vector<CUmemAccessDesc> acc;
    for (int p : cfg_.all_devices.empty() ? phys_ : cfg_.all_devices) {
        bool seen = false;
        for (auto& a : acc) seen = seen || a.location.id == p;
        if (seen) continue;
        CUmemAccessDesc d;
        d.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        d.location.id = p;
        d.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        acc.push_back(d);
    }
    if (g_drv.set_access(v.va + v.mapped, add, acc.data(), acc.size()) != CUDA_SUCCESS) {
        g_drv.unmap(v.va + v.mapped, add);
        g_drv.release(h);
        return false;
    }
    v.chunks.push_back({h, add});
    v.mapped = want;
    st_.vmm_mapped_bytes += add;
    st_.vmm_maps++;
    return true;
}

void Executor::vmm_release(VmmRegion& v) {
    if (!mc_groups_.empty()) mc_forget(&v);     // unbind multicast objects before the memory goes
    uint64_t o = 0;
    for (auto& c : v.chunks) {
        g_drv.unmap(v.va + o, c.second);
        g_drv.release(c.first);
        o += c.second;
    }
    v.chunks.clear();
    if (v.va) g_drv.addr_free(v.va, v.reserved);
    v.va = 0;
    v.mapped = 0;
}

// Unmap freed VMM allocations whose free instruction has completed (all: the
// device is idle, e.g. at destruction).
void Executor::vmm_reap(bool all) {
    for (auto it = vmm_free_.begin(); it != vmm_free_.end();) {
        bool done = all;
        if (!done) {
            done = true;
            for (const TokEntry& e : it->second.local) done = done && e.seq <= streams_[e.stream].done;
        }
        if (done) {
            vmm_release(*it->first);
            it = vmm_free_.erase(it);
        } else {
            ++it;
        }
    }
}

// ------------------------------------------------------------ setup
Executor::Executor(const ExecConfig& cfg, Scheduler* sched) : cfg_(cfg), sched_(sched) {
    G_ = int(cfg_.cuda_devices.size());
    const char* tr = getenv("CEL_TRACE");
    trace_ = tr && tr[0] == '1';
    // small contiguous pushes to another GPU go to a copy engine: a 64 KiB halo
    // push as an SM kernel took SM time from the running stencil (kernel share
    // 0.940 -> 0.986 of the step at 4 GPUs with DMA); CEL_PEER_DMA=0 for A/B
    const char* pd = getenv("CEL_PEER_DMA");
    peer_dma_ = !(pd && pd[0] == '0');
    const char* jv = getenv("CEL_JACOBI");
    if (jv && jv[0] == 'l') kernel_variant_ |= kVarJacobiLsu;
    const char* rv = getenv("CEL_RSIM");
    if (rv && rv[0] == '0') kernel_variant_ |= kVarRsimRegs;
    const char* ds = getenv("CEL_DIRECT_SENDS");
    direct_sends_ = cfg_.comm && !(ds && ds[0] == '0');
    const char* cmb = getenv("CEL_COLL_MIN_BYTES");
    if (cmb && cmb[0]) coll_min_bytes_ = strtoull(cmb, nullptr, 10);
    const char* cv = getenv("CEL_COPY");
    tma_copy_ = cv && cv[0] == 't';
    const char* fp = getenv("CEL_FORCE_PEER");
    force_peer_ = fp && fp[0] == '1';
    const char* ns = getenv("CEL_NO_SPLIT");
    split_ = !(ns && ns[0] == '1');
    const char* ng = getenv("CEL_NO_GROW");
    no_grow_ = ng && ng[0] == '1';
    const char* ra = getenv("CEL_ROW_ALIGN");
    if (ra && atoi(ra) >= 16 && (atoi(ra) & (atoi(ra) - 1)) == 0) row_align_ = uint32_t(atoi(ra));
    const char* np = getenv("CEL_NO_PAD");
    no_pad_ = np && np[0] == '1';
    grown_ = !no_grow_;
}

Executor::~Executor() {
    if (threaded_) {
        drain();
        {
            std::lock_guard<std::mutex> l(qm_);
            stop_ = true;
        }
        qcv_.notify_one();
        thr_.join();
        threaded_ = false;
    }
    if (err_ == 0) sync_all();
    else
        for (auto& s : streams_)
            if (s.s) cudaStreamSynchronize(s.s);
    mc_teardown();
    vmm_reap(true);
    for (auto& kv : allocs_)
        if (kv.second.vmm && !kv.second.absorbed_into && kv.second.vmm->va) vmm_release(*kv.second.vmm);
    for (auto& p : prof_pending_) {
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    for (auto& pool : prof_pool_)
        for (cudaEvent_t e : pool) cudaEventDestroy(e);
    for (void* c : comms_)
        if (c) g_nccl.destroy(static_cast<ncclComm_t>(c));
    comms_.clear();
    for (int d = 0; d < int(arenas_.size()); ++d) {
        if (!owned(d)) {
            if (cfg_.world > 1 && arenas_[d].base) cudaIpcCloseMemHandle(arenas_[d].base);
            continue;
        }
        set_dev(d);
        for (int k = 0; k < kStreamsPerDev; ++k) {
            Stream& s = streams_[d * kStreamsPerDev + k];
            for (auto& p : s.inflight) cudaEventDestroy(p.second);
            if (s.s) cudaStreamDestroy(s.s);
        }
        for (cudaEvent_t e : pool_[d]) cudaEventDestroy(e);
        // one cudaMalloc per physical device+virtual device
        if (arenas_[d].base) cudaFree(arenas_[d].base);
    }
    for (auto& kv : host_init_)
        if (kv.second.second) cudaFreeHost(kv.second.first);
    if (host_arena_.base) cudaFreeHost(host_arena_.base);
    for (auto& r : oob_pending_) cudaEventDestroy(r.ev);
    for (long long* p : oob_dev_)
        if (p) cudaFree(p);
    for (long long* p : oob_host_)
        if (p) cudaFreeHost(p);
}

void Executor::set_dev(int dev) { cudaSetDevice(phys_[dev]); }

Box Executor::padded_box(const Box& b, uint32_t buffer, uint32_t es) const {
    if (no_pad_ || (es != 4 && es != 8) || b.empty()) return b;
    const Box& ext = bufinfo_.at(buffer).extent;
    int d = 2;                                   // innermost dimension the buffer uses
    while (d > 0 && ext.hi[d] - ext.lo[d] <= 1) --d;
    if (d == 0) return b;                        // 1-D: whole rows are contiguous already
    const int64_t a = int64_t(row_align_) / int64_t(es);
    Box p = b;
    p.lo[d] = b.lo[d] - (b.lo[d] % a);           // coordinates are >= 0
    p.hi[d] = p.lo[d] + (b.hi[d] - p.lo[d] + a - 1) / a * a;
    return p;
}

void Executor::check(cudaError_t e, const char* what) {
    if (e == cudaSuccess || err_) return;
    errmsg_ = std::string(what) + ": " + cudaGetErrorString(e);
    err_ = E_CUDA;
    if (cfg_.comm) cfg_.comm->abort();
}

void Executor::checkd(CUresult e, const char* what) {
    if (e == CUDA_SUCCESS || err_) return;
    const char* s = nullptr;
    if (g_drv.errstr) g_drv.errstr(e, &s);
    errmsg_ = std::string(what) + ": " + (s ? s : "driver error");
    err_ = E_CUDA;
}

int Executor::init(std::string* err) {
    phys_ = cfg_.cuda_devices;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        *err = "no CUDA device visible (the coherence path has no CPU fallback)";
        return E_CUDA;
    }
    for (int p : phys_)
        if (p < 0 || p >= ndev) {
            *err = "cuda_devices names a device that does not exist";
            return E_INVALID;
        }
    if (cfg_.world > 1 && cfg_.world != G_) {
        *err = "multi-process mode needs n_devices == world (one device per rank)";
        return E_INVALID;
    }
    streams_.resize(size_t(G_) * kStreamsPerDev);
    pool_.resize(G_);
    prof_pool_.resize(G_);
    arenas_.resize(G_);
    uint64_t arena = cfg_.arena_bytes ? cfg_.arena_bytes : (16ull << 30);
    const uint64_t sig_bytes = cfg_.world > 1 ? uint64_t(cfg_.world) * kRing * 8 : 0;
    gather_off_ = round_up(sig_bytes, 4096);                  // then 4 KiB of gather counters
    const uint64_t data_off = round_up(gather_off_ + 4096, 2u << 20);
    gather_exp_.assign(G_, 0);
    // peer access between distinct physical devices (NVLink 5 / NVSwitch);
    // virtual-node mode: with every GPU of the process (device-direct sends
    // are pulled from another node's device memory)
    const std::vector<int>& peers = cfg_.all_devices.empty() ? phys_ : cfg_.all_devices;
    for (int a = 0; a < G_; ++a) {
        if (!owned(a)) continue;
        for (int pb : peers) {
            if (phys_[a] == pb) continue;
            int can = 0;
            cudaDeviceCanAccessPeer(&can, phys_[a], pb);
            if (can) {
                cudaSetDevice(phys_[a]);
                cudaError_t e = cudaDeviceEnablePeerAccess(pb, 0);
                if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            }
        }
    }
    for (int d = 0; d < G_; ++d) {
        Arena& A = arenas_[d];
        A.size = arena;
        A.data_off = data_off;
        A.free_[data_off] = FreeRange{arena - data_off, Token{}};
        if (!owned(d)) continue;
        set_dev(d);
        // copies, pushes and signals get the highest priority: their CTAs are
        // scheduled ahead of queued stencil CTAs, so a halo push never waits
        // for the next step's kernel to drain (P:L490 overlap of copies and kernels)
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        for (int k = 0; k < kStreamsPerDev; ++k) {
            Stream& s = streams_[d * kStreamsPerDev + k];
            s.dev = d;
            const int prio = k == S_COMPUTE ? prio_lo : prio_hi;
            if (cudaStreamCreateWithPriority(&s.s, cudaStreamNonBlocking, prio) != cudaSuccess) {
                *err = "cudaStreamCreate failed";
                return E_CUDA;
            }
        }
        cudaError_t e = cudaMalloc(&A.base, arena);
        if (e != cudaSuccess) {
            cudaGetLastError();
            char buf[200];
            snprintf(buf, sizeof buf, "cannot reserve a %.1f GiB arena on device %d (set arena_bytes)",
                     double(arena) / double(1ull << 30), phys_[d]);
            *err = buf;
            return E_OOM;
        }
        cudaMemset(A.base, 0, gather_off_ + 4096);         // flags and gather counters start at 0
    }
    if (cfg_.world > 1) {
        int v = 0;
        g_drv.load();
        if (g_drv.devattr)
            g_drv.devattr(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, CUdevice(phys_[cfg_.rank]));
        memops64_ = v != 0 && g_drv.wait64 && g_drv.write64;
        if (!memops64_) {
            *err = "multi-process mode needs 64-bit stream memory operations";
            return E_CUDA;
        }
    }
    // VMM allocations: one process owning all devices (multi-process runs
    // replay one deterministic arena layout instead, so every rank knows every
    // address without exchanging memory handles)
    const char* nv = getenv("CEL_NO_VMM");
    if (cfg_.world == 1 && !(nv && nv[0] == '1')) {
        g_drv.load();
        int sup = 1;
        for (int p : phys_) {
            int v = 0;
            if (!g_drv.devattr || g_drv.devattr(&v, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, CUdevice(p)) !=
                                      CUDA_SUCCESS)
                v = 0;
            sup = sup && v;
        }
        if (sup && g_drv.vmm()) {
            CUmemAllocationProp prop;
            memset(&prop, 0, sizeof prop);
            prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
            prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
            prop.location.id = phys_[0];
            size_t gr = 0;
            if (g_drv.granularity(&gr, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM) == CUDA_SUCCESS && gr > 0) {
                vmm_gran_ = gr;
                vmm_ = true;
            }
        }
    }
    if (cfg_.collective && G_ >= 2) {
        // one NCCL rank per GPU: the virtual devices must be distinct GPUs
        bool distinct = true;
        for (int a = 0; a < G_; ++a)
            for (int b = a + 1; b < G_; ++b)
                if (phys_[a] == phys_[b]) distinct = false;
        const char* cv = getenv("CEL_COLL");
        if (cv && cv[0] == '0') distinct = false;
        coll_ = distinct && g_nccl.load();
        // NVLS multicast gathers: one process, distinct GPUs, VMM allocations
        // P2P gather kernels: on by default in one process, and across
        // processes when every rank has a GPU of its own (two ranks folded onto
        // one GPU hung with them in the round-2 suite -- cross-process waits on
        // one GPU, which the profiling guide warns about; they keep pushes)
        const char* p2 = getenv("CEL_COLL_P2P");
        p2p_gather_ = p2 ? p2[0] == '1' : (cfg_.world == 1 || distinct);
        if (p2p_gather_) {                                    // receivers wait with 64-bit stream memory ops
            g_drv.load();
            int v = 0;
            if (g_drv.devattr)
                g_drv.devattr(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, CUdevice(phys_[owned(0) ? 0 : cfg_.rank]));
            p2p_gather_ = v != 0 && g_drv.wait64;
        }
        const char* fr = getenv("CEL_FUSE_ROWS");
        // (one process: the held-back kernel's flags to other ranks deadlocked
        // the 4-rank parity run, so multi-process runs do not fuse)
        fuse_rows_ = p2p_gather_ && cfg_.world == 1 && !(fr && fr[0] == '0');
        const char* mc = getenv("CEL_COLL_MC");
        mc_enabled_ = distinct && vmm_ && cfg_.world == 1 && mc && mc[0] == '1';
        if (coll_ && cfg_.world > 1 && cfg_.rank == 0) {
            ncclUniqueId id;
            if (g_nccl.get_id(&id) != ncclSuccess) {
                coll_ = false;
            } else {
                memcpy(nccl_id_, &id, sizeof id);
                nccl_id_set_ = true;
            }
        }
    }
    if (cfg_.bounds_check) {
        oob_dev_.assign(G_, nullptr);
        oob_host_.assign(G_, nullptr);
        oob_next_.assign(G_, 0);
        for (int d = 0; d < G_; ++d) {
            if (!owned(d)) continue;
            set_dev(d);
            const size_t bytes = size_t(kOobSlots) * kMaxAcc * 6 * sizeof(long long);
            void* h = nullptr;
            if (cudaMalloc(&oob_dev_[d], bytes) != cudaSuccess || cudaHostAlloc(&h, bytes, cudaHostAllocPortable) != cudaSuccess) {
                cudaGetLastError();
                *err = "cannot allocate bounds-check records";
                return E_OOM;
            }
            oob_host_[d] = static_cast<long long*>(h);
        }
    }
    if (cfg_.comm) {
        // virtual-node mode: M1 staging arena (pinned, mapped: copy kernels and
        // the communicator's pulls address it directly)
        void* h = nullptr;
        if (cudaHostAlloc(&h, cfg_.host_arena_bytes, cudaHostAllocPortable | cudaHostAllocMapped) != cudaSuccess) {
            cudaGetLastError();
            *err = "cannot allocate the M1 staging arena";
            return E_OOM;
        }
        host_arena_.base = static_cast<char*>(h);
        host_arena_.size = cfg_.host_arena_bytes;
        host_arena_.free_[0] = FreeRange{cfg_.host_arena_bytes, Token{}};
    }
    {
        int mp = 0;
        if (cudaDeviceGetAttribute(&mp, cudaDevAttrMaxPitch, phys_[0]) == cudaSuccess && mp > 0) max_pitch_ = size_t(mp);
        cudaGetLastError();
    }
    cudaDeviceSynchronize();
    const char* et = getenv("CEL_EXEC_THREAD");
    if (!(cfg_.comm || !(et && et[0] == '0'))) fuse_rows_ = false;   // parking needs the executor thread's drains
    {
        // halo pushes fused into the stencil (exec_halo.cu; default on,
        // CEL_FUSE_HALO=0 off): one process per GPU, every GPU distinct
        // (in-kernel waits across processes sharing a GPU are unsafe), the
        // executor thread (a drain releases held-back work).  4 B200: 7655-7689
        // vs 7505-7512 steps/s; 2: 4007-4020 vs 4021-4029; 3: 5849 vs 5809
        bool distinct = true;
        for (int a = 0; a < G_; ++a)
            for (int b = a + 1; b < G_; ++b)
                if (phys_[a] == phys_[b]) distinct = false;
        const char* fh = getenv("CEL_FUSE_HALO");
        fuse_halo_ = cfg_.world > 1 && G_ >= 2 && distinct && !cfg_.comm && !(et && et[0] == '0') && !(fh && fh[0] == '0');
    }
    if (cfg_.comm || !(et && et[0] == '0')) {   // nodes must progress independently
        threaded_ = true;
        thr_ = std::thread([this] { thread_main(); });
    }
    return err_.load();
}

// blob = arena IPC handle | flag byte | NCCL unique id (rank 0's is used)
static_assert(sizeof(cudaIpcMemHandle_t) == 64 && sizeof(ncclUniqueId) == 128, "IPC blob layout");
size_t Executor::ipc_blob_size() const { return kBlobBytes; }

int Executor::ipc_export(void* blob) const {
    if (cfg_.world <= 1) return E_STATE;
    cudaIpcMemHandle_t h;
    cudaSetDevice(phys_[cfg_.rank]);
    if (cudaIpcGetMemHandle(&h, arenas_[cfg_.rank].base) != cudaSuccess) return E_CUDA;
    char* b = static_cast<char*>(blob);
    memcpy(b, &h, sizeof h);
    b[sizeof h] = nccl_id_set_ ? 1 : 0;
    memcpy(b + sizeof h + 1, nccl_id_, sizeof(nccl_id_));
    return E_OK;
}

int Executor::ipc_import(int rank, const void* blob) {
    if (cfg_.world <= 1 || rank < 0 || rank >= G_) return E_INVALID;
    drain();
    if (rank == cfg_.rank) return E_OK;
    cudaIpcMemHandle_t h;
    memcpy(&h, blob, sizeof h);
    if (rank == 0) {
        const char* b = static_cast<const char*>(blob);
        if (b[sizeof h]) {
            memcpy(nccl_id_, b + sizeof h + 1, sizeof(nccl_id_));
            nccl_id_set_ = true;
        } else {
            coll_ = false;          // rank 0 runs without the collective: so must everyone
        }
    }
    void* p = nullptr;
    set_dev(cfg_.rank);
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        check(e, "cudaIpcOpenMemHandle");
        return E_CUDA;
    }
    arenas_[rank].base = static_cast<char*>(p);
    return E_OK;
}

int Executor::set_host_init(uint32_t bid, const void* data, size_t bytes, bool borrow) {
    char* p = const_cast<char*>(static_cast<const char*>(data));
    size_t owned_bytes = 0;
    if (!borrow) {
        void* q = nullptr;
        if (cudaHostAlloc(&q, bytes, cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            return E_OOM;
        }
        memcpy(q, data, bytes);
        p = static_cast<char*>(q);
        owned_bytes = bytes;
    }
    post([this, bid, p, owned_bytes] { host_init_[bid] = {p, owned_bytes}; });
    return E_OK;
}

void Executor::drop_host_init(uint32_t bid) {
    drain();
    auto it = host_init_.find(bid);
    if (it == host_init_.end()) return;
    sync_all();
    if (it->second.second) cudaFreeHost(it->second.first);
    host_init_.erase(it);
}

void Executor::set_readback(int64_t rb, void* dst, const Box& box, uint32_t es) {
    post([this, rb, dst, box, es] { readbacks_[rb] = Readback{static_cast<char*>(dst), box, es}; });
}

// ------------------------------------------------------------ events / tokens
cudaEvent_t Executor::get_event(int dev) {
    auto& p = pool_[dev];
    if (!p.empty()) {
        cudaEvent_t e = p.back();
        p.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    return e;
}

void Executor::put_event(int dev, cudaEvent_t e) { pool_[dev].push_back(e); }

void Executor::poll(bool prune) {
    for (auto& s : streams_) {
        while (!s.inflight.empty()) {
            cudaError_t q = cudaEventQuery(s.inflight.front().second);
            if (q == cudaErrorNotReady) break;
            if (q != cudaSuccess) {
                check(q, "asynchronous CUDA error");
                return;
            }
            s.done = s.inflight.front().first;
            put_event(s.dev, s.inflight.front().second);
            s.inflight.pop_front();
        }
    }
    (void)prune;
    if (!vmm_free_.empty()) vmm_reap(false);
    if (!oob_pending_.empty()) oob_check(false);
}

// §4.4 accessor bounds checking: claim the next record slot of `dev` and reset it
long long* Executor::oob_begin(int dev, int sidx, int n_acc) {
    // the ring slot must have been inspected: wait for its launch if still pending
    while (!oob_pending_.empty() && int(oob_pending_.size()) >= kOobSlots) {
        check(cudaEventSynchronize(oob_pending_.front().ev), "bounds-check wait");
        oob_check(false);
    }
    const int slot = oob_next_[dev];
    long long* rec = oob_dev_[dev] + size_t(slot) * kMaxAcc * 6;
    launch_oob_init(rec, n_acc, streams_[sidx].s);
    return rec;
}

void Executor::oob_end(int dev, int sidx, const Instr& ins, const TaskDesc& d, int n_acc) {
    const int slot = oob_next_[dev];
    oob_next_[dev] = (slot + 1) % kOobSlots;
    const size_t off = size_t(slot) * kMaxAcc * 6;
    check(cudaMemcpyAsync(oob_host_[dev] + off, oob_dev_[dev] + off, size_t(n_acc) * 6 * sizeof(long long),
                          cudaMemcpyDeviceToHost, streams_[sidx].s),
          "bounds-check record copy");
    OobRec r;
    r.dev = dev;
    r.slot = slot;
    check(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming), "cudaEventCreate");
    check(cudaEventRecord(r.ev, streams_[sidx].s), "cudaEventRecord");
    r.iid = ins.iid;
    r.task = ins.task;
    r.n_acc = n_acc;
    for (int i = 0; i < n_acc; ++i) {
        r.buf[i] = d.acc[i].buf;
        r.range[i] = map_access(d.acc[i].map, ins.chunk, bufinfo_.at(d.acc[i].buf).extent);
    }
    oob_pending_.push_back(r);
}

// Inspect the records of exited kernels ("report their bounding box in a
// runtime error message after the kernel exits").
void Executor::oob_check(bool wait) {
    while (!oob_pending_.empty()) {
        OobRec& r = oob_pending_.front();
        if (wait) {
            check(cudaEventSynchronize(r.ev), "bounds-check wait");
        } else {
            const cudaError_t q = cudaEventQuery(r.ev);
            if (q == cudaErrorNotReady) return;
        }
        const long long* h = oob_host_[r.dev] + size_t(r.slot) * kMaxAcc * 6;
        for (int i = 0; i < r.n_acc && !err_; ++i) {
            const long long* b = h + 6 * i;
            if (b[0] > b[3] - 1) continue;            // nothing recorded
            char msg[400];
            const Box& g = r.range[i];
            snprintf(msg, sizeof msg,
                     "accessor out of bounds: task %lld, device %d, accessor %d (buffer %u) accessed "
                     "[[%lld,%lld,%lld],[%lld,%lld,%lld]] outside its range-mapper region "
                     "[[%lld,%lld,%lld],[%lld,%lld,%lld]]",
                     (long long)r.task, r.dev, i, r.buf[i], b[0], b[1], b[2], b[3], b[4], b[5], (long long)g.lo[0],
                     (long long)g.lo[1], (long long)g.lo[2], (long long)g.hi[0], (long long)g.hi[1],
                     (long long)g.hi[2]);
            errmsg_ = msg;
            err_ = E_OUT_OF_BOUNDS;
        }
        cudaEventDestroy(r.ev);
        oob_pending_.pop_front();
    }
}

Token Executor::dep_token(uint64_t j) const {
    auto it = tok_.find(j);
    if (it != tok_.end()) return it->second;
    // copies and kernels another rank executes are not stored: their token is
    // the owner's flag (signalled to us through signal_deps on its side)
    if (cfg_.world > 1 && j >= prune_floor_) {
        int o = 0;
        if (owner_lookup(j, &o) && o >= 0 && owner_rank(o) != cfg_.rank) return Token{{}, {{owner_rank(o), j}}};
    }
    return Token{};
}

// Owner device of instruction j: recorded when this executor processed it, else
// (the scheduler's rank filter never handed it over) as the scheduler attached
// it to the instruction being processed (Instr::dep_owner).  The executor
// thread never reads the scheduler's own ring, which the API thread keeps
// overwriting while it runs ahead.
bool Executor::owner_lookup(uint64_t j, int* o) const {
    auto k = kind_of_.find(j);
    if (k != kind_of_.end()) {
        *o = k->second;
        return true;
    }
    const Instr* c = cur_ins_;
    if (!c || c->dep_owner.size() != c->deps.size()) return false;
    auto it = std::lower_bound(c->deps.begin(), c->deps.end(), j);
    if (it == c->deps.end() || *it != j) return false;
    const int v = c->dep_owner[size_t(it - c->deps.begin())];
    if (v == -2) return false;
    *o = v;
    return true;
}

// A dependency of the instruction being processed whose owner nobody knows
// although it may still be running: its completion would be dropped silently
// (ADVICE r1), so this is a state error instead.
void Executor::check_owner_known(const Instr& ins) {
    if (cfg_.world <= 1) return;
    for (uint64_t j : ins.deps) {
        int o = 0;
        if (j >= prune_floor_ && !tok_.count(j) && !owner_lookup(j, &o)) {
            char buf[160];
            snprintf(buf, sizeof buf, "instruction %llu: owner of dependency %llu unknown (scheduler ran too far ahead)",
                     (unsigned long long)ins.iid, (unsigned long long)j);
            errmsg_ = buf;
            err_ = E_STATE;
            return;
        }
    }
}

void Executor::merge(Token& into, const Token& t) const {
    for (const TokEntry& e : t.local) {
        if (e.seq <= streams_[e.stream].done) continue;
        bool found = false;
        for (TokEntry& x : into.local)
            if (x.stream == e.stream) {
                if (e.seq > x.seq) x = e;
                found = true;
                break;
            }
        if (!found) into.local.push_back(e);
    }
    for (auto& r : t.remote)
        if (std::find(into.remote.begin(), into.remote.end(), r) == into.remote.end()) into.remote.push_back(r);
}

uint64_t* Executor::sig_slot(int dev, int from_rank, uint64_t iid) {
    return reinterpret_cast<uint64_t*>(arenas_[dev].base) + (uint64_t(from_rank) * kRing + (iid % kRing));
}

void Executor::wait_token(int sidx, const Token& t) {
    Stream& s = streams_[sidx];
    for (const TokEntry& e : t.local) {
        if (e.stream == sidx || e.seq <= streams_[e.stream].done) continue;
        check(cudaStreamWaitEvent(s.s, e.ev, 0), "cudaStreamWaitEvent");
        st_.event_waits++;
        s.waits++;
    }
    for (auto& r : t.remote) {
        // a flag this stream already waited for is satisfied for everything
        // queued after it on the stream (FIFO): skip the repeat (e.g. the
        // lifetime dependency of every halo push on the peer's allocation)
        const uint64_t key = (uint64_t(r.first) << 56) ^ r.second;
        if (s.waited_remote.size() > (1u << 16)) s.waited_remote.clear();   // redundant waits are harmless
        if (!s.waited_remote.insert(key).second) continue;
        if (trace_)
            fprintf(stderr, "[cel r%d] stream %d waits for iid %llu from rank %d\n", cfg_.rank, sidx,
                    (unsigned long long)r.second, r.first);
        // the producer's process writes iid into this GPU's slot when done
        const uint64_t tw = now_ns();
        checkd(g_drv.wait64(reinterpret_cast<CUstream>(s.s),
                                   reinterpret_cast<CUdeviceptr>(sig_slot(s.dev, r.first, r.second)), r.second,
                                   CU_STREAM_WAIT_VALUE_GEQ),
               "cuStreamWaitValue64");
        st_.remote_wait_ns += now_ns() - tw;
        st_.remote_waits++;
        s.waits++;
    }
}

Token Executor::record(int sidx) {
    Stream& s = streams_[sidx];
    cudaEvent_t e = get_event(s.dev);
    check(cudaEventRecord(e, s.s), "cudaEventRecord");
    const uint64_t seq = ++s.seq;
    s.inflight.push_back({seq, e});
    Token t;
    t.local.push_back({sidx, seq, e});
    return t;
}

Token Executor::materialize(int dev, const Token& t) {
    const int sidx = dev * kStreamsPerDev + S_SYNC;
    wait_token(sidx, t);
    return record(sidx);
}

void Executor::throttle() {
    // virtual-node mode: never block here -- the oldest event may wait for a
    // pull another node's executor thread issues only after this thread has
    // posted a send further down its queue
    if (cfg_.comm) return;
    for (auto& s : streams_) {
        while (s.inflight.size() > 2048) {
            check(cudaEventSynchronize(s.inflight.front().second), "cudaEventSynchronize");
            st_.host_syncs++;
            s.done = s.inflight.front().first;
            put_event(s.dev, s.inflight.front().second);
            s.inflight.pop_front();
        }
    }
}

void Executor::sync_all() {
    drain();
    for (auto& s : streams_)
        if (s.s) cudaStreamSynchronize(s.s);
    poll(true);
}

// record which local work touched each allocation (in-place growth must
// order the grown allocation's users after it)
void Executor::note_use(const Instr& ins) {
    auto tit = tok_.find(ins.iid);
    if (tit == tok_.end() || tit->second.local.empty()) return;
    const Token loc{tit->second.local, {}};
    auto add = [&](int64_t aid) {
        auto a = allocs_.find(aid);
        if (a != allocs_.end()) merge(a->second.use, loc);
    };
    if (ins.kind == IKind::Copy) {
        add(ins.src_aid);
        add(ins.dst_aid);
    } else if (ins.kind == IKind::Kernel) {
        for (int64_t aid : ins.bindings) add(aid);
    }
}

void Executor::prune_tokens(uint64_t below) {
    prune_floor_ = below;
    for (auto it = tok_.begin(); it != tok_.end();) {
        if (it->first < below && !live_alloc_iid_.count(it->first))
            it = tok_.erase(it);
        else
            ++it;
    }
    for (auto it = ltok_.begin(); it != ltok_.end();) {
        if (it->first < below)
            it = ltok_.erase(it);
        else
            ++it;
    }
    for (auto it = copy_info_.begin(); it != copy_info_.end();) {
        if (it->first < below)
            it = copy_info_.erase(it);
        else
            ++it;
    }
    for (auto it = parts_.begin(); it != parts_.end();) {
        if (it->first < below)
            it = parts_.erase(it);
        else
            ++it;
    }
}

// Local part of a horizon / epoch (executed by every process): the full tokens
// of dependencies this process executes, the local parts of earlier horizons /
// epochs, nothing of dependencies executed elsewhere (their owners' parts are
// covered by the owners' own parts of this horizon / epoch).
Token Executor::multi_local_part(const std::vector<uint64_t>& deps) const {
    Token t;
    for (uint64_t j : deps) {
        int ko = 0;
        if (cfg_.world > 1 && owner_lookup(j, &ko)) {
            if (ko < 0) {
                auto lt = ltok_.find(j);
                if (lt != ltok_.end()) merge(t, lt->second);
                continue;
            }
            if (owner_rank(ko) != cfg_.rank) continue;
        }
        merge(t, dep_token(j));
    }
    return t;
}

// ------------------------------------------------------------ ownership
int Executor::instr_owner(const Instr& ins) const {
    switch (ins.kind) {
    case IKind::Alloc:
    case IKind::Free:
        return ins.mem >= 2 ? ins.mem - 2 : -1;
    case IKind::Kernel:
        return ins.device;
    case IKind::Copy:
        return ins.src_mem >= 2 ? ins.src_mem - 2 : (ins.dst_mem >= 2 ? ins.dst_mem - 2 : -1);   // push model: the producer's GPU
    default:
        return -1;
    }
}

// Local part of a set of dependencies: tokens of the deps this process executes
// (or multi-owner horizons/epochs); deps executed elsewhere appear as remote
// markers that their owner signals to us.
Token Executor::local_part(const std::vector<uint64_t>& deps) const {
    Token t;
    for (uint64_t j : deps) merge(t, dep_token(j));
    return t;
}

// Called on a process that does NOT execute `ins`: signal to the executing
// process every dependency whose (local part of the) completion lives here.
void Executor::signal_deps(const Instr& ins, int owner_dev) {
    const int o = owner_rank(owner_dev);
    for (uint64_t j : ins.deps) {
        int jo = 0;                           // owner device, -1 = all
        if (!owner_lookup(j, &jo)) continue;  // complete before any remote dependent existed
        if (jo >= 0 && owner_rank(jo) != cfg_.rank) continue;
        const uint64_t key = j * uint64_t(cfg_.world) + uint64_t(o);
        if (!signalled_.insert(key).second) continue;
        if (parked_iids_.count(j)) {          // not launched yet (exec_fuse.cu): signal once it is
            deferred_signals_.push_back({j, o});
            continue;
        }
        signal_one(j, jo, o);
    }
}

// Write "instruction j done" into rank o's flag slot once j's local work has
// completed (stream-ordered after it).
void Executor::signal_one(uint64_t j, int jo, int o) {
    Token t;
    if (jo < 0) {
        auto lt = ltok_.find(j);
        if (lt != ltok_.end()) t = lt->second;
    } else {
        t = dep_token(j);
    }
    Token live;
    merge(live, t);                               // drops entries already known complete
    int sidx = cfg_.rank * kStreamsPerDev + S_SYNC;
    if (live.remote.empty() && live.local.size() == 1)
        sidx = cfg_.rank * kStreamsPerDev + S_SIG0 + (live.local[0].stream % kStreamsPerDev) % kNumSigStreams;
    wait_token(sidx, live);
    if (trace_) fprintf(stderr, "[cel r%d] signal iid %llu -> rank %d\n", cfg_.rank, (unsigned long long)j, o);
    const uint64_t ts = now_ns();
    checkd(g_drv.write64(reinterpret_cast<CUstream>(streams_[sidx].s),
                         reinterpret_cast<CUdeviceptr>(sig_slot(o, cfg_.rank, j)), j, CU_STREAM_WRITE_VALUE_DEFAULT),
           "cuStreamWriteValue64");
    st_.signal_ns += now_ns() - ts;
    st_.signals++;
}

void Executor::flush_deferred_signals() {
    for (size_t i = 0; i < deferred_signals_.size();) {
        const auto p = deferred_signals_[i];
        if (parked_iids_.count(p.first)) {
            ++i;
            continue;
        }
        int jo = 0;
        if (!owner_lookup(p.first, &jo)) jo = cfg_.rank;
        signal_one(p.first, jo, p.second);
        deferred_signals_.erase(deferred_signals_.begin() + long(i));
    }
}

char* Executor::alloc_ptr(int64_t aid) {
    auto it = allocs_.find(aid);
    if (it == allocs_.end()) return nullptr;
    const AllocRec& r = it->second;
    return base_of(r);
}

// ------------------------------------------------------------ dispatch
void Executor::on_instr(const Instr& ins) {
    if (threaded_) {
        Item it;
        it.kind = 0;
        it.ins = ins;
        push(std::move(it));
        return;
    }
    const uint64_t t0 = now_ns();
    on_instr_impl(ins);
    cur_ins_ = nullptr;
    st_.exec_ns[int(ins.kind)] += now_ns() - t0;
}

// ------------------------------------------------------------ executor thread
void Executor::push(Item&& it) {
    bool wake;
    {
        std::unique_lock<std::mutex> l(qm_);
        // bounded run-ahead of the scheduler (not in virtual-node mode: a node's
        // executor may wait for pilots another node's compilation produces)
        while (q_.size() >= 16384 && !cfg_.comm) qfull_cv_.wait(l);
        q_.push_back(std::move(it));
        qsize_.store(q_.size(), std::memory_order_release);
        wake = sleeping_;
    }
    if (wake) qcv_.notify_one();
}

void Executor::post(std::function<void()> fn) {
    if (!threaded_) {
        fn();
        return;
    }
    Item it;
    it.kind = 1;
    it.fn = std::move(fn);
    push(std::move(it));
}

void Executor::drain() {
    if (!threaded_) return;
    Item it;
    it.kind = 2;
    it.mark = ++marks_posted_;
    const uint64_t m = it.mark;
    push(std::move(it));
    std::unique_lock<std::mutex> l(dm_);
    done_cv_.wait(l, [&] { return marks_done_ >= m; });
}

// Thread pinning ("pinned threads"): the executor
// thread, which spins for new instructions, gets a core of its own -- the
// process's affinity set counted from the top, one per rank / virtual node --
// when the set has at least 4 cores.  CEL_PIN=0 leaves scheduling to the OS.
void Executor::pin_thread() {
    const char* pin = getenv("CEL_PIN");
    if (pin && pin[0] == '0') return;
    cpu_set_t m;
    CPU_ZERO(&m);
    if (sched_getaffinity(0, sizeof m, &m) != 0) return;
    std::vector<int> cores;
    for (int c = 0; c < CPU_SETSIZE; ++c)
        if (CPU_ISSET(c, &m)) cores.push_back(c);
    if (cores.size() < 4) return;
    const int k = (cfg_.rank + cfg_.node) % int(cores.size());
    cpu_set_t one;
    CPU_ZERO(&one);
    CPU_SET(cores[cores.size() - 1 - size_t(k)], &one);
    if (pthread_setaffinity_np(pthread_self(), sizeof one, &one) == 0) pinned_core_ = cores[cores.size() - 1 - size_t(k)];
}

void Executor::thread_main() {
    pin_thread();
    for (;;) {
        Item it;
        {
            std::unique_lock<std::mutex> l(qm_);
            if (q_.empty()) {
                l.unlock();
                // spin briefly: the scheduler usually posts the next
                // instruction within microseconds (latency of
                // instruction selection matters for strong scaling)
                for (int i = 0; i < 20000 && qsize_.load(std::memory_order_acquire) == 0; ++i) _mm_pause();
                l.lock();
                while (q_.empty() && !stop_) {
                    sleeping_ = true;
                    qcv_.wait(l);
                    sleeping_ = false;
                }
                if (q_.empty() && stop_) return;
            }
            it = std::move(q_.front());
            q_.pop_front();
            qsize_.store(q_.size(), std::memory_order_release);
            if (q_.size() == 8192) qfull_cv_.notify_all();
        }
        if (it.kind == 0) {
            const uint64_t t0 = now_ns();
            on_instr_impl(it.ins);
            cur_ins_ = nullptr;
            if (err_ && cfg_.comm) cfg_.comm->abort();   // wake nodes waiting for this one
            st_.exec_ns[int(it.ins.kind)] += now_ns() - t0;
            if ((++since_publish_ & 255) == 0) publish_stats();
        } else if (it.kind == 1) {
            it.fn();
        } else {
            halo_flush();                                // a drain / epoch wait: nothing stays held back
            flush_parked();
            if (!deferred_signals_.empty()) flush_deferred_signals();
            publish_stats();
            {
                std::lock_guard<std::mutex> l(dm_);
                marks_done_ = it.mark;
            }
            done_cv_.notify_all();
        }
    }
}

void Executor::add_buffer(uint32_t bid, const Box& extent, uint32_t es) {
    post([this, bid, extent, es] { bufinfo_[bid] = BufInfo{extent, es}; });
}

void Executor::set_profile(int stride) {
    drain();
    cfg_.profile = stride > 0;
    prof_stride_ = stride > 0 ? stride : 1;
    for (auto& c : prof_ctr_) c = 0;
    if (!cfg_.profile) return;
    // time origin of the trace on every owned device
    trace_ref_.assign(G_, nullptr);
    trace_recs_.clear();
    for (int d = 0; d < G_; ++d) {
        if (!owned(d)) continue;
        set_dev(d);
        cudaEvent_t e = nullptr;
        check(cudaEventCreate(&e), "cudaEventCreate");
        check(cudaEventRecord(e, streams_[d * kStreamsPerDev + S_SYNC].s), "cudaEventRecord");
        trace_ref_[d] = e;
    }
    // the device is idle here (drained), so the reference event fires now
    for (int d = 0; d < G_; ++d)
        if (trace_ref_[d]) cudaEventSynchronize(trace_ref_[d]);
    trace_ref_ns_ = now_ns();
}

int Executor::trace_dump(const char* path) {
    double ms[kProfSlots];
    uint64_t c[kProfSlots];
    profile_read(ms, c, kProfSlots);          // resolves pending launches into trace_recs_
    FILE* f = fopen(path, "w");
    if (!f) return E_INVALID;
    static const char* names[] = {"fill_hash", "fill_const", "stencil3", "wave5",  "jacobi7", "nbody_step",
                                  "nbody_update", "rsim_row", "probe", "callback", "copy", "copy_peer", "shell", "coll"};
    static const char* snames[] = {"compute", "copy", "push", "sync", "halo", "hsig", "sig0", "sig1", "sig2", "sig3", "sig4"};
    for (const TraceRec& t : trace_recs_)
        fprintf(f,
                "{\"iid\":%llu,\"rank\":%d,\"device\":%d,\"stream\":\"%s\",\"kind\":\"%s\",\"start_us\":%.3f,"
                "\"end_us\":%.3f,\"host_issue_us\":%.3f}\n",
                (unsigned long long)t.iid, cfg_.rank, t.dev, snames[t.stream % kStreamsPerDev], names[t.kind],
                t.start_us, t.end_us, t.issue_us);
    fclose(f);
    return E_OK;
}

void Executor::on_instr_impl(const Instr& ins) {
    if (err_) return;
    cur_ins_ = &ins;
    check_owner_known(ins);
    if (err_) return;
    if (!staged_.empty()) {
        settle_staged(ins);
    } else if (direct_src_ >= 0 || !settle_tok_.empty()) {
        direct_src_ = -1;
        direct_staged_ = 0;
        settle_tok_ = Token{};
    }
    if (!pending_send_.empty()) resolve_sends(ins);
    // WaveSim halo exchange fused into the stencil launches (exec_halo.cu)
    if (fuse_halo_ && !halo_flushing_) {
        if (halo_parked_) {
            if (halo_attach(ins)) return;
            const bool dep = halo_depends(ins);
            if (ins.kind == IKind::Horizon && dep && halo_deferred_.size() < 4) {
                halo_deferred_.push_back(ins);           // waits with the held-back kernel
                halo_iids_.insert(ins.iid);
                return;
            }
            if (dep || ins.kind == IKind::Horizon || ins.kind == IKind::Epoch) {
                halo_flush();
                cur_ins_ = &ins;
            }
        }
        if (halo_candidate(ins)) {
            halo_kernel_ = ins;
            halo_parked_ = true;
            halo_iids_.insert(ins.iid);
            return;
        }
    }
    // rows fused with their gathers (exec_fuse.cu): hold back a fusable row
    // kernel, and whatever depends on something held back, except the
    // all-gather members (held as a set anyway)
    const bool gather_member = (coll_ || mc_enabled_ || p2p_gather_) && ins.kind == IKind::Copy && ins.coll_n;
    if (!flushing_ && !parked_iids_.empty() && !gather_member && depends_on_parked(ins)) {
        park(ins);
        return;
    }
    if (park_candidate(ins)) {
        if (cfg_.world > 1) kind_of_[ins.iid] = ins.device;
        park(ins);
        return;
    }
    const int od = instr_owner(ins);
    const bool mine = od < 0 || owner_rank(od) == cfg_.rank;
    if (trace_)
        fprintf(stderr, "[cel r%d] iid %llu kind %d owner %d %s\n", cfg_.rank, (unsigned long long)ins.iid,
                int(ins.kind), od, mine ? "exec" : "skip");
    if (gather_member) {
        // §8 a7: a member of an all-gather copy set.  Every rank takes part;
        // the source's and the destination's ranks each wait for the member's
        // dependencies, so the other ranks signal theirs to both.
        const int sd = ins.src_mem - 2, dd = ins.dst_mem - 2;
        if (cfg_.world > 1) {
            kind_of_[ins.iid] = -1;
            if (owner_rank(sd) != cfg_.rank) signal_deps(ins, sd);
            if (owner_rank(dd) != cfg_.rank) signal_deps(ins, dd);
        }
        copy_info_[ins.iid] = CopyInfo{ins.src_aid, ins.dst_aid, rbbox(ins.region), ins.region};
        auto& g = coll_pending_[ins.coll];
        g.push_back(ins);
        if (g.size() == ins.coll_n) {
            exec_coll(g);
            coll_pending_.erase(ins.coll);
        }
        return;
    }
    if (cfg_.world > 1) {
        if (od >= 0) kind_of_[ins.iid] = od;
        else kind_of_[ins.iid] = -1;
        if (!mine && ins.kind != IKind::Alloc) signal_deps(ins, od);
    }
    switch (ins.kind) {
    case IKind::Alloc: {
        const int dev = ins.mem - 2;
        const uint32_t es = bufinfo_.at(ins.buffer).es;
        // Physical layout: the allocation's innermost dimension is padded to
        // 16-byte boundaries (lower end rounded down, width rounded up), so rows
        // start aligned even when the box begins at a halo column (2-D split):
        // the vectorised kernels and 16-byte copy paths then apply.  The IDAG's
        // box is unchanged; every address is computed from the padded box.
        const Box pbox = padded_box(ins.box, ins.buffer, es);
        const uint64_t bytes = pbox.volume() * es;
        uint64_t off = 0;
        Token t;
        // In-place growth: a resize that keeps a live
        // allocation's rows as the prefix of the new box (same lo, same row
        // pitch, growth at the end of dim 0) takes the old allocation's
        // address when the arena range right after it is free.  Its resize
        // copies then move nothing and its free releases nothing.  Every rank
        // replays this decision identically (it depends only on the
        // instruction stream and the arena state).
        AllocRec* grow = nullptr;
        for (auto& kv : allocs_) {
            AllocRec& o = kv.second;
            if (no_grow_ || o.dev != dev || o.buffer != ins.buffer || o.absorbed_into) continue;
            const Box& ob = o.box;
            if (ob.lo[0] == pbox.lo[0] && ob.lo[1] == pbox.lo[1] && ob.lo[2] == pbox.lo[2] &&
                ob.hi[1] == pbox.hi[1] && ob.hi[2] == pbox.hi[2] && ob.hi[0] <= pbox.hi[0]) {
                grow = &o;
                break;
            }
        }
        // Placement (single process with VMM; multi-process runs use the arena
        // only, the layout every rank replays):
        //  1. growing a VMM allocation: map granules behind its rows, in place;
        //  2. growing an arena allocation whose successor range is free: in place;
        //  3. growing otherwise: a VMM allocation reserved up to the buffer's end
        //     along dim 0 (one copy now, later growth in place);
        //  4. anything else from the pre-reserved arena (allocation instructions
        //     cost nothing on the hot path), VMM when the arena is full -- the
        //     arena size is no cap on the buffers' allocations.
        std::shared_ptr<VmmRegion> vreg;
        const bool vmm_ok = vmm_ && dev >= 0;
        auto vmm_new = [&](bool growth) {
            uint64_t reserve = bytes;
            if (growth) {        // R9 growth keeps lo and the row pitch: room to the buffer's end along dim 0
                const uint64_t slice = bytes / uint64_t(std::max<int64_t>(1, pbox.extent(0)));
                const int64_t rows_max = bufinfo_.at(ins.buffer).extent.hi[0] - pbox.lo[0];
                reserve = std::min<uint64_t>(slice * uint64_t(std::max<int64_t>(rows_max, 1)), 1ull << 40);
            }
            vreg = vmm_create(dev, bytes, reserve);
            return vreg != nullptr;
        };
        if (vmm_ok && grow && grow->vmm && vmm_map_more(*grow->vmm, bytes)) {
            vreg = grow->vmm;                                           // 1
            grow->absorbed_into = ins.aid;
            if (mine) merge(t, grow->use);
        } else if (grow && !grow->vmm && !(vmm_ok && mc_enabled_ && bytes >= vmm_gran_) &&
                   arena(dev).extend(grow->off, grow->bytes, bytes, &t)) {
            // 2: the grown allocation's users write memory the old one's readers
            // may still read: follow every local use of the old allocation
            // (remote ranks only write it, and those writes reach the new
            // allocation's users through the resize copies' dependencies)
            off = grow->off;
            grow->absorbed_into = ins.aid;
            if (mine) merge(t, grow->use);
        } else if (vmm_ok && grow && vmm_new(true)) {
            // 3
        } else if (vmm_ok && mc_enabled_ && bytes >= vmm_gran_ && vmm_new(false)) {
            // multicast gathers bind VMM memory: large allocations are mapped
        } else if (!arena(dev).alloc(bytes, &off, &t) && !(vmm_ok && vmm_new(false))) {
            char buf[200];
            snprintf(buf, sizeof buf, "device %d: cannot allocate %.3f GiB (arena exhausted%s)", dev,
                     double(bytes) / (1ull << 30), vmm_ok ? ", VMM mapping failed" : "");
            errmsg_ = buf;
            err_ = E_OOM;
            return;
        }
        allocs_[ins.aid] = AllocRec{dev, off, bytes, pbox, es, ins.iid, ins.buffer};
        if (vreg) allocs_[ins.aid].vmm = vreg;
        live_alloc_iid_.insert(ins.iid);
        Token mt;
        if (mine) merge(mt, t);
        else mt.remote.push_back({owner_rank(dev), ins.iid});
        if (mt.remote.size() > 8) mt = materialize(dev, mt);
        tok_[ins.iid] = mt;
        return;
    }
    case IKind::Free: {
        auto it = allocs_.find(ins.aid);
        if (it == allocs_.end()) {
            errmsg_ = "free of an unknown allocation";
            err_ = E_STATE;
            return;
        }
        const AllocRec r = it->second;
        Token t;
        if (mine) {
            t = local_part(ins.deps);
            for (uint64_t j : ins.deps) {
                int ko = 0;
                if (cfg_.world > 1 && owner_lookup(j, &ko) && ko >= 0 && owner_rank(ko) != cfg_.rank &&
                    std::find(t.remote.begin(), t.remote.end(), std::make_pair(owner_rank(ko), j)) == t.remote.end())
                    t.remote.push_back({owner_rank(ko), j});
            }
            if (t.remote.size() > 8) t = materialize(r.dev, t);
        } else {
            t.remote.push_back({owner_rank(r.dev), ins.iid});
        }
        if (!settle_tok_.empty()) merge(t, settle_tok_);   // elided staging copies that read it just now
        if (!r.absorbed_into) {                   // else: lives on in the grown one
            if (r.vmm)
                vmm_free_.push_back({r.vmm, t});  // unmapped once the free's dependencies have completed
            else
            {
                // coalesced ranges accumulate their frees' tokens: fold a
                // long one into one event (each later allocation from the
                // range merges it; lookahead none across processes freed a
                // range per row and spent ~1.4 ms per row merging)
                // (another rank's arena is bookkeeping here: its tokens are never used)
                Token& ft = arena(r.dev).release(r.off, r.bytes, mine ? t : Token{});
                if (mine && (ft.remote.size() > 8 || ft.local.size() > 16)) ft = materialize(r.dev, ft);
            }
        }
        tok_[ins.iid] = t;
        live_alloc_iid_.erase(r.iid);
        allocs_.erase(it);
        return;
    }
    case IKind::Copy:
        // the interior / shell split of this rank's kernels inspects copies
        // into its own allocations too (executed by their producer's rank)
        if (mine || (ins.dst_mem >= 2 && owner_rank(ins.dst_mem - 2) == cfg_.rank))
            copy_info_[ins.iid] = CopyInfo{ins.src_aid, ins.dst_aid, rbbox(ins.region), ins.region};
        if (!mine) return;                        // token: dep_token() -> the owner's flag
        exec_copy(ins);
        break;
    case IKind::Kernel:
        if (!mine) return;
        exec_kernel(ins);
        break;
    case IKind::Horizon: {
        // completion of a horizon tells us everything before it is done;
        // deps older than the applied (previous) horizon are never referenced again.
        Token lt = multi_local_part(ins.deps);
        ltok_[ins.iid] = lt;
        if (cfg_.comm && prev_horizon_) {
            // virtual-node mode bounds the run-ahead here (throttle() must not
            // block): wait for the previous horizon, which only depends on
            // sends / pulls every node has already issued
            auto pit = ltok_.find(prev_horizon_);
            if (pit != ltok_.end())
                for (const TokEntry& e : pit->second.local)
                    if (e.seq > streams_[e.stream].done) check(cudaEventSynchronize(e.ev), "horizon wait");
            st_.host_syncs++;
        }
        Token t = lt;
        for (int r = 0; r < cfg_.world; ++r)
            if (r != cfg_.rank) t.remote.push_back({r, ins.iid});
        if (cfg_.world > 1) {
            // every rank will need this horizon's parts (deps subsumed into it,
            // P:L429): publish ours to all ranks now, on a stream of its own
            const int hs = cfg_.rank * kStreamsPerDev + S_HSIG;
            wait_token(hs, lt);
            for (int r = 0; r < cfg_.world; ++r) {
                if (r == cfg_.rank) continue;
                signalled_.insert(ins.iid * uint64_t(cfg_.world) + uint64_t(r));
                checkd(g_drv.write64(reinterpret_cast<CUstream>(streams_[hs].s),
                                     reinterpret_cast<CUdeviceptr>(sig_slot(r, cfg_.rank, ins.iid)), ins.iid,
                                     CU_STREAM_WRITE_VALUE_DEFAULT),
                       "cuStreamWriteValue64");
                st_.signals++;
            }
        }
        tok_[ins.iid] = t;
        poll(false);
        throttle();
        // prune tokens below the previously emitted horizon (allocation tokens stay)
        if (prev_horizon_) prune_tokens(prev_horizon_);
        prev_horizon_ = ins.iid;
        return;
    }
    case IKind::Epoch:
        exec_epoch(ins);
        return;
    case IKind::Send:
    case IKind::Receive:
    case IKind::SplitReceive:
    case IKind::AwaitReceive:
        exec_transfer(ins);
        break;
    }
    if (grown_) note_use(ins);
    if (++since_poll_ >= 64) {
        since_poll_ = 0;
        poll(false);
        throttle();
    }
}

void Executor::exec_epoch(const Instr& ins) {
    Token t = multi_local_part(ins.deps);
    // an epoch synchronises with the main thread
    if (cfg_.world > 1) {
        const int sidx = cfg_.rank * kStreamsPerDev + S_SYNC;
        wait_token(sidx, t);
        check(cudaStreamSynchronize(streams_[sidx].s), "epoch synchronize");
    } else {
        for (const TokEntry& e : t.local)
            if (e.seq > streams_[e.stream].done) check(cudaEventSynchronize(e.ev), "epoch synchronize");
    }
    st_.host_syncs++;
    poll(true);
    if (!oob_pending_.empty()) oob_check(true);
    for (uint32_t bid : host_drop_) {
        auto it = host_init_.find(bid);
        if (it != host_init_.end()) {
            if (it->second.second) cudaFreeHost(it->second.first);
            host_init_.erase(it);
        }
    }
    host_drop_.clear();
    if (pending_send_.empty()) msg_tok_.clear();
    for (auto it = elided_iids_.begin(); it != elided_iids_.end();)
        it = (*it < ins.iid && !pending_send_.count(*it) && !staged_.count(*it)) ? elided_iids_.erase(it) : std::next(it);
    Token mine;
    for (int r = 0; r < cfg_.world; ++r)
        if (r != cfg_.rank) mine.remote.push_back({r, ins.iid});
    // everything before the epoch is complete locally: drop old tokens
    prune_tokens(ins.iid);
    prev_horizon_ = 0;
    for (auto& st : streams_) st.waited_remote.clear();
    for (auto it = signalled_.begin(); it != signalled_.end();) {
        const uint64_t j = *it / uint64_t(cfg_.world);
        if (j < ins.iid && !live_alloc_iid_.count(j))
            it = signalled_.erase(it);
        else
            ++it;
    }
    tok_[ins.iid] = mine;
    ltok_[ins.iid] = Token{};
    if (cfg_.world > 1) {
        // remote markers older than the epoch stay valid (their slots keep the value)
        for (auto it = kind_of_.begin(); it != kind_of_.end();) {
            if (it->first + kRing / 2 < ins.iid) it = kind_of_.erase(it);
            else ++it;
        }
    }
}

cudaEvent_t Executor::prof_event(int dev) {
    auto& p = prof_pool_[dev];
    if (!p.empty()) {
        cudaEvent_t e = p.back();
        p.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    check(cudaEventCreate(&e), "cudaEventCreate");   // timing-enabled
    return e;
}

int Executor::profile_read(double* ms, uint64_t* count, int n) {
    drain();
    for (auto& p : prof_pending_) {
        float t = 0.f;
        cudaEventSynchronize(p.b);
        cudaEventElapsedTime(&t, p.a, p.b);
        prof_ms_[p.kind] += t;
        prof_n_[p.kind]++;
        if (p.dev < int(trace_ref_.size()) && trace_ref_[p.dev] && trace_recs_.size() < 200000) {
            float s0 = 0.f, s1 = 0.f;
            cudaEventElapsedTime(&s0, trace_ref_[p.dev], p.a);
            cudaEventElapsedTime(&s1, trace_ref_[p.dev], p.b);
            trace_recs_.push_back(TraceRec{p.iid, p.dev, p.stream, p.kind, s0 * 1e3, s1 * 1e3,
                                           (double(p.issue_ns) - double(trace_ref_ns_)) / 1e3});
        }
        prof_pool_[p.dev].push_back(p.a);
        prof_pool_[p.dev].push_back(p.b);
    }
    prof_pending_.clear();
    for (int i = 0; i < n && i < kProfSlots; ++i) {
        ms[i] = prof_ms_[i];
        count[i] = prof_n_[i];
    }
    return E_OK;
}

void Executor::profile_reset() {
    double ms[kProfSlots];
    uint64_t c[kProfSlots];
    profile_read(ms, c, kProfSlots);
    for (int i = 0; i < kProfSlots; ++i) {
        prof_ms_[i] = 0;
        prof_n_[i] = 0;
    }
}

}  // namespace cel
