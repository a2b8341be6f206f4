// C-ABI (include/cel.h) over the scheduler and executor.
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>

#include "../../include/cel.h"
#include "exec.hpp"
#include "sched.hpp"

using namespace cel;

namespace {
thread_local std::string g_err;

int fail(int rc, const std::string& msg) {
    g_err = msg;
    return rc;
}

Box to_box(const cel_box& b) {
    int64_t lo[3], hi[3];
    for (int d = 0; d < 3; ++d) {
        lo[d] = int64_t(b.min[d]);
        hi[d] = int64_t(b.max[d]);
    }
    return Box::make(lo, hi);
}

uint64_t now_ns() {
    return uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now().time_since_epoch())
                        .count());
}
}  // namespace

struct cel_runtime {
    cel_config cfg;
    FILE* log = nullptr;
    std::unique_ptr<Executor> exec;
    std::unique_ptr<Scheduler> sched;
    // virtual-node mode (n_nodes > 1): one scheduler (and executor) per node
    std::unique_ptr<Cluster> cluster;
    std::vector<FILE*> node_logs;
    std::vector<std::unique_ptr<Executor>> node_exec;
    std::shared_ptr<Communicator> comm;
    uint64_t gen_ns = 0;
    int poisoned = 0;
    bool destroyed = false;
};

namespace {
std::vector<Executor*> execs(cel_runtime* rt) {
    std::vector<Executor*> v;
    if (rt->exec) v.push_back(rt->exec.get());
    for (auto& e : rt->node_exec) v.push_back(e.get());
    return v;
}
Scheduler& sched0(cel_runtime* rt) { return rt->cluster ? rt->cluster->node(0) : *rt->sched; }
Executor* exec0(cel_runtime* rt) { return rt->cluster ? (rt->node_exec.empty() ? nullptr : rt->node_exec[0].get()) : rt->exec.get(); }
int check_poison(cel_runtime* rt) {
    if (!rt) return fail(CEL_E_INVALID, "null runtime");
    if (rt->poisoned) return rt->poisoned;
    for (Executor* e : execs(rt))
        if (e->error()) {
            rt->poisoned = e->error();
            return fail(rt->poisoned, e->error_msg());
        }
    return 0;
}
int after(cel_runtime* rt, int rc) {
    for (Executor* e : execs(rt))
        if (e->error()) {
            rt->poisoned = e->error();
            return fail(rt->poisoned, e->error_msg());
        }
    return rc;
}
void drain_all(cel_runtime* rt) {
    for (Executor* e : execs(rt)) e->drain();
}
}  // namespace

extern "C" {

const char* cel_last_error(void) { return g_err.c_str(); }

size_t cel_ipc_blob_size(void) { return Executor::kBlobBytes; }

int cel_runtime_create(const cel_config* cfg, cel_runtime** out) {
    if (!cfg || !out) return fail(CEL_E_INVALID, "null argument");
    if (cfg->n_devices < 1 || cfg->n_devices > 30) return fail(CEL_E_INVALID, "n_devices must be 1..30");
    if (cfg->lookahead < 0 || cfg->lookahead > 2) return fail(CEL_E_INVALID, "lookahead must be 0, 1 or 2");
    const int world = cfg->world > 0 ? cfg->world : 1;
    if (world > 1 && (cfg->rank < 0 || cfg->rank >= world || world != cfg->n_devices))
        return fail(CEL_E_INVALID, "multi-process mode needs 0 <= rank < world == n_devices");
    const int nodes = cfg->n_nodes > 1 ? cfg->n_nodes : 1;
    if (nodes > 1 && world > 1) return fail(CEL_E_INVALID, "virtual-node mode runs in one process (world must be 1)");
    if (nodes > 30) return fail(CEL_E_INVALID, "n_nodes must be <= 30");
    auto rt = std::make_unique<cel_runtime>();
    rt->cfg = *cfg;
    rt->cfg.world = world;
    if (nodes > 1) {
        // virtual-node mode: node k = its own scheduler (+ executor) over devices
        // cuda_devices[k * n_devices ...]
        for (int k = 0; k < nodes; ++k) {
            FILE* f = nullptr;
            if (cfg->instr_log_path && cfg->instr_log_path[0]) {
                const std::string path = std::string(cfg->instr_log_path) + "." + std::to_string(k);
                f = fopen(path.c_str(), "w");
                if (!f) {
                    for (FILE* g : rt->node_logs)
                        if (g) fclose(g);
                    return fail(CEL_E_INVALID, "cannot open " + path);
                }
            }
            rt->node_logs.push_back(f);
        }
        std::vector<InstrSink*> sinks(nodes, nullptr);
        if (cfg->execute) {
            auto comm = std::make_shared<Communicator>(nodes);
            rt->comm = comm;
            for (int k = 0; k < nodes; ++k) {
                ExecConfig ec;
                for (int d = 0; d < cfg->n_devices; ++d) {
                    const int v = k * cfg->n_devices + d;
                    ec.cuda_devices.push_back(cfg->cuda_devices ? cfg->cuda_devices[v] : v);
                }
                ec.arena_bytes = cfg->arena_bytes;
                ec.fast_math = cfg->fast_math != 0;
                ec.collective = false;
                ec.bounds_check = cfg->bounds_check != 0;
                ec.node = k;
                ec.comm = comm;
                for (int v = 0; v < nodes * cfg->n_devices; ++v)
                    ec.all_devices.push_back(cfg->cuda_devices ? cfg->cuda_devices[v] : v);
                // M1 staging: a pushed or awaited region is staged in one contiguous
                // allocation over its bounding box, up to a node's whole chunk
                if (cfg->arena_bytes) ec.host_arena_bytes = cfg->arena_bytes;
                rt->node_exec.emplace_back(new Executor(ec, nullptr));
                std::string err;
                const int rc = rt->node_exec.back()->init(&err);
                if (rc != 0) {
                    std::string msg = err.empty() ? rt->node_exec.back()->error_msg() : err;
                    rt->node_exec.clear();
                    for (FILE* g : rt->node_logs)
                        if (g) fclose(g);
                    return fail(rc, msg);
                }
                sinks[k] = rt->node_exec.back().get();
            }
        }
        const int step = cfg->horizon_step > 0 ? cfg->horizon_step : 4;
        rt->cluster = std::make_unique<Cluster>(nodes, cfg->n_devices, cfg->lookahead, step, cfg->checks != 0, sinks,
                                                rt->node_logs);
        for (int k = 0; k < int(rt->node_exec.size()); ++k) rt->node_exec[k]->set_scheduler(&rt->cluster->node(k));
        if (rt->comm) {
            // pilots reach the receivers' arbitration as they are compiled
            std::shared_ptr<Communicator> comm = rt->comm;
            for (int k = 0; k < nodes; ++k)
                rt->cluster->node(k).set_pilot_sink([comm](const Pilot& p) { comm->add_pilot(p); });
        }
        *out = rt.release();
        return CEL_OK;
    }
    if (cfg->instr_log_path && cfg->instr_log_path[0]) {
        rt->log = fopen(cfg->instr_log_path, "w");
        if (!rt->log) return fail(CEL_E_INVALID, std::string("cannot open ") + cfg->instr_log_path);
    }
    if (cfg->execute) {
        ExecConfig ec;
        for (int d = 0; d < cfg->n_devices; ++d) ec.cuda_devices.push_back(cfg->cuda_devices ? cfg->cuda_devices[d] : d);
        ec.rank = world > 1 ? cfg->rank : 0;
        ec.world = world;
        ec.arena_bytes = cfg->arena_bytes;
        ec.fast_math = cfg->fast_math != 0;
        ec.collective = cfg->collective != 0;
        ec.bounds_check = cfg->bounds_check != 0;
        rt->exec = std::make_unique<Executor>(ec, nullptr);
        std::string err;
        const int rc = rt->exec->init(&err);
        if (rc != 0) {
            if (rt->log) fclose(rt->log);
            return fail(rc, err.empty() ? rt->exec->error_msg() : err);
        }
    }
    const int step = cfg->horizon_step > 0 ? cfg->horizon_step : 4;
    rt->sched = std::make_unique<Scheduler>(cfg->n_devices, cfg->lookahead, step, cfg->checks != 0, rt->exec.get(),
                                            rt->log);
    const char* nf = getenv("CEL_NO_FILTER");
    if (world > 1 && !(nf && nf[0] == '1')) rt->sched->set_rank_filter(cfg->rank, world);   // before any instruction is emitted
    if (rt->exec) rt->exec->set_scheduler(rt->sched.get());
    if (rt->exec && rt->exec->gathers_any_size()) rt->sched->set_coll_min_bytes(0);
    *out = rt.release();
    return CEL_OK;
}

int cel_ipc_export(cel_runtime* rt, void* blob) {
    if (int rc = check_poison(rt)) return rc;
    if (rt->cluster) return fail(CEL_E_STATE, "virtual-node mode runs in one process");
    if (!rt->exec) return fail(CEL_E_STATE, "runtime does not execute");
    return after(rt, rt->exec->ipc_export(blob));
}

int cel_ipc_import(cel_runtime* rt, int32_t rank, const void* blob) {
    if (int rc = check_poison(rt)) return rc;
    if (rt->cluster) return fail(CEL_E_STATE, "virtual-node mode runs in one process");
    if (!rt->exec) return fail(CEL_E_STATE, "runtime does not execute");
    return after(rt, rt->exec->ipc_import(rank, blob));
}

int cel_buffer_create(cel_runtime* rt, int32_t dims, const uint64_t extent[3], uint32_t elem_size,
                      const void* host_init, cel_buffer* out) {
    return cel_buffer_create_ex(rt, dims, extent, elem_size, host_init, 0, out);
}

int cel_buffer_create_ex(cel_runtime* rt, int32_t dims, const uint64_t extent[3], uint32_t elem_size,
                         const void* host_init, uint32_t flags, cel_buffer* out) {
    if (int rc = check_poison(rt)) return rc;
    if (!extent || !out) return fail(CEL_E_INVALID, "null argument");
    int64_t ext[3] = {1, 1, 1};
    uint64_t n = 1;
    for (int d = 0; d < dims && d < 3; ++d) {
        ext[d] = int64_t(extent[d]);
        n *= extent[d];
    }
    uint32_t bid = 0;
    const int rc = rt->cluster ? rt->cluster->buffer_create(dims, ext, elem_size, host_init != nullptr, &bid)
                               : rt->sched->buffer_create(dims, ext, elem_size, host_init != nullptr, &bid);
    if (rc != 0) return fail(rc, "invalid buffer (dims 1..3, extents > 0, elem_size > 0)");
    for (Executor* e : execs(rt)) {
        e->add_buffer(bid, sched0(rt).extent(bid), elem_size);
        if (host_init) {   // every (virtual) node holds the user's host data
            const int r2 = e->set_host_init(bid, host_init, size_t(n) * elem_size, (flags & CEL_BUFFER_BORROW_HOST) != 0);
            if (r2 != 0) return fail(r2, "cannot pin host memory for host_init");
        }
    }
    *out = bid;
    return CEL_OK;
}

int cel_task_submit(cel_runtime* rt, const cel_task_desc* d, cel_task* out) {
    if (int rc = check_poison(rt)) return rc;
    if (!d || (d->n_acc > 0 && !d->acc) || d->n_acc < 0) return fail(CEL_E_INVALID, "null argument");
    if (d->kernel < 0 || d->kernel > CEL_K_CALLBACK) return fail(CEL_E_INVALID, "unknown kernel");
    if (d->kernel == CEL_K_CALLBACK && !d->fn) return fail(CEL_E_INVALID, "CALLBACK kernel without fn");
    if (d->n_acc > kMaxAcc) return fail(CEL_E_INVALID, "too many accessors");
    TaskDesc t;
    t.dims = d->dims;
    t.range = to_box(d->range);
    t.split = d->split;
    t.kernel = d->kernel;
    t.params.seed = d->params.seed;
    t.params.value = d->params.value;
    t.params.t = d->params.t;
    t.params.salt = d->params.salt;
    t.fn = reinterpret_cast<KernelFn>(d->fn);
    t.fn_user = d->fn_user;
    for (int i = 0; i < d->n_acc; ++i) {
        const cel_access& a = d->acc[i];
        Access x;
        x.buf = a.buf;
        x.mode = a.mode;
        x.map.kind = MapKind(a.map.kind);
        for (int k = 0; k < 3; ++k) {
            x.map.border[k] = a.map.border[k];
            x.map.fixed.lo[k] = int64_t(a.map.fixed.min[k]);
            x.map.fixed.hi[k] = int64_t(a.map.fixed.max[k]);
            x.map.from_kernel_dim[k] = a.map.from_kernel_dim[k];
        }
        t.acc.push_back(x);
    }
    std::string err;
    uint64_t tid = 0;
    const uint64_t t0 = now_ns();
    const int rc = rt->cluster ? rt->cluster->task_submit(t, &tid, &err) : rt->sched->task_submit(t, &tid, &err);
    rt->gen_ns += now_ns() - t0;
    if (rc < 0) return fail(rc, err);
    if (out) *out = tid;
    return after(rt, rc);
}

int cel_wait(cel_runtime* rt) {
    if (int rc = check_poison(rt)) return rc;
    const uint64_t t0 = now_ns();
    if (rt->cluster)
        rt->cluster->wait();
    else
        rt->sched->wait();
    drain_all(rt);                         // the epoch has been executed
    rt->gen_ns += now_ns() - t0;
    return after(rt, CEL_OK);
}

int cel_buffer_read(cel_runtime* rt, cel_buffer buf, const cel_box* box, void* host_dst) {
    if (int rc = check_poison(rt)) return rc;
    if (!box || !host_dst) return fail(CEL_E_INVALID, "null argument");
    if (!sched0(rt).has_buffer(buf)) return fail(CEL_E_INVALID, "unknown buffer");
    const Box b = to_box(*box);
    if (Executor* e0 = exec0(rt))        // node 0's executor owns the user pointer
        e0->set_readback(sched0(rt).next_readback_id(), host_dst, b, sched0(rt).elem_size(buf));
    std::string err;
    int64_t rb = 0;
    const int rc = rt->cluster ? rt->cluster->readback(buf, b, &rb, &err) : rt->sched->readback(buf, b, &rb, &err);
    if (rc < 0) return fail(rc, err);
    drain_all(rt);
    return after(rt, CEL_OK);
}

int cel_buffer_destroy(cel_runtime* rt, cel_buffer buf) {
    if (int rc = check_poison(rt)) return rc;
    std::string err;
    const int rc = rt->cluster ? rt->cluster->destroy(buf, &err) : rt->sched->destroy(buf, &err);
    if (rc < 0) return fail(rc, err);
    for (Executor* e : execs(rt)) e->drop_host_init_later(buf);
    return after(rt, CEL_OK);
}

int cel_stats(cel_runtime* rt, cel_stats_t* o) {
    if (int rc = check_poison(rt)) return rc;
    if (!o) return fail(CEL_E_INVALID, "null argument");
    memset(o, 0, sizeof *o);
    SchedStats s = sched0(rt).stats();
    o->memo_hits = sched0(rt).memo_hits();
    o->memo_misses = sched0(rt).memo_misses();
    if (rt->cluster)            // virtual-node mode: totals over the nodes
        for (int k = 1; k < rt->cluster->nodes(); ++k) {
            const SchedStats& x = rt->cluster->node(k).stats();
            for (int i = 0; i < 16; ++i) s.n_by_kind[i] += x.n_by_kind[i];
            for (int i = 0; i < 3; ++i) {
                s.copies_by_reason[i] += x.copies_by_reason[i];
                s.bytes_by_reason[i] += x.bytes_by_reason[i];
            }
            s.bytes_d2d_peer += x.bytes_d2d_peer;
            s.alloc_bytes_peak += x.alloc_bytes_peak;
            s.flushes += x.flushes;
            s.gather_sets += x.gather_sets;
        }
    o->n_send = s.n_by_kind[int(IKind::Send)];
    o->n_receive = s.n_by_kind[int(IKind::Receive)];
    o->n_split_receive = s.n_by_kind[int(IKind::SplitReceive)];
    o->n_await_receive = s.n_by_kind[int(IKind::AwaitReceive)];
    o->n_alloc = s.n_by_kind[int(IKind::Alloc)];
    o->n_free = s.n_by_kind[int(IKind::Free)];
    o->n_copy = s.n_by_kind[int(IKind::Copy)];
    o->n_kernel = s.n_by_kind[int(IKind::Kernel)];
    o->n_horizon = s.n_by_kind[int(IKind::Horizon)];
    o->n_epoch = s.n_by_kind[int(IKind::Epoch)];
    o->copies_resize = s.copies_by_reason[REASON_RESIZE];
    o->copies_coherence = s.copies_by_reason[REASON_COHERENCE];
    o->copies_readback = s.copies_by_reason[REASON_READBACK];
    o->bytes_resize = s.bytes_by_reason[REASON_RESIZE];
    o->bytes_coherence = s.bytes_by_reason[REASON_COHERENCE];
    o->bytes_readback = s.bytes_by_reason[REASON_READBACK];
    o->bytes_d2d_peer = s.bytes_d2d_peer;
    o->alloc_bytes_peak = s.alloc_bytes_peak;
    o->flushes = s.flushes;
    o->gather_sets = s.gather_sets;
    o->gen_ns = rt->gen_ns;
    for (Executor* ex : execs(rt)) {
        const ExecStats e = ex->stats();      // the executor thread's published copy
        o->kernel_launches += e.kernel_launches;
        o->copy_launches += e.copy_launches;
        o->memcpy_calls += e.memcpy_calls;
        o->event_waits += e.event_waits;
        o->remote_waits += e.remote_waits;
        o->signals += e.signals;
        o->host_syncs += e.host_syncs;
        o->exec_ns_alloc += e.exec_ns[0];
        o->exec_ns_free += e.exec_ns[1];
        o->exec_ns_copy += e.exec_ns[2];
        o->exec_ns_kernel += e.exec_ns[3];
        o->exec_ns_horizon += e.exec_ns[4];
        o->exec_ns_epoch += e.exec_ns[5];
        o->signal_ns += e.signal_ns;
        o->remote_wait_ns += e.remote_wait_ns;
        o->copies_elided += e.copies_elided;
        o->bytes_elided += e.bytes_elided;
        o->coll_groups += e.coll_groups;
        o->coll_copies += e.coll_copies;
        o->coll_allgathers += e.coll_allgathers;
        o->tma_copy_launches += e.tma_copy_launches;
        o->vmm_maps += e.vmm_maps;
        o->vmm_mapped_bytes += e.vmm_mapped_bytes;
        o->coll_multicast += e.coll_multicast;
        o->coll_p2p += e.coll_p2p;
        o->coll_fused += e.coll_fused;
        o->halo_fused += e.halo_fused;
        o->halo_in_waits += e.halo_in_waits;
        o->halo_chained += e.halo_chained;
        o->staging_elided += e.staging_elided;
        o->staging_materialized += e.staging_materialized;
    }
    if (rt->comm) {
        o->pulls = rt->comm->pulls();
        o->pull_bytes = rt->comm->pull_bytes();
    }
    return CEL_OK;
}

int cel_stats_get(cel_runtime* rt, cel_stats_t* o) { return cel_stats(rt, o); }

int cel_profile_enable(cel_runtime* rt, int32_t on) {
    if (int rc = check_poison(rt)) return rc;
    if (execs(rt).empty()) return fail(CEL_E_STATE, "runtime does not execute");
    for (Executor* e : execs(rt)) {
        e->set_profile(on > 0 ? on : 0);
        if (on > 0) e->profile_reset();
    }
    return after(rt, CEL_OK);
}

int cel_profile_read(cel_runtime* rt, double* ms, uint64_t* count, int32_t n) {
    if (int rc = check_poison(rt)) return rc;
    if (execs(rt).empty()) return fail(CEL_E_STATE, "runtime does not execute");
    if (!ms || !count || n < 0) return fail(CEL_E_INVALID, "null argument");
    for (int i = 0; i < n; ++i) {
        ms[i] = 0;
        count[i] = 0;
    }
    std::vector<double> m2(size_t(n) + 1);
    std::vector<uint64_t> c2(size_t(n) + 1);
    for (Executor* e : execs(rt)) {      // virtual-node mode: totals over the nodes
        const int rc = e->profile_read(m2.data(), c2.data(), n);
        if (rc != 0) return after(rt, rc);
        for (int i = 0; i < n; ++i) {
            ms[i] += m2[i];
            count[i] += c2[i];
        }
    }
    return after(rt, CEL_OK);
}

int cel_trace_dump(cel_runtime* rt, const char* path) {
    if (int rc = check_poison(rt)) return rc;
    if (!exec0(rt)) return fail(CEL_E_STATE, "runtime does not execute");
    if (!path) return fail(CEL_E_INVALID, "null path");
    return after(rt, exec0(rt)->trace_dump(path));
}

int cel_runtime_destroy(cel_runtime* rt) {
    if (!rt) return fail(CEL_E_INVALID, "null runtime");
    int rc = CEL_OK;
    int err = rt->poisoned;
    for (Executor* e : execs(rt))
        if (!err && e->error()) err = e->error();
    if (!err) {
        if (rt->cluster)
            rt->cluster->shutdown();
        else
            rt->sched->shutdown();
        drain_all(rt);
        for (Executor* e : execs(rt))
            if (e->error() && rc == CEL_OK) rc = fail(e->error(), e->error_msg());
    } else {
        rc = err;
        if (rt->comm) rt->comm->abort();   // wake nodes waiting for a failed peer
    }
    rt->sched.reset();
    rt->exec.reset();
    rt->cluster.reset();
    rt->node_exec.clear();
    rt->comm.reset();
    if (rt->log) fclose(rt->log);
    for (FILE* f : rt->node_logs)
        if (f) fclose(f);
    delete rt;
    return rc;
}

}  // extern "C"
