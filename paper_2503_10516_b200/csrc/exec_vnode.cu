// Executor: virtual-node mode transfers -- Communicator (receive arbitration,
// P:L534-544), send / receive / split receive / await receive (Table 1, §3.4).
#include "exec_impl.hpp"

namespace cel {

// ------------------------------------------------------------ virtual-node communicator
namespace {
// one box of a row-major allocation copied into another: a copy-kernel segment
void box_seg(CopyArgs& args, const char* sb, const Box& S, char* db, const Box& D, const Box& b, uint32_t es) {
    const int64_t sn1 = S.extent(1), sn2 = S.extent(2), dn1 = D.extent(1), dn2 = D.extent(2);
    CopySeg g;
    const int64_t so = ((b.lo[0] - S.lo[0]) * sn1 + (b.lo[1] - S.lo[1])) * sn2 + (b.lo[2] - S.lo[2]);
    const int64_t dof = ((b.lo[0] - D.lo[0]) * dn1 + (b.lo[1] - D.lo[1])) * dn2 + (b.lo[2] - D.lo[2]);
    g.src = sb + so * es;
    g.dst = db + dof * es;
    g.row_bytes = uint64_t(b.extent(2)) * es;
    g.rows = uint32_t(b.extent(1));
    g.planes = uint32_t(b.extent(0));
    g.src_row_stride = uint64_t(sn2) * es;
    g.dst_row_stride = uint64_t(dn2) * es;
    g.src_plane_stride = uint64_t(sn1 * sn2) * es;
    g.dst_plane_stride = uint64_t(dn1 * dn2) * es;
    if (g.row_bytes == g.src_row_stride && g.row_bytes == g.dst_row_stride) {
        g.row_bytes *= g.rows;
        g.rows = 1;
        if (g.row_bytes == g.src_plane_stride && g.row_bytes == g.dst_plane_stride) {
            g.row_bytes *= g.planes;
            g.planes = 1;
        }
    }
    uint64_t a = uintptr_t(g.src) | uintptr_t(g.dst) | g.row_bytes;
    if (g.rows > 1) a |= g.src_row_stride | g.dst_row_stride;
    if (g.planes > 1) a |= g.src_plane_stride | g.dst_plane_stride;
    g.vec = (a & 15) == 0 ? 16 : (a & 7) == 0 ? 8 : (a & 3) == 0 ? 4 : (a & 1) == 0 ? 2 : 1;
    g.units_begin = args.total_units;
    const uint64_t units = seg_units(g);
    args.seg[args.nseg++] = g;
    args.total_units += units;
}
}  // namespace

void Communicator::add_pilot(const Pilot& p) {
    std::lock_guard<std::mutex> l(m_);
    pilots_[Key{p.receiver, p.transfer, p.buffer}].push_back(PilotRec{p.sender, p.msg, p.box});
    cv_.notify_all();
}

void Communicator::post_send(int node, uint64_t msg, const Mem& src, cudaEvent_t ready) {
    std::lock_guard<std::mutex> l(m_);
    sends_[{node, msg}] = Send{src, ready};
    cv_.notify_all();
}

void Communicator::abort() {
    std::lock_guard<std::mutex> l(m_);
    abort_ = true;
    cv_.notify_all();
}

int Communicator::pull_region(int node, int64_t tid, uint32_t buf, const Region& reg, const Mem& dst,
                              cudaStream_t stream) {
    std::unique_lock<std::mutex> l(m_);
    const Key k{node, tid, buf};
    const uint64_t need = rvolume(reg);
    // wait until the pilots covering reg are known and their sends issued
    // (pilots of one transfer are disjoint and tile the awaited region)
    for (;;) {
        if (abort_) return E_STATE;
        uint64_t covered = 0;
        bool posted = true;
        auto it = pilots_.find(k);
        if (it != pilots_.end())
            for (const PilotRec& p : it->second) {
                const uint64_t v = rvolume(rinter(Region{p.box}, reg));
                if (!v) continue;
                covered += v;
                if (!p.pulled && !sends_.count({p.sender, p.msg})) posted = false;
            }
        if (covered >= need && posted) break;
        cv_.wait(l);
    }
    for (PilotRec& p : pilots_[k]) {
        if (p.pulled || rinter(Region{p.box}, reg).empty()) continue;
        auto sit = sends_.find({p.sender, p.msg});
        Send snd = sit->second;
        sends_.erase(sit);
        cudaStreamWaitEvent(stream, snd.ready, 0);           // the sender's staged data
        cudaEventDestroy(snd.ready);
        CopyArgs args;
        args.nseg = 0;
        args.total_units = 0;
        args.peer = 0;
        box_seg(args, snd.src.base, snd.src.box, dst.base, dst.box, p.box, dst.es);
        launch_copy(args, stream);
        cudaEvent_t done = nullptr;
        cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
        cudaEventRecord(done, stream);
        pulled_[{p.sender, p.msg}] = done;
        p.pulled = true;
        pulls_++;
        pull_bytes_ += uint64_t(p.box.volume()) * dst.es;
    }
    cv_.notify_all();
    return cudaGetLastError() == cudaSuccess ? E_OK : E_CUDA;
}

cudaEvent_t Communicator::wait_pulled(int node, uint64_t msg) {
    std::unique_lock<std::mutex> l(m_);
    for (;;) {
        auto it = pulled_.find({node, msg});
        if (it != pulled_.end()) {
            cudaEvent_t e = it->second;
            pulled_.erase(it);
            return e;
        }
        if (abort_) return nullptr;
        cv_.wait(l);
    }
}

// Send / receive / split receive / await receive (virtual-node mode, Table 1).
void Executor::exec_transfer(const Instr& ins) {
    Communicator& comm = *cfg_.comm;
    const Token deps = local_part(ins.deps);
    const uint32_t es = bufinfo_.at(ins.buffer).es;
    set_dev(0);
    const int s_sync = S_SYNC, s_recv = S_SIG0;          // streams of the node's first device
    const int64_t key = (ins.transfer << 20) ^ int64_t(ins.buffer);
    auto mem = [&](int64_t aid) {
        const AllocRec& a = allocs_.at(aid);
        return Communicator::Mem{base_of(a), a.box, es};
    };
    auto pull = [&](const Region& reg, const Communicator::Mem& dst) {
        wait_token(s_recv, deps);                         // the receive's own dependencies (M1 readers, writers)
        const int rc = comm.pull_region(cfg_.node, ins.transfer, ins.buffer, reg, dst, streams_[s_recv].s);
        if (rc != E_OK && !err_) {
            errmsg_ = "receive arbitration failed";
            err_ = rc;
        }
        return record(s_recv);
    };
    switch (ins.kind) {
    case IKind::Send: {
        wait_token(s_sync, deps);                         // the staging copy (or, elided, its inputs)
        cudaEvent_t ready = nullptr;
        check(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "cudaEventCreate");
        check(cudaEventRecord(ready, streams_[s_sync].s), "cudaEventRecord");
        // device-direct: one elided copy staged the whole box -> publish the
        // device allocation it came from; the receiver pulls over NVLink
        Communicator::Mem src = mem(ins.src_aid);
        auto sg = staged_.find(direct_staged_);
        if (direct_src_ >= 0 && sg != staged_.end()) {
            src = mem(direct_src_);
            sg->second.consumed = true;
            pending_send_[direct_staged_].push_back(ins.msg);   // readers of the source: after the pull
        }
        comm.post_send(cfg_.node, ins.msg, src, ready);
        pending_send_[ins.iid].push_back(ins.msg);        // completes with the receiver's pull
        st_.bytes_copy[5] += uint64_t(ins.box.volume()) * es;
        break;
    }
    case IKind::Receive:
        tok_[ins.iid] = pull(ins.region, mem(ins.dst_aid));
        break;
    case IKind::SplitReceive:
        recv_dst_[key] = mem(ins.dst_aid);
        tok_[ins.iid] = deps;
        break;
    case IKind::AwaitReceive: {
        auto it = recv_dst_.find(key);
        if (it == recv_dst_.end()) {
            errmsg_ = "await receive without its split receive";
            err_ = E_STATE;
            return;
        }
        tok_[ins.iid] = pull(ins.region, it->second);
        break;
    }
    default:
        break;
    }
}

// A send completes when the receiver has pulled its box: resolved when an
// instruction depending on it is issued (blocking until the receiver has
// issued the pull -- it only waits for sends of this or earlier tasks).
void Executor::resolve_sends(const Instr& ins) {
    for (uint64_t j : ins.deps) {
        auto it = pending_send_.find(j);
        if (it == pending_send_.end()) continue;
        // another send of an elided staging copy's bytes needs only the copy's
        // inputs (its token until resolved), not the first send's pull: waiting
        // for that pull could deadlock when both go to one receiver, whose
        // receive waits for every send of its region to be posted
        // an elided staging copy waits for the pulls that read its source
        // allocation only for instructions that may write that allocation:
        // sends, receives and copies into M1 need the copy's inputs (its token),
        // and waiting for a pull there could deadlock when the receiver's
        // receive waits for a send this node posts later
        if (elided_iids_.count(j) && (ins.kind == IKind::Send || ins.kind == IKind::Receive ||
                                       ins.kind == IKind::SplitReceive || ins.kind == IKind::AwaitReceive ||
                                       (ins.kind == IKind::Copy && ins.dst_mem == 1)))
            continue;
        const std::vector<uint64_t> msgs = it->second;
        pending_send_.erase(it);
        Token t = tok_.count(j) ? tok_[j] : Token{};
        for (uint64_t msg : msgs) {
            auto mt = msg_tok_.find(msg);
            if (mt == msg_tok_.end()) {
                cudaEvent_t e = cfg_.comm->wait_pulled(cfg_.node, msg);
                if (!e) {
                    if (!err_) {
                        errmsg_ = "communicator aborted";
                        err_ = E_STATE;
                    }
                    return;
                }
                const int sidx = S_HSIG;                  // device 0 of the node
                set_dev(0);
                check(cudaStreamWaitEvent(streams_[sidx].s, e, 0), "cudaStreamWaitEvent");
                cudaEventDestroy(e);
                mt = msg_tok_.emplace(msg, record(sidx)).first;
            }
            merge(t, mt->second);
        }
        tok_[j] = t;
    }
}

// Before `ins` runs (device-direct sends): readers of M1 bytes that an elided
// staging copy would have written are found by allocation and region -- not
// by dependencies, which horizons subsume (R7) -- and either go device-direct
// (a send whose whole box one elided copy staged) or get those copies
// executed first.  Before an allocation is freed, the elided copies sourced
// from it are executed (a later send of the same, still up-to-date M1 bytes
// must find them there).  Writes into M1 shrink the elided copies' regions.
void Executor::settle_staged(const Instr& ins) {
    direct_src_ = -1;
    direct_staged_ = 0;
    settle_tok_ = Token{};
    int64_t m1_read = -1;
    Region rd;
    if (ins.kind == IKind::Send) {
        m1_read = ins.src_aid;
        rd = Region{ins.box};
    } else if (ins.kind == IKind::Copy && ins.src_mem == 1) {
        m1_read = ins.src_aid;
        rd = ins.region;
    }
    std::vector<uint64_t> todo;
    if (m1_read >= 0) {
        for (auto& kv : staged_) {
            const Staged& e = kv.second;
            if (e.ins.dst_aid != m1_read || rinter(e.ins.region, rd).empty()) continue;
            bool whole = false;
            if (ins.kind == IKind::Send)
                for (const Box& b : e.ins.region) whole = whole || b.contains(ins.box);
            if (whole && direct_src_ < 0) {
                direct_src_ = e.ins.src_aid;
                direct_staged_ = kv.first;
            } else {
                todo.push_back(kv.first);
            }
        }
        if (!todo.empty() && direct_src_ >= 0) {            // mixed: the send reads M1 after all
            todo.push_back(direct_staged_);
            direct_src_ = -1;
            direct_staged_ = 0;
        }
    }
    if (ins.kind == IKind::Free)
        for (auto& kv : staged_)
            if (kv.second.ins.src_aid == ins.aid) todo.push_back(kv.first);
    std::sort(todo.begin(), todo.end());
    todo.erase(std::unique(todo.begin(), todo.end()), todo.end());
    for (uint64_t j : todo) materialize_staged(j);
    int64_t m1 = -1;
    if (ins.kind == IKind::Copy && ins.dst_mem == 1) m1 = ins.dst_aid;
    if (ins.kind == IKind::Receive || ins.kind == IKind::SplitReceive) m1 = ins.dst_aid;
    if (ins.kind == IKind::Free) m1 = ins.aid;
    if (m1 < 0) return;
    for (auto it = staged_.begin(); it != staged_.end();) {
        Staged& e = it->second;
        if (e.ins.dst_aid != m1 || it->first == ins.iid) {
            ++it;
            continue;
        }
        if (ins.kind != IKind::Free) e.ins.region = rdiff(e.ins.region, ins.region);
        it = (ins.kind == IKind::Free || e.ins.region.empty()) ? staged_.erase(it) : std::next(it);
    }
}

void Executor::materialize_staged(uint64_t iid) {
    auto it = staged_.find(iid);
    if (it == staged_.end()) return;
    const Instr c = it->second.ins;
    staged_.erase(it);
    const Token before = tok_.count(iid) ? tok_[iid] : Token{};
    const Instr* saved = cur_ins_;
    cur_ins_ = &c;
    materializing_ = true;
    exec_copy(c);                                         // really copies this time
    materializing_ = false;
    cur_ins_ = saved;
    Token t = tok_[iid];
    merge(settle_tok_, t);                                // e.g. a free of the source waits for it
    merge(t, before);                                     // e.g. the pull that read the source
    tok_[iid] = t;
    st_.staging_materialized++;
}

}  // namespace cel
