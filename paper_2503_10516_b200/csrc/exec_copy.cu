// Executor: copy instructions (Table 1 `copy`):
// copy kernels between allocations, DMA to / from host memory, host copies.
#include "exec_impl.hpp"

namespace cel {

// Copies between host-side memories (M0 host data / user pointer and the M1
// staging arena): plain host copies once the dependencies have completed.
void Executor::exec_host_copy(const Instr& ins, const Token& deps) {
    const uint32_t es = bufinfo_.at(ins.buffer).es;
    for (const TokEntry& e : deps.local)
        if (e.seq > streams_[e.stream].done) check(cudaEventSynchronize(e.ev), "host copy wait");
    const char* sb;
    Box sbox;
    if (ins.src_mem == 1) {
        const AllocRec& S = allocs_.at(ins.src_aid);
        sb = base_of(S);
        sbox = S.box;
    } else {
        auto hi = host_init_.find(ins.buffer);
        if (hi == host_init_.end()) {
            errmsg_ = "host copy of a buffer without host data";
            err_ = E_STATE;
            return;
        }
        sb = hi->second.first;
        sbox = bufinfo_.at(ins.buffer).extent;
    }
    char* db;
    Box dbox;
    if (ins.dst_aid == USER_AID) {
        auto rb = readbacks_.find(ins.readback);
        if (rb == readbacks_.end()) {
            errmsg_ = "readback copy without a destination";
            err_ = E_STATE;
            return;
        }
        db = rb->second.dst;
        dbox = rb->second.box;
    } else {
        const AllocRec& D = allocs_.at(ins.dst_aid);
        db = base_of(D);
        dbox = D.box;
    }
    for (const Box& b : ins.region)
        for (int64_t z = b.lo[0]; z < b.hi[0]; ++z)
            for (int64_t y = b.lo[1]; y < b.hi[1]; ++y) {
                const int64_t so = ((z - sbox.lo[0]) * sbox.extent(1) + (y - sbox.lo[1])) * sbox.extent(2) +
                                   (b.lo[2] - sbox.lo[2]);
                const int64_t dof = ((z - dbox.lo[0]) * dbox.extent(1) + (y - dbox.lo[1])) * dbox.extent(2) +
                                    (b.lo[2] - dbox.lo[2]);
                memcpy(db + dof * es, sb + so * es, size_t(b.extent(2)) * es);
            }
    st_.bytes_copy[5] += rvolume(ins.region) * es;
    tok_[ins.iid] = Token{};
}

// Strided boxes (rows at a pitch, or one row per plane) of a copy between
// device allocations of one GPU by TMA tensor maps (north_star "TMA tensor-map
// box loads and stores for 2D/3D strided regions"; SASS UTMALDG / UTMASTG).
// All-or-nothing per instruction: false (nothing launched) if any box is one
// contiguous run or not expressible, and the LSU copy kernel takes it.
bool Executor::exec_copy_tma(const Instr& ins, const AllocRec& S, const AllocRec& D, uint32_t es, int sidx, int dev) {
    std::vector<TmaBox> boxes;
    for (const Box& b : ins.region) {
        TmaBox t;
        t.src = base_of(S);
        t.dst = base_of(D);
        t.es = es;
        for (int k = 0; k < 3; ++k) {
            t.sn[k] = S.box.extent(k);
            t.dn[k] = D.box.extent(k);
            t.so[k] = b.lo[k] - S.box.lo[k];
            t.dof[k] = b.lo[k] - D.box.lo[k];
            t.ext[k] = b.extent(k);
        }
        boxes.push_back(t);
    }
    std::vector<TmaCopyArgs> launches(1);
    memset(&launches.back(), 0, sizeof(TmaCopyArgs));
    for (const TmaBox& t : boxes) {
        int r = tma_copy_add(launches.back(), t);
        if (r == 0 && launches.back().nseg == kMaxTmaSegs) {
            launches.emplace_back();
            memset(&launches.back(), 0, sizeof(TmaCopyArgs));
            r = tma_copy_add(launches.back(), t);
        }
        if (r != 1) return false;                 // a contiguous run or not expressible: LSU for the instruction
    }
    for (const TmaCopyArgs& a : launches) {
        if (cfg_.profile && prof_sample(K_NUM)) {
            Prof p{K_NUM, prof_event(dev), prof_event(dev), dev, ins.iid, sidx, now_ns()};
            cudaEventRecord(p.a, streams_[sidx].s);
            st_.kernel_launches += launch_copy_tma(a, streams_[sidx].s);
            cudaEventRecord(p.b, streams_[sidx].s);
            prof_pending_.push_back(p);
        } else {
            st_.kernel_launches += launch_copy_tma(a, streams_[sidx].s);
        }
        st_.copy_launches++;
        st_.tma_copy_launches++;
    }
    st_.bytes_copy[ins.reason == REASON_RESIZE ? 0 : 1] += rvolume(ins.region) * es;
    return true;
}

void Executor::exec_copy(const Instr& ins) {
    const uint32_t es = bufinfo_.at(ins.buffer).es;
    Token deps;
    for (uint64_t j : ins.deps) {
        // a copy that reads only rows a split kernel wrote in its shell launch
        // waits for that launch, not for the interior (computation /
        // communication overlap)
        auto pit = parts_.find(j);
        if (pit != parts_.end() && pit->second.write_aid == ins.src_aid && ins.src_mem >= 2 &&
            std::find(pit->second.bound.begin(), pit->second.bound.end(), ins.dst_aid) == pit->second.bound.end()) {
            bool touches = false;
            for (const Box& b : ins.region)
                if (!intersect(b, pit->second.interior).empty()) touches = true;
            if (!touches) {
                merge(deps, pit->second.shell);
                continue;
            }
        }
        merge(deps, dep_token(j));
    }
    if (direct_sends_ && !materializing_ && ins.src_mem >= 2 && ins.dst_mem == 1 && ins.reason == REASON_COHERENCE &&
        ins.src_aid >= 0) {
        // a push's staging copy: elided; its sends publish the device
        // allocation (settle_staged / exec_transfer)
        staged_[ins.iid] = Staged{ins, deps, false};
        elided_iids_.insert(ins.iid);
        tok_[ins.iid] = deps;
        st_.staging_elided++;
        return;
    }
    if (ins.src_mem >= 1 && ins.dst_mem >= 1) {
        // allocation to allocation: device memories, or the pinned + mapped M1
        // staging arena of virtual-node mode on either side (copy kernel)
        const AllocRec& S = allocs_.at(ins.src_aid);
        const AllocRec& D = allocs_.at(ins.dst_aid);
        if (S.dev == D.dev && base_of(S) == base_of(D) && S.box.lo[0] == D.box.lo[0] && S.box.lo[1] == D.box.lo[1] &&
            S.box.lo[2] == D.box.lo[2] && S.box.extent(1) == D.box.extent(1) && S.box.extent(2) == D.box.extent(2)) {
            // in-place growth: source and destination bytes coincide.  The
            // copy's token is its dependencies'; a long one (other ranks'
            // flags pile up along a chain of elided copies) folds into one
            // event, or every later merge of it grows with the program
            st_.copies_elided++;
            st_.bytes_elided += rvolume(ins.region) * es;
            if (deps.remote.size() > 8 || deps.local.size() > 16) deps = materialize(S.dev >= 0 ? S.dev : D.dev, deps);
            tok_[ins.iid] = deps;
            return;
        }
        const int dev = S.dev >= 0 ? S.dev : (D.dev >= 0 ? D.dev : 0);
        const bool peer = S.dev >= 0 && D.dev >= 0 && S.dev != D.dev;
        const int sidx = dev * kStreamsPerDev + (peer ? S_PUSH : S_COPY);
        set_dev(dev);
        wait_token(sidx, deps);
        const char* sb = base_of(S);
        char* db = base_of(D);
        CopyArgs args;
        args.nseg = 0;
        args.total_units = 0;
        // peer: the destination is another GPU's memory (NVLink push).  CEL_FORCE_PEER=1
        // treats distinct virtual devices of one GPU the same way (DMA plan and the
        // fenced peer copy kernel), so one-GPU tests cover that path
        args.peer = peer && (phys_[S.dev] != phys_[D.dev] || force_peer_) ? 1 : 0;
        const int64_t sn1 = S.box.extent(1), sn2 = S.box.extent(2);
        const int64_t dn1 = D.box.extent(1), dn2 = D.box.extent(2);
        if (args.peer && peer_dma_) {
            // small pushes to another GPU on a copy engine (DMA): no SM time taken
            // from the running stencil.  Each box must be one byte run in both
            // allocations, or one run per row at a constant pitch in each
            // (a 2-D copy: e.g. a y-face of a 3-D halo, 256 rows of 4 KiB)
            struct Dma {
                int64_t so, dof;
                size_t width, height, spitch, dpitch;
            };
            SmallVec<Dma, 4> plan;
            bool ok = ins.region.size() <= 4;
            uint64_t total = 0;
            for (const Box& b : ins.region) {
                if (!ok) break;
                Dma m;
                m.so = ((b.lo[0] - S.box.lo[0]) * sn1 + (b.lo[1] - S.box.lo[1])) * sn2 + (b.lo[2] - S.box.lo[2]);
                m.dof = ((b.lo[0] - D.box.lo[0]) * dn1 + (b.lo[1] - D.box.lo[1])) * dn2 + (b.lo[2] - D.box.lo[2]);
                const bool cs = b.extent(2) == sn2 && (b.extent(1) == sn1 || b.extent(0) == 1);
                const bool cd = b.extent(2) == dn2 && (b.extent(1) == dn1 || b.extent(0) == 1);
                if ((cs && cd) || (b.extent(0) == 1 && b.extent(1) == 1)) {
                    m.width = size_t(b.volume()) * es;       // one run
                    m.height = 1;
                    m.spitch = m.dpitch = m.width;
                } else if (b.extent(0) == 1) {                // rows of one plane
                    m.width = size_t(b.extent(2)) * es;
                    m.height = size_t(b.extent(1));
                    m.spitch = size_t(sn2) * es;
                    m.dpitch = size_t(dn2) * es;
                } else if (b.extent(1) == 1) {                // one row per plane
                    m.width = size_t(b.extent(2)) * es;
                    m.height = size_t(b.extent(0));
                    m.spitch = size_t(sn1 * sn2) * es;
                    m.dpitch = size_t(dn1 * dn2) * es;
                } else {
                    ok = false;
                }
                // cudaMemcpy2DAsync rejects pitches above the device limit: those boxes
                // stay on the copy kernel instead of poisoning the runtime
                if (m.height > 1 && (m.spitch > max_pitch_ || m.dpitch > max_pitch_ || m.width > max_pitch_)) ok = false;
                // narrow rows (a column halo of a 2-D tile: one element per row)
                // are a descriptor per row for the copy engine: the copy kernel
                // moves them a thread per row
                if (m.height > 1 && m.width < 512) ok = false;
                plan.push_back(m);
                total += b.volume() * es;
            }
            if (ok && total <= peer_dma_max_) {
                for (const Dma& m : plan) {
                    if (m.height == 1)
                        check(cudaMemcpyAsync(db + m.dof * es, sb + m.so * es, m.width, cudaMemcpyDeviceToDevice,
                                              streams_[sidx].s),
                              "cudaMemcpyAsync (peer DMA)");
                    else
                        check(cudaMemcpy2DAsync(db + m.dof * es, m.dpitch, sb + m.so * es, m.spitch, m.width, m.height,
                                                cudaMemcpyDeviceToDevice, streams_[sidx].s),
                              "cudaMemcpy2DAsync (peer DMA)");
                    st_.memcpy_calls++;
                }
                st_.bytes_copy[2] += total;
                tok_[ins.iid] = record(sidx);
                return;
            }
        }
        uint64_t bytes = 0;
        if (tma_copy_ && !args.peer && S.dev >= 0 && D.dev >= 0 && exec_copy_tma(ins, S, D, es, sidx, dev)) {
            tok_[ins.iid] = record(sidx);
            return;
        }
        auto flush = [&]() {
            if (args.nseg == 0) return;
            if (cfg_.profile && prof_sample(args.peer ? K_NUM + 1 : K_NUM)) {
                Prof p{args.peer ? K_NUM + 1 : K_NUM, prof_event(dev), prof_event(dev), dev, ins.iid, sidx, now_ns()};
                cudaEventRecord(p.a, streams_[sidx].s);
                st_.kernel_launches += launch_copy(args, streams_[sidx].s);
                cudaEventRecord(p.b, streams_[sidx].s);
                prof_pending_.push_back(p);
            } else {
                st_.kernel_launches += launch_copy(args, streams_[sidx].s);
            }
            st_.copy_launches++;
            args.nseg = 0;
            args.total_units = 0;
        };
        for (const Box& b : ins.region) {
            CopySeg g;
            const int64_t so = ((b.lo[0] - S.box.lo[0]) * sn1 + (b.lo[1] - S.box.lo[1])) * sn2 + (b.lo[2] - S.box.lo[2]);
            const int64_t dof = ((b.lo[0] - D.box.lo[0]) * dn1 + (b.lo[1] - D.box.lo[1])) * dn2 + (b.lo[2] - D.box.lo[2]);
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

            // huge planes x rows: split so that units stay below 2^63 (never in practice)
            if (args.nseg == kMaxSegs) flush();
            g.units_begin = args.total_units;
            args.seg[args.nseg++] = g;
            args.total_units += seg_units(args.seg[args.nseg - 1]);
            bytes += b.volume() * es;
        }
        flush();
        const int kind = ins.reason == REASON_RESIZE ? 0 : (args.peer ? 2 : 1);
        st_.bytes_copy[kind] += bytes;
        tok_[ins.iid] = record(sidx);
        return;
    }
    // host <-> device: DMA (cudaMemcpy3DAsync per box)
    const bool h2d = ins.src_mem == 0 && ins.dst_mem >= 2;
    const bool d2h = ins.src_mem >= 2 && ins.dst_aid == USER_AID;
    if (!h2d && !d2h && (ins.src_mem == 1 || ins.dst_mem == 1)) {
        exec_host_copy(ins, deps);           // M1 <-> M0 / user pointer (virtual-node mode)
        return;
    }
    if (!h2d && !d2h) {
        // host implicit allocation -> user pointer: plain host copy
        auto hi = host_init_.find(ins.buffer);
        auto rb = readbacks_.find(ins.readback);
        if (hi == host_init_.end() || rb == readbacks_.end()) {
            errmsg_ = "host copy without source or destination";
            err_ = E_STATE;
            return;
        }
        const Box E = bufinfo_.at(ins.buffer).extent;
        const Box& R = rb->second.box;
        for (const Box& b : ins.region)
            for (int64_t z = b.lo[0]; z < b.hi[0]; ++z)
                for (int64_t y = b.lo[1]; y < b.hi[1]; ++y) {
                    const int64_t so = ((z * E.extent(1)) + y) * E.extent(2) + b.lo[2];
                    const int64_t dof = (((z - R.lo[0]) * R.extent(1)) + (y - R.lo[1])) * R.extent(2) + (b.lo[2] - R.lo[2]);
                    memcpy(rb->second.dst + dof * es, hi->second.first + so * es, size_t(b.extent(2)) * es);
                }
        st_.bytes_copy[5] += rvolume(ins.region) * es;
        tok_[ins.iid] = Token{};
        return;
    }
    const int dev = h2d ? ins.dst_mem - 2 : ins.src_mem - 2;
    const int sidx = dev * kStreamsPerDev + S_COPY;
    set_dev(dev);
    wait_token(sidx, deps);
    char* hbase;
    Box hbox;
    char* dbase;
    Box dbox;
    if (h2d) {
        auto hi = host_init_.find(ins.buffer);
        if (hi == host_init_.end()) {
            errmsg_ = "H2D copy of a buffer without host data";
            err_ = E_STATE;
            return;
        }
        hbase = hi->second.first;
        hbox = bufinfo_.at(ins.buffer).extent;
        const AllocRec& D = allocs_.at(ins.dst_aid);
        dbase = base_of(D);
        dbox = D.box;
    } else {
        auto rb = readbacks_.find(ins.readback);
        if (rb == readbacks_.end()) {
            errmsg_ = "readback copy without a destination";
            err_ = E_STATE;
            return;
        }
        hbase = rb->second.dst;
        hbox = rb->second.box;
        const AllocRec& S = allocs_.at(ins.src_aid);
        dbase = base_of(S);
        dbox = S.box;
    }
    for (const Box& b : ins.region) {
        // DMA: collapse to one linear copy when the box is contiguous in both
        // layouts (full rows / planes), else a 2-D copy per plane, else 3-D
        const size_t hrow = size_t(hbox.extent(2)) * es, drow = size_t(dbox.extent(2)) * es;
        const size_t width = size_t(b.extent(2)) * es;
        auto hoff = [&](int64_t z, int64_t y) {
            return ((size_t(z - hbox.lo[0]) * size_t(hbox.extent(1)) + size_t(y - hbox.lo[1])) * hrow) +
                   size_t(b.lo[2] - hbox.lo[2]) * es;
        };
        auto doff = [&](int64_t z, int64_t y) {
            return ((size_t(z - dbox.lo[0]) * size_t(dbox.extent(1)) + size_t(y - dbox.lo[1])) * drow) +
                   size_t(b.lo[2] - dbox.lo[2]) * es;
        };
        char* hp0 = hbase + hoff(b.lo[0], b.lo[1]);
        char* dp0 = dbase + doff(b.lo[0], b.lo[1]);
        const bool rows_contig = width == hrow && width == drow;
        const bool planes_contig = rows_contig && b.extent(1) == hbox.extent(1) && b.extent(1) == dbox.extent(1);
        const cudaStream_t st = streams_[sidx].s;
        if (planes_contig || (rows_contig && b.extent(0) == 1)) {
            const size_t bytes = width * size_t(b.extent(1)) * size_t(b.extent(0));
            check(h2d ? cudaMemcpyAsync(dp0, hp0, bytes, cudaMemcpyHostToDevice, st)
                      : cudaMemcpyAsync(hp0, dp0, bytes, cudaMemcpyDeviceToHost, st),
                  "cudaMemcpyAsync");
            st_.memcpy_calls++;
            continue;
        }
        if (b.extent(0) == 1) {
            check(h2d ? cudaMemcpy2DAsync(dp0, drow, hp0, hrow, width, size_t(b.extent(1)), cudaMemcpyHostToDevice, st)
                      : cudaMemcpy2DAsync(hp0, hrow, dp0, drow, width, size_t(b.extent(1)), cudaMemcpyDeviceToHost, st),
                  "cudaMemcpy2DAsync");
            st_.memcpy_calls++;
            continue;
        }
        cudaMemcpy3DParms p;
        memset(&p, 0, sizeof p);
        cudaPitchedPtr hp = make_cudaPitchedPtr(hbase, hrow, hrow, size_t(hbox.extent(1)));
        cudaPitchedPtr dp = make_cudaPitchedPtr(dbase, drow, drow, size_t(dbox.extent(1)));
        cudaPos hpos = make_cudaPos(size_t(b.lo[2] - hbox.lo[2]) * es, size_t(b.lo[1] - hbox.lo[1]),
                                    size_t(b.lo[0] - hbox.lo[0]));
        cudaPos dpos = make_cudaPos(size_t(b.lo[2] - dbox.lo[2]) * es, size_t(b.lo[1] - dbox.lo[1]),
                                    size_t(b.lo[0] - dbox.lo[0]));
        if (h2d) {
            p.srcPtr = hp;
            p.srcPos = hpos;
            p.dstPtr = dp;
            p.dstPos = dpos;
            p.kind = cudaMemcpyHostToDevice;
        } else {
            p.srcPtr = dp;
            p.srcPos = dpos;
            p.dstPtr = hp;
            p.dstPos = hpos;
            p.kind = cudaMemcpyDeviceToHost;
        }
        p.extent = make_cudaExtent(width, size_t(b.extent(1)), size_t(b.extent(0)));
        check(cudaMemcpy3DAsync(&p, st), "cudaMemcpy3DAsync");
        st_.memcpy_calls++;
    }
    st_.bytes_copy[h2d ? 3 : 4] += rvolume(ins.region) * es;
    tok_[ins.iid] = record(sidx);
}

}  // namespace cel
