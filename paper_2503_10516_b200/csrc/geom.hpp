// Box / Region / RegionMap for the host scheduler.
//
// Paper basis: buffer state is tracked per "subregion" (§3.3) and
// transfers per "rectangular region" (§3.4).  Representation follows
// DESIGN.md R1-R3: half-open 3-D boxes (unused dims [0,1)), regions as
// disjoint boxes in maximal-slab canonical form (dim 0 cut exactly where the
// (dim1, dim2) cross-section changes, recursively; sorted by min), region
// maps as value -> canonical region.
#pragma once

#include <algorithm>
#include <initializer_list>
#include <cstdint>
#include <utility>
#include <vector>

namespace cel {

struct Box {
    int64_t lo[3] = {0, 0, 0};
    int64_t hi[3] = {0, 0, 0};

    static Box make(const int64_t* l, const int64_t* h) {
        Box b;
        for (int d = 0; d < 3; ++d) { b.lo[d] = l[d]; b.hi[d] = h[d]; }
        return b.normalized();
    }
    bool empty() const { return hi[0] <= lo[0] || hi[1] <= lo[1] || hi[2] <= lo[2]; }
    Box normalized() const { return empty() ? Box{} : *this; }
    int64_t extent(int d) const { return hi[d] - lo[d]; }
    uint64_t volume() const {
        return empty() ? 0 : uint64_t(hi[0] - lo[0]) * uint64_t(hi[1] - lo[1]) * uint64_t(hi[2] - lo[2]);
    }
    bool operator==(const Box& o) const {
        for (int d = 0; d < 3; ++d)
            if (lo[d] != o.lo[d] || hi[d] != o.hi[d]) return false;
        return true;
    }
    bool operator!=(const Box& o) const { return !(*this == o); }
    bool contains(const Box& in) const {
        if (in.empty()) return true;
        if (empty()) return false;
        for (int d = 0; d < 3; ++d)
            if (in.lo[d] < lo[d] || in.hi[d] > hi[d]) return false;
        return true;
    }
    Box with_dim(int d, int64_t l, int64_t h) const {
        Box b = *this;
        b.lo[d] = l;
        b.hi[d] = h;
        return b;
    }
};

inline bool lex_less(const Box& a, const Box& b) {
    for (int d = 0; d < 3; ++d)
        if (a.lo[d] != b.lo[d]) return a.lo[d] < b.lo[d];
    for (int d = 0; d < 3; ++d)
        if (a.hi[d] != b.hi[d]) return a.hi[d] < b.hi[d];
    return false;
}

inline Box intersect(const Box& a, const Box& b) {
    Box r;
    for (int d = 0; d < 3; ++d) {
        r.lo[d] = std::max(a.lo[d], b.lo[d]);
        r.hi[d] = std::min(a.hi[d], b.hi[d]);
    }
    return r.normalized();
}

// a and b share a point (both non-empty): the intersection test of the hot
// scans, without building the intersection
inline bool overlaps(const Box& a, const Box& b) {
    return a.lo[0] < b.hi[0] && b.lo[0] < a.hi[0] && a.lo[1] < b.hi[1] && b.lo[1] < a.hi[1] && a.lo[2] < b.hi[2] &&
           b.lo[2] < a.hi[2] && !a.empty() && !b.empty();
}

inline Box bbox(const Box& a, const Box& b) {
    if (a.empty()) return b.normalized();
    if (b.empty()) return a;
    Box r;
    for (int d = 0; d < 3; ++d) {
        r.lo[d] = std::min(a.lo[d], b.lo[d]);
        r.hi[d] = std::max(a.hi[d], b.hi[d]);
    }
    return r;
}

// Small vector with inline storage: most regions on the hot path hold 1-3
// boxes, so region algebra should not touch the heap.
template <class T, unsigned N>
class SmallVec {
public:
    using value_type = T;
    using iterator = T*;
    using const_iterator = const T*;
    SmallVec() = default;
    SmallVec(std::initializer_list<T> il) {
        reserve(il.size());
        for (const T& x : il) push_back(x);
    }
    template <class It, class = decltype(*std::declval<It>())>
    SmallVec(It b, It e) {
        for (; b != e; ++b) push_back(*b);
    }
    SmallVec(const SmallVec& o) {
        reserve(o.n_);
        for (unsigned i = 0; i < o.n_; ++i) data()[i] = o.data()[i];
        n_ = o.n_;
    }
    SmallVec(SmallVec&& o) noexcept { steal(o); }
    SmallVec& operator=(const SmallVec& o) {
        if (this != &o) {
            n_ = 0;
            reserve(o.n_);
            for (unsigned i = 0; i < o.n_; ++i) data()[i] = o.data()[i];
            n_ = o.n_;
        }
        return *this;
    }
    SmallVec& operator=(SmallVec&& o) noexcept {
        if (this != &o) {
            release();
            steal(o);
        }
        return *this;
    }
    ~SmallVec() { release(); }
    T* data() { return heap_ ? heap_ : reinterpret_cast<T*>(buf_); }
    const T* data() const { return heap_ ? heap_ : reinterpret_cast<const T*>(buf_); }
    T* begin() { return data(); }
    T* end() { return data() + n_; }
    const T* begin() const { return data(); }
    const T* end() const { return data() + n_; }
    size_t size() const { return n_; }
    bool empty() const { return n_ == 0; }
    T& operator[](size_t i) { return data()[i]; }
    const T& operator[](size_t i) const { return data()[i]; }
    T& back() { return data()[n_ - 1]; }
    const T& back() const { return data()[n_ - 1]; }
    void clear() { n_ = 0; }
    void reserve(size_t c) {
        if (c <= cap_) return;
        unsigned nc = cap_ * 2;
        if (nc < c) nc = unsigned(c);
        T* h = static_cast<T*>(::operator new(sizeof(T) * nc));
        for (unsigned i = 0; i < n_; ++i) h[i] = data()[i];
        if (heap_) ::operator delete(heap_);
        heap_ = h;
        cap_ = nc;
    }
    void push_back(const T& x) {
        if (n_ == cap_) reserve(n_ + 1);
        data()[n_++] = x;
    }
    template <class It>
    void insert(T* pos, It b, It e) {  // append only (pos == end())
        (void)pos;
        for (; b != e; ++b) push_back(*b);
    }
    T* insert_at(T* pos, const T& x) {
        const size_t i = size_t(pos - data());
        push_back(x);
        T* d = data();
        for (size_t k = n_ - 1; k > i; --k) d[k] = d[k - 1];
        d[i] = x;
        return d + i;
    }
    bool operator<(const SmallVec& o) const {
        return std::lexicographical_compare(begin(), end(), o.begin(), o.end());
    }
    T* erase(T* first, T* last) {
        T* d = data();
        const size_t f = size_t(first - d), l = size_t(last - d);
        for (size_t i = l; i < n_; ++i) d[f + i - l] = d[i];
        n_ -= unsigned(l - f);
        return d + f;
    }
    void swap(SmallVec& o) {
        SmallVec t(std::move(o));
        o = std::move(*this);
        *this = std::move(t);
    }
    bool operator==(const SmallVec& o) const {
        if (n_ != o.n_) return false;
        for (unsigned i = 0; i < n_; ++i)
            if (!(data()[i] == o.data()[i])) return false;
        return true;
    }
    bool operator!=(const SmallVec& o) const { return !(*this == o); }

private:
    void release() {
        if (heap_) ::operator delete(heap_);
        heap_ = nullptr;
        cap_ = N;
        n_ = 0;
    }
    void steal(SmallVec& o) {
        if (o.heap_) {
            heap_ = o.heap_;
            cap_ = o.cap_;
            n_ = o.n_;
            o.heap_ = nullptr;
            o.cap_ = N;
            o.n_ = 0;
        } else {
            heap_ = nullptr;
            cap_ = N;
            n_ = o.n_;
            for (unsigned i = 0; i < n_; ++i) reinterpret_cast<T*>(buf_)[i] = reinterpret_cast<const T*>(o.buf_)[i];
            o.n_ = 0;
        }
    }
    alignas(T) unsigned char buf_[sizeof(T) * N];
    T* heap_ = nullptr;
    unsigned n_ = 0, cap_ = N;
};

using Region = SmallVec<Box, 3>;  // canonical (R2) unless stated otherwise

// a \ b as disjoint boxes appended to out (peel slabs off dim 0, 1, 2).
template <class Vec>
inline void subtract_into(const Box& a, const Box& b, Vec& out) {
    Box i = intersect(a, b);
    if (i.empty()) {
        if (!a.empty()) out.push_back(a);
        return;
    }
    Box cur = a;
    for (int d = 0; d < 3; ++d) {
        if (cur.lo[d] < i.lo[d]) out.push_back(cur.with_dim(d, cur.lo[d], i.lo[d]));
        if (i.hi[d] < cur.hi[d]) out.push_back(cur.with_dim(d, i.hi[d], cur.hi[d]));
        cur = cur.with_dim(d, i.lo[d], i.hi[d]);
    }
}

namespace detail {
// Canonical boxes for the union of `bs` over dims d..2 (dims < d identical).
inline void canon_dim(Region& bs, int d, Region& out) {
    if (d == 2) {
        std::sort(bs.begin(), bs.end(), [](const Box& a, const Box& b) {
            return a.lo[2] != b.lo[2] ? a.lo[2] < b.lo[2] : a.hi[2] < b.hi[2];
        });
        int64_t cl = 0, ch = 0;
        bool open = false;
        const Box proto = bs[0];
        for (const Box& b : bs) {
            if (open && b.lo[2] <= ch) {
                ch = std::max(ch, b.hi[2]);
            } else {
                if (open) out.push_back(proto.with_dim(2, cl, ch));
                cl = b.lo[2];
                ch = b.hi[2];
                open = true;
            }
        }
        if (open) out.push_back(proto.with_dim(2, cl, ch));
        return;
    }
    std::vector<int64_t> cuts;
    cuts.reserve(bs.size() * 2);
    for (const Box& b : bs) {
        cuts.push_back(b.lo[d]);
        cuts.push_back(b.hi[d]);
    }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    // slabs: [lo, hi) with their canonical cross-section
    std::vector<std::pair<std::pair<int64_t, int64_t>, Region>> slabs;
    Region cover, sub;
    for (size_t k = 0; k + 1 < cuts.size(); ++k) {
        const int64_t lo = cuts[k], hi = cuts[k + 1];
        cover.clear();
        for (const Box& b : bs)
            if (b.lo[d] <= lo && hi <= b.hi[d]) cover.push_back(b.with_dim(d, 0, 1));
        if (cover.empty()) continue;
        sub.clear();
        canon_dim(cover, d + 1, sub);
        if (!slabs.empty() && slabs.back().first.second == lo && slabs.back().second == sub) {
            slabs.back().first.second = hi;
        } else {
            slabs.push_back({{lo, hi}, sub});
        }
    }
    for (auto& s : slabs)
        for (const Box& b : s.second) out.push_back(b.with_dim(d, s.first.first, s.first.second));
}
}  // namespace detail

namespace detail {
// canon_dim for boxes that all share one dim-2 range (1-D and 2-D buffers):
// the same dissection -- dim-0 slabs cut where the set of dim-1 intervals
// changes, each slab's merged dim-1 intervals -- on the stack.  false: too
// many boxes for the fixed arrays (the caller takes the general path).
inline bool canon_2d(const Region& bs, Region& out) {
    constexpr int kN = 16;
    const int n = int(bs.size());
    if (n > kN) return false;
    int64_t cuts[2 * kN];
    int nc = 0;
    for (const Box& b : bs) {
        cuts[nc++] = b.lo[0];
        cuts[nc++] = b.hi[0];
    }
    std::sort(cuts, cuts + nc);
    nc = int(std::unique(cuts, cuts + nc) - cuts);
    const int64_t z0 = bs[0].lo[2], z1 = bs[0].hi[2];
    int64_t pa[kN], pb[kN], ca[kN], cb[kN];
    int np = 0;
    int64_t s0 = 0, s1 = 0;
    auto flush = [&]() {
        for (int i = 0; i < np; ++i) {
            Box b;
            b.lo[0] = s0; b.hi[0] = s1;
            b.lo[1] = pa[i]; b.hi[1] = pb[i];
            b.lo[2] = z0; b.hi[2] = z1;
            out.push_back(b);
        }
        np = 0;
    };
    for (int k = 0; k + 1 < nc; ++k) {
        const int64_t lo = cuts[k], hi = cuts[k + 1];
        int m = 0;
        for (const Box& b : bs)
            if (b.lo[0] <= lo && hi <= b.hi[0]) {
                // insertion by start, then merge
                int p = m++;
                while (p > 0 && ca[p - 1] > b.lo[1]) {
                    ca[p] = ca[p - 1];
                    cb[p] = cb[p - 1];
                    --p;
                }
                ca[p] = b.lo[1];
                cb[p] = b.hi[1];
            }
        int w = 0;
        for (int i = 0; i < m; ++i) {
            if (w > 0 && ca[i] <= cb[w - 1]) {
                if (cb[i] > cb[w - 1]) cb[w - 1] = cb[i];
            } else {
                ca[w] = ca[i];
                cb[w] = cb[i];
                ++w;
            }
        }
        m = w;
        if (m == 0) {
            flush();
            continue;
        }
        bool same = np == m && s1 == lo;
        for (int i = 0; same && i < m; ++i) same = pa[i] == ca[i] && pb[i] == cb[i];
        if (same) {
            s1 = hi;
        } else {
            flush();
            for (int i = 0; i < m; ++i) {
                pa[i] = ca[i];
                pb[i] = cb[i];
            }
            np = m;
            s0 = lo;
            s1 = hi;
        }
    }
    flush();
    return true;
}
}  // namespace detail

inline Region canon(Region boxes) {
    boxes.erase(std::remove_if(boxes.begin(), boxes.end(), [](const Box& b) { return b.empty(); }), boxes.end());
    Region out;
    if (boxes.empty()) return out;
    if (boxes.size() == 1) {
        out.push_back(boxes[0]);
        return out;
    }
    // fast path: every box has the same (dim1, dim2) cross-section (row slabs,
    // plane slabs) -> the canonical form is the merged dim-0 intervals
    const Box& f = boxes[0];
    bool same = true;
    for (const Box& b : boxes)
        if (b.lo[1] != f.lo[1] || b.hi[1] != f.hi[1] || b.lo[2] != f.lo[2] || b.hi[2] != f.hi[2]) {
            same = false;
            break;
        }
    if (same) {
        std::sort(boxes.begin(), boxes.end(), [](const Box& a, const Box& b) { return a.lo[0] < b.lo[0]; });
        out.reserve(boxes.size());
        for (const Box& b : boxes) {
            if (!out.empty() && b.lo[0] <= out.back().hi[0]) {
                if (b.hi[0] > out.back().hi[0]) out.back().hi[0] = b.hi[0];
            } else {
                out.push_back(b);
            }
        }
        return out;
    }
    bool flat = true;                             // one dim-2 range: the stack path
    for (const Box& b : boxes)
        if (b.lo[2] != f.lo[2] || b.hi[2] != f.hi[2]) {
            flat = false;
            break;
        }
    if (flat && detail::canon_2d(boxes, out)) return out;
    out.clear();
    detail::canon_dim(boxes, 0, out);
    return out;
}

inline Region region_of(const Box& b) { return b.empty() ? Region{} : Region{b}; }

inline Region runion(const Region& a, const Region& b) {
    if (a.empty()) return b;
    if (b.empty()) return a;
    Region all(a);
    all.insert(all.end(), b.begin(), b.end());
    return canon(std::move(all));
}

inline Region rinter(const Region& a, const Region& b) {
    if (a.empty() || b.empty()) return {};
    if (a.size() == 1 && b.size() == 1) {
        Box i = intersect(a[0], b[0]);
        return i.empty() ? Region{} : Region{i};
    }
    Region out;
    for (const Box& x : a)
        for (const Box& y : b) {
            Box i = intersect(x, y);
            if (!i.empty()) out.push_back(i);
        }
    if (out.size() <= 1) return out;
    return canon(std::move(out));
}

inline Region rinter(const Region& a, const Box& b) {
    if (b.empty() || a.empty()) return {};
    Region out;
    bool whole = true;
    for (const Box& x : a) {
        Box i = intersect(x, b);
        if (i.empty()) {
            whole = false;
            continue;
        }
        if (i != x) whole = false;
        out.push_back(i);
    }
    if (whole) return a;              // a ⊆ b: already canonical
    if (out.size() <= 1) return out;
    return canon(std::move(out));
}

inline Box rbbox(const Region& r);
inline Region rdiff_nobb(const Region& a, const Region& b);
inline Region rdiff(const Region& a, const Region& b) {
    if (a.empty() || b.empty()) return a;
    if (intersect(rbbox(a), rbbox(b)).empty()) return a;
    return rdiff_nobb(a, b);
}
inline Region rdiff_nobb(const Region& a, const Region& b) {
    Region cur(a), nxt;
    bool changed = false;
    for (const Box& y : b) {
        nxt.clear();
        for (const Box& x : cur) {
            if (!overlaps(x, y)) {
                nxt.push_back(x);
            } else {
                changed = true;
                subtract_into(x, y, nxt);
            }
        }
        cur.swap(nxt);
        if (cur.empty()) break;
    }
    if (!changed) return a;
    return canon(std::move(cur));
}

inline uint64_t rvolume(const Region& r) {
    uint64_t v = 0;
    for (const Box& b : r) v += b.volume();
    return v;
}

inline Box rbbox(const Region& r) {
    Box out;
    for (const Box& b : r) out = bbox(out, b);
    return out;
}

inline bool rintersects(const Region& a, const Box& b) {
    for (const Box& x : a)
        if (overlaps(x, b)) return true;
    return false;
}

// Total map extent -> V (R3).  Entries sorted by value; regions canonical and
// pairwise disjoint; their union is the extent.
template <class V>
struct RegionMap {
    struct Entry {
        V first;
        Region second;
        Box bb;                        // bounding box of `second` (cheap rejects)
    };
    Box extent;
    std::vector<Entry> e;             // sorted by value

    RegionMap() = default;
    RegionMap(const Box& ext, const V& dflt) : extent(ext) {
        if (!ext.empty()) e.push_back({dflt, Region{ext}, ext});
    }

    void put(const V& v, const Region& r) {
        if (r.empty()) return;
        auto it = std::lower_bound(e.begin(), e.end(), v, [](const Entry& p, const V& x) { return p.first < x; });
        if (it != e.end() && it->first == v) {
            it->second = runion(it->second, r);
            it->bb = bbox(it->bb, rbbox(r));
        } else {
            e.insert(it, Entry{v, r, rbbox(r)});
        }
    }

    void update(const Region& reg0, const V& v) {
        Region reg = rinter(reg0, extent);
        if (reg.empty()) return;
        const Box rb = rbbox(reg);
        // only entries touching reg change; the rest stay in place
        size_t w = 0;
        for (size_t i = 0; i < e.size(); ++i) {
            Entry& p = e[i];
            if (overlaps(p.bb, rb)) {
                Region rr = rdiff_nobb(p.second, reg);
                if (rr.empty()) continue;
                if (rr.size() != p.second.size() || !(rr == p.second)) {
                    p.bb = rbbox(rr);
                    p.second = std::move(rr);
                }
            }
            if (w != i) e[w] = std::move(p);
            ++w;
        }
        e.resize(w);
        put(v, reg);
    }

    template <class F>
    void apply(const Region& reg0, F fn) {
        Region reg = rinter(reg0, extent);
        if (reg.empty()) return;
        const Box rb = rbbox(reg);
        // entries not touching reg stay in place; touched ones are split
        std::vector<std::pair<V, Region>> inside;
        size_t w = 0;
        for (size_t i = 0; i < e.size(); ++i) {
            Entry& p = e[i];
            if (overlaps(p.bb, rb)) {
                Region in = rinter(p.second, reg);
                if (!in.empty()) {
                    Region out = rdiff_nobb(p.second, reg);
                    inside.push_back({fn(p.first), std::move(in)});
                    if (out.empty()) continue;
                    p.bb = rbbox(out);
                    p.second = std::move(out);
                }
            }
            if (w != i) e[w] = std::move(p);
            ++w;
        }
        e.resize(w);
        for (auto& p : inside) put(p.first, p.second);
    }

    template <class F>
    void map_values(F fn) {
        std::vector<Entry> old;
        old.swap(e);
        // a non-decreasing fn (the horizon renaming, R7) keeps the order: equal
        // new values are adjacent, and their regions (disjoint) merge in one canon
        bool mono = true;
        for (size_t i = 1; i < old.size() && mono; ++i) mono = !(fn(old[i].first) < fn(old[i - 1].first));
        if (!mono) {
            for (auto& p : old) put(fn(p.first), p.second);
            return;
        }
        e.reserve(old.size());
        for (size_t i = 0; i < old.size();) {
            const V v = fn(old[i].first);
            size_t j = i + 1;
            while (j < old.size() && fn(old[j].first) == v) ++j;
            if (j == i + 1) {
                old[i].first = v;
                e.push_back(std::move(old[i]));
            } else {
                Region all;
                Box bb;
                for (size_t k = i; k < j; ++k) {
                    all.insert(all.end(), old[k].second.begin(), old[k].second.end());
                    bb = bbox(bb, old[k].bb);
                }
                e.push_back(Entry{v, canon(std::move(all)), bb});
            }
            i = j;
        }
    }

    // Partition of reg by value, sorted by value.
    std::vector<std::pair<Region, V>> query(const Region& reg) const {
        std::vector<std::pair<Region, V>> out;
        if (reg.empty()) return out;
        const Box rb = rbbox(reg);
        for (auto& p : e) {
            if (!overlaps(p.bb, rb)) continue;
            Region i = rinter(p.second, reg);
            if (!i.empty()) out.push_back({std::move(i), p.first});
        }
        return out;
    }

    // Values present on reg (no regions computed).
    template <class F>
    void for_values_in(const Region& reg, F fn) const {
        if (reg.empty()) return;
        const Box rb = rbbox(reg);
        for (auto& p : e) {
            if (!overlaps(p.bb, rb)) continue;
            bool hit = false;
            for (const Box& x : p.second) {
                if (!overlaps(x, rb)) continue;
                for (const Box& y : reg)
                    if (overlaps(x, y)) {
                        hit = true;
                        break;
                    }
                if (hit) break;
            }
            if (hit) fn(p.first);
        }
    }

    template <class P>
    Region where(P pred) const {
        Region all;
        for (auto& p : e)
            if (pred(p.first)) all.insert(all.end(), p.second.begin(), p.second.end());
        if (all.size() <= 1) return all;
        return canon(std::move(all));
    }
};

}  // namespace cel
