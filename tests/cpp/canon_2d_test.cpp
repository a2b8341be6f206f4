// The stack path of the region canonical form (geom.hpp detail::canon_2d,
// boxes sharing one dim-2 range) against the general dissection
// (detail::canon_dim): equal on 400,000 random regions of 2-15 boxes.
// Built and run by tests/test_geom_canon.py.
#include "geom.hpp"
#include <cstdio>
#include <random>
using namespace cel;
int main() {
    std::mt19937 g(7);
    long bad = 0, n = 0;
    for (int it = 0; it < 400000; ++it) {
        Region r;
        int k = 2 + g() % 14;
        int64_t z0 = g() % 3, z1 = z0 + 1 + g() % 2;
        for (int i = 0; i < k; ++i) {
            Box b;
            int64_t a0 = g() % 12, a1 = a0 + 1 + g() % 6, b0 = g() % 12, b1 = b0 + 1 + g() % 6;
            b.lo[0] = a0; b.hi[0] = a1; b.lo[1] = b0; b.hi[1] = b1; b.lo[2] = z0; b.hi[2] = z1;
            r.push_back(b);
        }
        Region gen;
        Region tmp = r;
        detail::canon_dim(tmp, 0, gen);
        Region fast;
        detail::canon_2d(r, fast);
        ++n;
        if (!(gen == fast)) ++bad;
    }
    printf("%ld / %ld differ\n", bad, n);
    return bad != 0;
}
