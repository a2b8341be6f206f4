// Private declarations shared by sched.cpp and cluster.cpp.
#pragma once

#include <vector>

#include "sched.hpp"

namespace cel {
namespace detail {
void split_1d(const Box& rng, int n, int dim, std::vector<Box>& out);
std::vector<Box> split(const Box& rng, int n, int kind);        // R4: 0 = 1D, 1 = 2D
int apply_mapper(const Mapper& m, const Box& chunk, const Box& ext, Box* out);   // R5
// the region a chunk accesses: the mapper's box, except the cross of NeighborhoodAxes
int mapper_region(const Mapper& m, const Box& chunk, const Box& ext, Region* out);
bool is_read(int mode);
bool is_write(int mode);
uint64_t memo_hash(const std::vector<int64_t>& v);    // sched_memo.cpp
}  // namespace detail
}  // namespace cel
