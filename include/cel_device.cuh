/* Device-side helper for CALLBACK kernels (include/cel.h): accessor bounds
 * checking (§4.4 "Accessor Bounds Checking").
 *
 * A user kernel that receives cel_accessor structs may call
 * cel_check_access(&acc, z, y, x) for every element it touches (buffer
 * coordinates; unused dimensions 0).  When the runtime was created with
 * cel_config.bounds_check = 1, accesses outside acc.range are recorded (their
 * bounding box, by atomic min / max on acc.oob) and reported by the runtime
 * after the kernel exits, as a CEL_E_OUT_OF_BOUNDS error.  The function returns
 * 1 when the access is inside the range mapper's region (always 1 when
 * checking is off).  Header only; include from .cu files.
 */
#pragma once

#include "cel.h"

static __device__ __forceinline__ int cel_check_access(const cel_accessor* a, long long z, long long y, long long x) {
    if (!a->oob) return 1;
    if (z >= (long long)a->range.min[0] && z < (long long)a->range.max[0] && y >= (long long)a->range.min[1] &&
        y < (long long)a->range.max[1] && x >= (long long)a->range.min[2] && x < (long long)a->range.max[2])
        return 1;
    atomicMin(&a->oob[0], z);
    atomicMin(&a->oob[1], y);
    atomicMin(&a->oob[2], x);
    atomicMax(&a->oob[3], z + 1);
    atomicMax(&a->oob[4], y + 1);
    atomicMax(&a->oob[5], x + 1);
    return 0;
}
