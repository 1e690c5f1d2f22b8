// profile.cuh -- the profile-first exact path for rank-deficient input (see profile.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#include "pluq.cuh"

namespace ffg {

// tile_rec's P and Q (to_array form, m and n words) from the rank profile matrix: pivots
// (prow[k], pcol[k]), k < rank, any order (rpsim.cu).  Returns rank.  Host only.
size_t tile_rec_perms(size_t m, size_t n, size_t thr, size_t rank, const uint32_t* prow, const uint32_t* pcol,
                      uint32_t* P, uint32_t* Q);

}  // namespace ffg
