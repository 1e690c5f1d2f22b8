// profile.cuh -- the profile-first exact path for rank-deficient input (see profile.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "pluq.cuh"

namespace ffg {

// tile_rec's P and Q (to_array form, m and n words) from the rank profile matrix: pivots
// (prow[k], pcol[k]), k < rank, any order (rpsim.cu).  Returns rank.  Host only.
size_t tile_rec_perms(size_t m, size_t n, size_t thr, size_t rank, const uint32_t* prow, const uint32_t* pcol,
                      uint32_t* P, uint32_t* Q);

// phase 1: the rank profile of W (m x n, reduced in place) -- pivots in rr_base's discovery order
// (row-major greedy search, rankrev.hpp:40-57): prow[k], pcol[k] = rr_base's P[k], Q[k], k < rank
size_t rank_profile_dev(const Blas& b, DView W, std::vector<uint32_t>& prow, std::vector<uint32_t>& pcol);

// phases 2 + 3: tile_rec's outputs on `a` given its rank profile; P/Q host arrays; scratch: m x n
// device words (ld n)
void pluq_from_profile_dev(const Blas& b, DView a, size_t threshold, size_t rank, const uint32_t* prow,
                           const uint32_t* pcol, uint32_t* P, uint32_t* Q, uint32_t* scratch);

// the whole profile-first path: pluq_tile_recursive's outputs, bit for bit
size_t pluq_profile_first_dev(const Blas& b, DView a, size_t threshold, uint32_t* P, uint32_t* Q);

// true on a thread inside pluq_profile_first_dev / pluq_from_profile_dev
bool profile_first_active();

// whether the slab kernel takes n columns (n <= ~80K)
bool profile_first_fits(size_t n);

}  // namespace ffg
