// pluq.cu -- placeholder until the TRSM / base case / driver land.
#include "pluq.cuh"

namespace ffg {

void ftrsm_dev(const Blas&, int, int, int, DView, DView, bool) { throw Error(FFG_ERR_INTERNAL, "ftrsm: not built yet"); }
size_t rr_base_dev(const Blas&, DView, uint32_t*, uint32_t*) { throw Error(FFG_ERR_INTERNAL, "rr_base: not built yet"); }
size_t pluq_tile_recursive_dev(const Blas&, DView, size_t, uint32_t*, uint32_t*) {
    throw Error(FFG_ERR_INTERNAL, "pluq: not built yet");
}
void apply_perm_dev(const Blas&, DView, int, int, const uint32_t*) { throw Error(FFG_ERR_INTERNAL, "perm: not built yet"); }

}  // namespace ffg
