// Instantiations of the fast pass kernels for lengths 1024, 2048, 4096, 8192.
#include "fl_fastpass.cuh"
#include "fl_gpass.cuh"
#include "fl_wpass.cuh"

namespace fl {
namespace fpk {

Entry make_1024(bool strided, int kind, bool epi) { return make_any<1024>(strided, kind, epi); }
Entry make_2048(bool strided, int kind, bool epi) { return make_any<2048>(strided, kind, epi); }
Entry make_4096(bool strided, int kind, bool epi) { return make_any<4096>(strided, kind, epi); }
Entry make_8192(bool strided, int kind, bool epi) { return make_any<8192>(strided, kind, epi); }

// contiguous m = 1024: two-stage warp passes (fl_wpass.cuh); 2048: group-decoupled passes (fl_gpass.cuh)
Entry make_warp_1024(int kind, bool epi, bool nrm) { return wpk::make_warp<1024>(kind, epi, nrm); }
Entry make_group_2048(int kind, bool epi) { return gpk::make_group<2048>(kind, epi); }

// strided m = 1024: the mirrored 8 x 16 x 8 engine (fl_mirror.cuh)
Entry make_mirror_1024(int kind) { return make_mirror1024<1024>(kind); }

}  // namespace fpk
}  // namespace fl
