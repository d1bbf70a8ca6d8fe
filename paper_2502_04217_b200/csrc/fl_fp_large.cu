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
Entry make_warp_1024(int kind, bool epi) { return wpk::make_warp<1024>(kind, epi); }
Entry make_group_2048(int kind, bool epi) { return gpk::make_group<2048>(kind, epi); }

// strided m = 1024 as two mirrored 512-point halves (fl_split.cuh)
Entry make_split_1024(int kind) {
  Entry e;
  if (kind == K_SYNTH) e.fn = split::split_pass<K_SYNTH>;
  else if (kind == K_ANALYZE) e.fn = split::split_pass<K_ANALYZE>;
  e.threads = split::T;
  e.smem = split::SMEM;
  e.w = split::W;
  return e;
}

}  // namespace fpk
}  // namespace fl
