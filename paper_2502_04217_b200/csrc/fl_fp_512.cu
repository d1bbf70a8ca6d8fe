// Instantiations of the fast pass kernels for lengths 512.
#include "fl_fastpass.cuh"
#include "fl_gpass.cuh"

namespace fl {
namespace fpk {

Entry make_512(bool strided, int kind, bool epi) { return make_any<512>(strided, kind, epi); }
Entry make_group_512(int kind, bool epi) { return gpk::make_group<512>(kind, epi); }

}  // namespace fpk
}  // namespace fl
