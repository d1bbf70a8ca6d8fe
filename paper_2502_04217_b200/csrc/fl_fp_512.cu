// Instantiations of the fast pass kernels for lengths 512.
#include "fl_fastpass.cuh"

namespace fl {
namespace fpk {

Entry make_512(bool strided, int kind, bool epi) { return make_any<512>(strided, kind, epi); }

}  // namespace fpk
}  // namespace fl
