// Instantiations of the fast pass kernels for lengths 1024, 2048, 4096, 8192.
#include "fl_fastpass.cuh"

namespace fl {
namespace fpk {

Entry make_1024(bool strided, int kind, bool epi) { return make_any<1024>(strided, kind, epi); }
Entry make_2048(bool strided, int kind, bool epi) { return make_any<2048>(strided, kind, epi); }
Entry make_4096(bool strided, int kind, bool epi) { return make_any<4096>(strided, kind, epi); }
Entry make_8192(bool strided, int kind, bool epi) { return make_any<8192>(strided, kind, epi); }

}  // namespace fpk
}  // namespace fl
