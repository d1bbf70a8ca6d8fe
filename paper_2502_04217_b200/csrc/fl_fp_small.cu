// Instantiations of the fast pass kernels for lengths 16, 32, 64, 128, 256.
#include "fl_fastpass.cuh"

namespace fl {
namespace fpk {

Entry make_16(bool strided, int kind, bool epi) { return make_any<16>(strided, kind, epi); }
Entry make_32(bool strided, int kind, bool epi) { return make_any<32>(strided, kind, epi); }
Entry make_64(bool strided, int kind, bool epi) { return make_any<64>(strided, kind, epi); }
Entry make_128(bool strided, int kind, bool epi) { return make_any<128>(strided, kind, epi); }
Entry make_256(bool strided, int kind, bool epi) { return make_any<256>(strided, kind, epi); }

}  // namespace fpk
}  // namespace fl
