#include "format.hpp"
#include "preshuffle.hpp"

namespace rfl {
ShuffleResult run_shuffle_gpu(const ShuffleArgs&) { invalid("run_shuffle: GPU pre-shuffle not built yet"); }
}  // namespace rfl
