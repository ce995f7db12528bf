// Host/device record of a failed peer-memory wait (see ptx::wait_epoch).
#pragma once

#include <cstdint>

namespace c3d {
namespace ptx {

// Where a peer-memory wait reports a failure (the reference poisons the group and throws
// Desync, cube3d/transport.hpp:67-78, 305-319): word[0] = code (1 timeout, 2 header
// mismatch), word[1] = site, word[2] = expected epoch / own header, word[3] = seen epoch /
// peer header. `word` is mapped pinned host memory, read by the host after the stream
// synchronises (Cube::check_fault).
struct Fault {
  uint32_t* word = nullptr;
  unsigned long long timeout_ns = 30ull * 1000000000ull;
};

}  // namespace ptx
using ptx::Fault;
}  // namespace c3d
