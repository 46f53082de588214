// load_cameras -> save_cameras through the drop-in C++ API (include/sof_b200/sof.hpp):
//   camera_io <in.json> <out.json>; prints the exception message and exits 3 on error.
// Driven by tests/test_io_cpu.py against the compiled reference's save_cameras.
#include <cstdio>
#include <exception>

#include "sof_b200/sof.hpp"

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  try {
    sof::save_cameras(sof::load_cameras(argv[1]), argv[2]);
  } catch (const std::exception& e) {
    std::printf("%s\n", e.what());
    return 3;
  }
  return 0;
}
