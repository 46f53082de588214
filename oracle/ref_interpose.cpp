// ELF interposition of exp/log for the reference build (TEST INFRASTRUCTURE).
//
// The reference calls std::exp / std::log (gaussian.hpp:48,55,62;
// opacity_field.hpp:162). libstdc++'s std::exp(double) is ::exp, so defining
// ::exp / ::log here (executables: definition wins over libm; shared objects:
// linked with -Wl,-Bsymbolic) routes the UNMODIFIED reference headers through the
// framework's sof_exp / sof_log — the same bits the CUDA kernels compute.
// Compile with -fno-builtin-exp -fno-builtin-log so GCC cannot constant-fold.
#include "../paper_2506_19139_b200/csrc/sof_math.h"

extern "C" double exp(double x) noexcept { return sof_exp(x); }
extern "C" double log(double x) noexcept { return sof_log(x); }
