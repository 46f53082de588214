// ELF interposition of exp/log for the reference build (TEST INFRASTRUCTURE).
//
// The reference calls std::exp / std::log (gaussian.hpp:48,55,62;
// opacity_field.hpp:162). libstdc++'s std::exp(double) is ::exp, so defining
// ::exp / ::log here (executables: the definition wins over libm; shared objects: hidden
// visibility binds every call inside the library to it) routes the UNMODIFIED reference headers through the
// framework's sof_exp / sof_log — the same bits the CUDA kernels compute.
// Compile with -fno-builtin-exp -fno-builtin-log so GCC cannot constant-fold.
#include "../paper_2506_19139_b200/csrc/sof_math.h"

// In the shared library these definitions are hidden: calls from the other objects
// of the same link unit bind to them directly (no PLT, no interposition by libm),
// and nothing is exported, so the host process's own exp/log stay untouched.
#define SOF_LOCAL __attribute__((visibility("hidden")))
extern "C" SOF_LOCAL double exp(double x) noexcept { return sof_exp(x); }
extern "C" SOF_LOCAL double log(double x) noexcept { return sof_log(x); }
