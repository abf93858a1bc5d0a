// cw_jit.cuh -- run-time compiled fused-kernel instances (see cw_jit.cu).
#pragma once
#include <string>

namespace cwb {

struct LaunchFn;

// the fused kernel can take this geometry (tables, shared memory, threads)
bool jit_supported(int kx, int ky, int kz, int bx, int by, int nlx, int nly);
// the instance Geo<kx, ky, kz, bx, by> with NL = nl (0: runtime lag loops),
// from the cubin cache or compiled now; false (+ message) if unavailable
bool jit_instance(int kx, int ky, int kz, int bx, int by, int nl, LaunchFn *out, std::string *err);
// compile into `dir` unless cached there already (build-time prebuild)
int jit_prebuild(int kx, int ky, int kz, int bx, int by, int nl, const char *dir, std::string *err);

}  // namespace cwb
