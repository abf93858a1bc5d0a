// cw_inst.cu -- one kernel instance per translation unit: compiled once per
// CW_INSTANCES entry with -DCW_IKX=.. -DCW_IKY=.. -DCW_IKZ=.. -DCW_IBX=..
// -DCW_IBY=.. -DCW_INL=.. (see _native.build), so the instances build in
// parallel.
#include "cw_inst.cuh"

#if !defined(CW_IKX) || !defined(CW_IKY) || !defined(CW_IKZ) || !defined(CW_IBX) || !defined(CW_IBY) || !defined(CW_INL)
#error "compile with -DCW_IKX=.. -DCW_IKY=.. -DCW_IKZ=.. -DCW_IBX=.. -DCW_IBY=.. -DCW_INL=.."
#endif

#define CW_DEFINE(a, b, c, d, e, n) \
    cwb::LaunchFn CW_INST_FN(a, b, c, d, e, n)() { return cwb::make_inst<a, b, c, d, e, n>(); }
#define CW_DEFINE_X(a, b, c, d, e, n) CW_DEFINE(a, b, c, d, e, n)
CW_DEFINE_X(CW_IKX, CW_IKY, CW_IKZ, CW_IBX, CW_IBY, CW_INL)
