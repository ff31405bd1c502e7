// Both include orders of the reference C header and this library's header in one program
// (compiled -fsyntax-only, as C++ and as C, by tests/test_integration_cpu.py).
#ifdef LAB_FIRST
#include "compass_lab.h"
#include "compass_moe.h"
#else
#include "compass_moe.h"
#include "compass_lab.h"
#endif

int statuses_agree(void) {
  cl_status s = CL_ERR_CONFIG;
  return s == 2 && CL_ERR_RUN == 1 && CL_OK == 0 && sizeof(cl_moe_config) > 0;
}
