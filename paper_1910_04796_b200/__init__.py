"""B200-native DBCSR dense-multiply hot path (arXiv 1910.04796).

The product is libdbm.so (CUDA for sm_100a behind the C ABI in include/dbm.h); this package is
its thin Python binding.  See DESIGN.md.
"""
from .dbm import (EXPORTS, K_DENSIFY, K_DGEMM, K_EXCHANGE, K_SMM, K_STACKGEN, K_UNDENSIFY, LIB_PATH, PATH_AUTO, PATH_BLOCKED,
                  PATH_DENSIFIED, Context, DbmError, Matrix, debug_dgemm, debug_first_step, debug_pack_panel, debug_stacks, load,
                  multiply,
                  multiply_host, multiply_workspace, pattern_product, pattern_random, plan_exchange, plan_tallskinny)

__all__ = ["Context", "Matrix", "multiply", "multiply_host", "multiply_workspace", "plan_exchange", "plan_tallskinny",
           "pattern_random", "pattern_product", "debug_stacks", "debug_first_step", "debug_pack_panel", "debug_dgemm", "load", "DbmError", "EXPORTS", "LIB_PATH", "PATH_AUTO",
           "PATH_BLOCKED", "PATH_DENSIFIED", "K_DGEMM", "K_SMM", "K_DENSIFY", "K_UNDENSIFY", "K_STACKGEN", "K_EXCHANGE"]
