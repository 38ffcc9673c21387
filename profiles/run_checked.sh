#!/bin/bash
# The GPU test suite against a checked build of the library: NASG_CHECK
# invariants (shared / tensor memory ranges, tile and list indices) and every
# mbarrier wait bounded to ~4 s, each trapping with a message (tc_ptx.cuh).
# compute-sanitizer is closed on this pool (r2_compute_sanitizer_closed.txt).
set -e
make -C paper_2303_08064_b200/csrc -j8 OUT=$PWD/paper_2303_08064_b200/lib_exp/checked EXTRA=-DNASG_CHECKED
NASG_LIB=paper_2303_08064_b200/lib_exp/checked/libnasg_b200.so python -m pytest tests/ -m gpu -q -p no:cacheprovider
