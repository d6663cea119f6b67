#!/bin/bash
# List local-memory (spill) accesses and warp reductions of one kernel's SASS, in
# address order, to see whether a spill sits inside the iteration loop.
# usage: tools/sass_spills.sh <mangled-name-substring> [lib]
LIB=${2:-paper_2202_13926_b200/libfsr.so}
cuobjdump -sass "$LIB" | awk -v pat="$1" '/Function :/ {on = index($0, pat) > 0} on' |
  grep -E "LDL|STL|CREDUX|EXIT" | sed 's@/\* 0x[0-9a-f]* \*/@@; s/  */ /g'
