#!/bin/bash
# usage: sass_region.sh <kernel-name-regex> -> dumps SASS of the first matching kernel to /tmp/k.sass
cuobjdump -sass /root/repo/paper_2202_13926_b200/libfsr.so | awk -v pat="$1" '$0 ~ "Function : .*"pat {f=1;print;next} f&&/Function : /{f=0} f' > /tmp/k.sass
grep -c "" /tmp/k.sass
