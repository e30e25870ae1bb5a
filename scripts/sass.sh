#!/bin/bash
# usage: scripts/sass.sh <mangled-name-substring>  -> SASS of that function (no encodings)
cuobjdump -sass paper_2503_01253_b200/libnmspmm.so | awk -v pat="$1" '$0 ~ "Function : .*"pat {f=1;next} /Function :/{f=0} f' | grep -v "^\s*/\* 0x" | sed -E 's@/\*[0-9a-f]{4}\*/@@; s@;\s*/\*.*@@'
