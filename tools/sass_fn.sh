#!/bin/bash
# Dump the SASS of one kernel (regex on the mangled name) from a .so: tools/sass_fn.sh LIB REGEX > out
LIB=$1; RE=$2
F=$(cuobjdump -sass "$LIB" | grep -o "Function : .*" | sed 's/Function : //' | grep -E "$RE" | head -1)
cuobjdump -sass "$LIB" | awk -v f="$F" 'index($0, "Function : " f) {p=1; next} /Function :/ {p=0} p' \
  | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed 's#/\* 0x[0-9a-f]* \*/##; s/ *;.*//'
