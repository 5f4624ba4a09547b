#!/bin/bash
# usage: tools/sass.sh <substring of mangled kernel name>  -> SASS of the first match
LIB=${LIB:-paper_1407_3535_b200/lib/libtmatch_cuda.so}
F=$(cuobjdump -sass "$LIB" 2>/dev/null | grep "Function : " | grep -- "$1" | head -1 | awk '{print $3}')
cuobjdump -sass -fun "$F" "$LIB" 2>/dev/null | grep -E "^\s+/\*[0-9a-f]+\*/" | sed 's@/\* 0x[0-9a-f]* \*/@@'
