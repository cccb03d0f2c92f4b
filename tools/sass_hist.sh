#!/bin/bash
# usage: tools/sass_hist.sh <lib.so> <kernel-name-regex>   -- static opcode histogram of one kernel
cuobjdump -sass "$1" | awk -v pat="$2" 'f&&/Function : /{exit} $0 ~ "Function : .*"pat {f=1} f{print}' \
 | grep -oE "/\*[0-9a-f]{4}\*/ +[@!UP0-9 ]*[A-Z][A-Z0-9_.]+" | awk '{print $NF}' | sort | uniq -c | sort -rn | head -${3:-25}
