#!/bin/bash
# static SASS opcode mix of one kernel: sass_mix.sh <lib.so> <mangled-name-substring>
cuobjdump -sass "$1" 2>/dev/null | awk -v k="$2" '/Function :/ {on = index($0, k) > 0} on' \
  | grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9.]+" | awk '{print $2}' | sed 's/\..*//' | sort | uniq -c | sort -rn \
  | awk '{t+=$1; printf "%s:%s ",$2,$1} END {print "\nTOTAL",t}'
