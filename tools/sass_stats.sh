#!/bin/bash
# Build libarv_b200.so and print per-opcode counts of one kernel's main loop.
#   tools/sass_stats.sh <mangled-name-regex> [start_line end_line]
set -e
cd /root/repo
python paper_2012_09715_b200/_build.py > /dev/null
cuobjdump -sass paper_2012_09715_b200/libarv_b200.so 2>/dev/null | awk -v pat="$1" '/Function : /{f = ($0 ~ pat)} f' \
  | grep -E '^\s+/\*[0-9a-f]{4}\*/' | sed 's@/\* 0x[0-9a-f]* \*/@@;s@^\s*/\*[0-9a-f]*\*/\s*@@' > /tmp/k.sass
grep -n "STG\|BRA" /tmp/k.sass | head -20
if [ -n "$2" ]; then
  sed -n "$2,$3p" /tmp/k.sass | awk '{op=$1; if(op ~ /^@/) op=$2; print op}' | sed 's/\..*//' | sort | uniq -c | sort -rn
fi
