#!/bin/bash
# usage: tools/sass_mix.sh <kernel-name-regex>  -- instruction mix of one kernel in libccnn.so
cd "$(dirname "$0")/.." && python paper_1508_01292_b200/build.py >/dev/null || exit 1
cuobjdump -sass paper_1508_01292_b200/libccnn.so | awk -v pat="$1" '/Function : /{p = ($0 ~ pat)} p' > build_tools/mix.sass
grep -A2 "$1" paper_1508_01292_b200/build/ptxas.log | grep -E "registers|spill" | head -2
echo "total instructions: $(grep -cE '^\s+/\*[0-9a-f]+\*/' build_tools/mix.sass)"
grep -oE "^\s+/\*[0-9a-f]+\*/\s+[A-Z0-9_.]+" build_tools/mix.sass | awk '{print $2}' | sort | uniq -c | sort -rn | head -${2:-14}
