#!/bin/bash
# A/B of experiment builds of libfastb200.so on the config-5 synthesis bench.
# usage: tools/ab_synth.sh [bench args] -- lib1.so lib2.so ...   ("default" = in-tree build)
args=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do args+=("$1"); shift; done
shift
for l in "$@"; do
  if [ "$l" = default ]; then unset FASTB200_LIB; else export FASTB200_LIB=$l; fi
  python bench.py --no-cpu-baseline --no-e2e "${args[@]}" 2>/dev/null |
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$l', d['value'], d['roofline']['kernel_ms'])"
done
