#!/bin/bash
# dev aid: A/B timings of library variants (_variants/<name>/libsupra_bf.so; "cur" = in-tree build)
# usage: bash scripts/ab.sh "cur orig r64" "C2:100 C3:16 C4a:1 C4b:8" ["0 1 2" debug modes]
# (debug modes 1/2 need a variant built with -DSUPRA_DEV_KNOBS, e.g.
#  python -m paper_1711_06127_b200.build --variant=dev -DSUPRA_DEV_KNOBS)
for v in $1; do
  lib=$PWD/_variants/$v/libsupra_bf.so; [ "$v" = cur ] && lib=""
  for d in ${3:-0}; do
    for spec in $2; do
      c=${spec%%:*}; f=${spec##*:}
      echo -n "$v dbg=$d "; SUPRA_BF_DEBUG=$d python scripts/quick_time.py --lib=$lib $c $f 2>&1 | grep -E "beamform [0-9]"
    done
  done
done
