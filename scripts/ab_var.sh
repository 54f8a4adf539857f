#!/bin/bash
# dev aid: beamform timing of library variants; usage: ab_var.sh "cur ch ord" "C2:100 C4a:1" [reps]
for r in $(seq ${3:-1}); do
for v in $1; do
  lib=$PWD/_variants/$v/libsupra_bf.so; [ "$v" = cur ] && lib=""
  for spec in $2; do
    c=${spec%%:*}; f=${spec##*:}
    echo -n "$v $c:$f "; python scripts/quick_time.py --lib=$lib $c $f 2>&1 | grep -E "beamform [0-9]|rror"
  done
done
done
