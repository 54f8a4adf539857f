#!/bin/bash
# dev aid: scan-conversion timing per library variant, u8 line images; usage: sc_time.sh "cur v1" "C4b:1 C3:16"
for v in $1; do
  lib=$PWD/_variants/$v/libsupra_bf.so; [ "$v" = cur ] && lib=""
  for spec in $2; do c=${spec%%:*}; f=${spec##*:}
    echo -n "$v $c:$f "; python scripts/sc_time.py --lib=$lib $c $f 2>&1 | tail -1
  done
done
