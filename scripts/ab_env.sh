#!/bin/bash
# dev aid: beamform timing of the dev variant (-DSUPRA_DEV_KNOBS) over the values of one knob
# usage: ab_env.sh SUPRA_BF_L2AHEAD "0 1 2" "C2:100 C4a:1" [variant]
lib=$PWD/_variants/${4:-dev}/libsupra_bf.so
for v in $2; do
  for spec in $3; do
    c=${spec%%:*}; f=${spec##*:}
    echo -n "$1=$v $c:$f "; env $1=$v python scripts/quick_time.py --lib=$lib $c $f 2>&1 | grep -E "beamform [0-9]|rror"
  done
done
