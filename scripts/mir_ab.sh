#!/bin/bash
# dev aid: DAS time per config with 1 / 2 / 4 mirror lines per CTA (dev build:
# python -m paper_1711_06127_b200.build --variant=dev -DSUPRA_DEV_KNOBS)
lib=$PWD/_variants/dev/libsupra_bf.so
SPECS=${1:-"C4a:1 C4b:1 C4p:1 C4b:8 C4p:4 C3:16 C3:2"}
for spec in $SPECS; do
  c=${spec%%:*}; f=${spec##*:}
  for m in 1 2 4; do
    echo -n "$c F=$f MIR=$m: "; SUPRA_BF_MIR=$m python scripts/quick_time.py --lib=$lib $c $f 2>&1 | grep -E "beamform [0-9]|Error|error" | head -2
  done
done
