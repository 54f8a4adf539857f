#!/bin/bash
# dev aid: DAS time under forced launch shapes (dev build with -DSUPRA_DEV_KNOBS)
lib=$PWD/_variants/dev/libsupra_bf.so
for s in "" 16x4 8x4 8x8; do echo -n "C3:16 shape=$s "; SUPRA_BF_SHAPE=$s python scripts/quick_time.py --lib=$lib C3 16 | grep -E "beamform [0-9]"; done
for s in "" 8x4 8x8; do echo -n "C3:32 shape=$s "; SUPRA_BF_SHAPE=$s python scripts/quick_time.py --lib=$lib C3 32 | grep -E "beamform [0-9]"; done
for m in 1 2 4; do echo -n "C4p:1 MIR=$m "; SUPRA_BF_MIR=$m python scripts/quick_time.py --lib=$lib C4p 1 | grep -E "beamform [0-9]"; done
for m in 1 2 4; do echo -n "C4b:1 MIR=$m "; SUPRA_BF_MIR=$m python scripts/quick_time.py --lib=$lib C4b 1 | grep -E "beamform [0-9]"; done
