#!/bin/bash
# dev aid: C2 A/B -- in-tree lib, dev lib with SUPRA_BF_MIR=1/2, round-1 tree
for i in 1 2; do
python scripts/quick_time.py C2 100 2>&1 | grep -E "beamform|GB/s"
for m in 1 2; do echo "MIR=$m"; SUPRA_BF_MIR=$m python scripts/quick_time.py --lib=$PWD/_variants/dev/libsupra_bf.so C2 100 2>&1 | grep -E "beamform|GB/s|'das"; done
echo r1; (cd _variants/r1tree && python scripts/quick_time.py C2 100 2>&1 | grep -E "beamform|GB/s")
done
