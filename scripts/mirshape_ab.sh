#!/bin/bash
# dev aid: C4a / C4b single volume under forced mirror shapes (dev build)
lib=$PWD/_variants/dev/libsupra_bf.so
for c in C4a C4b; do for s in "" 4x8 4x4; do echo -n "$c:1 mirshape=$s "; SUPRA_BF_MIRSHAPE=$s python scripts/quick_time.py --lib=$lib $c 1 | grep -E "beamform [0-9]"; done; done
for s in "" 4x4; do echo -n "C4a:1 dbg1 mirshape=$s "; SUPRA_BF_DEBUG=1 SUPRA_BF_MIRSHAPE=$s python scripts/quick_time.py --lib=$lib C4a 1 | grep -E "beamform [0-9]"; done
for s in "" 4x4; do echo -n "C4a:1 dbg2 mirshape=$s "; SUPRA_BF_DEBUG=2 SUPRA_BF_MIRSHAPE=$s python scripts/quick_time.py --lib=$lib C4a 1 | grep -E "beamform [0-9]"; done
