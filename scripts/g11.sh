mkdir -p gpurun_out
( for v in cur v2 v3 v6; do lib=$PWD/_variants/$v/libsupra_bf.so; [ $v = cur ] && lib=""; for c in "C4p 1" "C4p 4" "C4b 1" "C3 32"; do set -- $c; echo -n "$v "; python scripts/sc_time.py --lib=$lib $1 $2 2>&1 | tail -1; done; done ) > gpurun_out/sc_v.log 2>&1
