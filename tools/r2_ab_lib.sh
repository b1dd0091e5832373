#!/bin/bash
# Same-box A/B of the whole step: the current library vs gpurun_in/libkvp_old.so (a previous build), C5 and C4 8x.
mkdir -p gpurun_out/r2
L=paper_2603_23914_b200/libkvp_b200.so
cp $L /tmp/libkvp_new.so
for rep in 1 2; do
  for v in new old; do
    if [ $v = old ]; then cp gpurun_in/libkvp_old.so $L; else cp /tmp/libkvp_new.so $L; fi
    for cfg in ${CFGS:-c5 c4_8x c2}; do
      echo "== $v $cfg $rep" >> gpurun_out/r2/ab_lib.txt
      timeout 600 python bench.py --config $cfg --steps 64 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['ms_per_layer']*1e3,2), d['compaction_ms'] if 'compaction_ms' in d else '')" >> gpurun_out/r2/ab_lib.txt
    done
  done
done
cp /tmp/libkvp_new.so $L
