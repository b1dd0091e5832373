# A/B of decode launch knobs on one box (rebuilds decode_fused.cu with EXTRA flags)
B="python bench.py --no-cpu-baseline --factor-init placeholder --steps 30 --warmup 5"
C=paper_2603_23914_b200/csrc
touch $C/decode_fused.cu; make -s -C $C > /dev/null 2>&1
$B > gpurun_out/ab_base.json 2> gpurun_out/ab_base.err
KVP_GROUPS=2 $B > gpurun_out/ab_g2.json 2>&1
for t in 512 1024; do
  touch $C/decode_fused.cu; make -s -C $C EXTRA=-DKVP_STREAM_THREADS=$t > /dev/null 2>&1
  $B > gpurun_out/ab_$t.json 2> gpurun_out/ab_$t.err
done
touch $C/decode_fused.cu; make -s -C $C > /dev/null 2>&1
$B > gpurun_out/ab_base2.json 2>&1
