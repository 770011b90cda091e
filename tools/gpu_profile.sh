#!/bin/bash
# ncu evidence for profiles/: launch list of the bench command + one --set full capture per kernel.
# usage (on the GPU box): tools/gpu_profile.sh TAG
TAG=${1:-r}
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu --decode-steps 64 > /dev/null 2>&1
full() {  # name kernel-regex skip env...
  local name=$1 re=$2 skip=$3; shift 3
  env "$@" timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 \
      -o $OUT/prof_${name}_$TAG python tools/prof_driver.py > $OUT/prof_${name}_$TAG.log 2>&1
  tail -1 $OUT/prof_${name}_$TAG.log
}
full cfg2_prefill prefill_tc_pipe 2 PROF_SHAPE=8,32,8192,128
full cfg3_prefill tmem_state 2 PROF_SHAPE=4,16,16384,256,512
full cfg5_statepass prefill_tc_pipe 4 PROF_SHAPE=1,32,131072,128
full cfg5_prefill prefill_tc_pipe 5 PROF_SHAPE=1,32,131072,128
timeout 600 ncu --set full --clock-control none --import-source on -k regex:simt -s 1 -c 1 \
    -o $OUT/prof_fp32_prefill_$TAG python tools/f32_once.py > $OUT/prof_fp32_prefill_$TAG.log 2>&1
PROF_DTYPE=f32 PROF_KERNEL=tf32 PROF_SHAPE=8,32,8192,128 timeout 600 ncu --set full --clock-control none \
    --import-source on -k regex:prefill_tf32 -s 2 -c 1 -o $OUT/prof_tf32_prefill_$TAG python tools/prof_driver.py \
    > $OUT/prof_tf32_prefill_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_step -s 5 -c 1 \
    -o $OUT/prof_decode_$TAG python bench.py --steps 1 --warmup 3 --no-cpu --no-extra --decode-steps 64 \
    > $OUT/prof_decode_$TAG.log 2>&1
ls -la $OUT
