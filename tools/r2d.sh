OUT=${OUT:-gpurun_out/r2d}; mkdir -p $OUT
timeout 600 python tools/timeline.py c2 8 $OUT/timeline_c2.json > $OUT/timeline_c2.log 2>&1
timeout 600 python tools/timeline.py c3-stage 16 $OUT/timeline_c3.json > $OUT/timeline_c3.log 2>&1
PM_FUSED_FIXUP=1 timeout 600 python tools/timeline.py c3-stage 16 $OUT/timeline_c3_fused.json > $OUT/timeline_c3_fused.log 2>&1
