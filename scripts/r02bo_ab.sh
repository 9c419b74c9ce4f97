# round 2, call bo: interleaved A/B of the TMA consumer math — previous build (per-element
# intrinsics) vs adam_quad (warp-uniform fast paths): SM-budget sweep + whole-GPU, 3 rounds
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/r02bo_ab.jsonl
LIBF=paper_2403_06504_b200/lib/liboffsim.so.0
for rep in 1 2 3; do for v in prev new; do
  cp build/ab/liboffsim_$v.so.0 $LIBF
  timeout 300 python scripts/budget_default_probe.py 6 2>/dev/null | sed "s/^{/{\"build\": \"$v\", \"rep\": $rep, /" >> $OUT/r02bo_ab.jsonl
done; done
cp build/ab/liboffsim_new.so.0 $LIBF
