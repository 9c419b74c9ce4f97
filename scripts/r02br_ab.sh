# round 2, call br: budgeted split + uniform shape below 48 CTAs? A/B current (single DMA, 4 stages
# below 48) vs a build whose split window starts at 16 CTAs; 16..48 CTAs, 2 rounds
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/r02br_ab.jsonl
LIBF=paper_2403_06504_b200/lib/liboffsim.so.0
cp $LIBF build/ab/liboffsim_cur.so.0
for rep in 1 2; do for v in cur low; do
  cp build/ab/liboffsim_$v.so.0 $LIBF
  timeout 300 python scripts/budget_default_probe.py 6 16,24,32,40,48 2>/dev/null | sed "s/^{/{\"build\": \"$v\", \"rep\": $rep, /" >> $OUT/r02br_ab.jsonl
done; done
cp build/ab/liboffsim_cur.so.0 $LIBF
