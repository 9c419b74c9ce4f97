O=gpurun_out/zc.log; : > $O
for c in ce e2e:0:4 e2e:0:8 str:0:4 str:0:8 e2e:1:3 e2e:1:6 str:1:3 str:1:6; do
  timeout 180 python scripts/zero_copy_probe.py $c >> $O 2>&1 || echo "{\"case\": \"$c\", \"rc\": $?}" >> $O
done
cat $O
