# round 2, call ai: streamed step, 4 vs 8 vs 16 pieces per 65B chunk
OUT=gpurun_out; mkdir -p $OUT
for P in 4 8 16 4 8 16; do
  timeout 600 python bench.py --streamed-pieces $P --no-configs --no-swap-sweep --no-iteration --no-e2e --shard-blocks 0 --no-cpu-baseline --no-backward-overlap --steps 3 --warmup 3 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['streamed']
print(json.dumps({'pieces': $P, 'value': s['value'], 'd2h_gbs': s['d2h_gbs'], 'frac': s['roofline']['frac'], 'd2h_busy': s['d2h_engine_busy_frac'], 'h2d_busy': s['h2d_engine_busy_frac']}))" >> $OUT/r02ai_pieces.jsonl
done
