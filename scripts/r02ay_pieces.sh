# round 2, call ay: streamed step pieces per 65B chunk, interleaved A/B (16 / 32 / 64)
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/r02ay_pieces.jsonl
for rep in 1 2; do for p in 16 32 64; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-configs --no-iteration --no-swap-sweep \
    --no-cpu-baseline --shard-blocks 0 --no-backward-overlap --streamed-pieces $p > $OUT/r02ay_p.json 2>/dev/null
  python - "$p" >> $OUT/r02ay_pieces.jsonl <<'PY'
import json, sys
d = json.loads(open("gpurun_out/r02ay_p.json").read().strip().splitlines()[-1])
s = d["streamed"]
print(json.dumps({"pieces": int(sys.argv[1]), "value": s["value"], "d2h_gbs": s["d2h_gbs"],
                  "frac": s["roofline"]["frac"], "d2h_busy": s["d2h_engine_busy_frac"],
                  "h2d_busy": s["h2d_engine_busy_frac"]}))
PY
done; done
