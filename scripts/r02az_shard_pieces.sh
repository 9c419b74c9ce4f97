# round 2, call az: streamed-shard pieces A/B (16 per block = the old default vs the streamed
# phase's 25M-param pieces = 72 per 175B block), interleaved; plus one default bench line
OUT=gpurun_out; mkdir -p $OUT; : > $OUT/r02az_shard_pieces.jsonl
for rep in 1 2; do for pp in 113246208 25165824; do
  timeout 400 python bench.py --steps 3 --warmup 3 --no-e2e --no-configs --no-iteration --no-swap-sweep \
    --no-cpu-baseline --no-backward-overlap --streamed-chunks 1 --shard-piece-params $pp > $OUT/r02az_p.json 2>/dev/null
  python - "$pp" >> $OUT/r02az_shard_pieces.jsonl <<'PY'
import json, sys
d = json.loads(open("gpurun_out/r02az_p.json").read().strip().splitlines()[-1])
s = d["streamed_shard"]
print(json.dumps({"piece_params": int(sys.argv[1]), "pieces": s.get("pieces_per_block_slice"), "value": s["value"],
                  "d2h_gbs": s["d2h_gbs_whole_job"], "frac": s["roofline"]["frac"]}))
PY
done; done
