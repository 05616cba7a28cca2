mkdir -p gpurun_out/gram
python tools/gram_bench.py > gpurun_out/gram/g_default.jsonl 2>&1; cat gpurun_out/gram/g_default.jsonl
for c in 2 3 4 6; do PG_TILE_CTAS_P3=$c python tools/gram_bench.py > gpurun_out/gram/g_$c.jsonl 2>&1; cat gpurun_out/gram/g_$c.jsonl; done
