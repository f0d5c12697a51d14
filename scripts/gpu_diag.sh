# pipe-rate microbenchmark + K2 twiddle-cost diagnostic (constant twiddles, wrong results)
./scripts/micro_pipes > gpurun_out/micro_pipes.log 2>&1; cat gpurun_out/micro_pipes.log
./scripts/micro_bfly > gpurun_out/micro_bfly.log 2>&1; cat gpurun_out/micro_bfly.log
python bench.py --no-cpu --no-e2e --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('normal', d['stages_ms'])"
HK_K2_DIAG=1 python bench.py --no-cpu --no-e2e --steps 50 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('diag const tw', d['stages_ms'])"
