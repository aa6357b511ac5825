python -m pytest tests -m gpu -q -x > gpurun_out/r2av_tests.log 2>&1
python bench.py --sweep 131072,262144,1048576 --fuse 100 --steps 3 --warmup 1 --sweep-warm 300 > gpurun_out/r2av_fused.jsonl 2>/dev/null
python -m paper_2605_20577_b200.cli bench --rule no-red --sweep 1024,4096,65536,1048576 --steps 100 > gpurun_out/r2av_cli.csv 2>&1
