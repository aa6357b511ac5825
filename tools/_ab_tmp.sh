python -m pytest tests -m gpu -q -x > gpurun_out/r2ah_tests.log 2>&1
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2ah_ref.json 2> gpurun_out/r2ah_ref.err
python bench.py --steps 20 --warmup 5 > gpurun_out/r2ah_bench.json 2> gpurun_out/r2ah_bench.err && ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r2ah_launches.csv python bench.py --steps 20 --warmup 5 > gpurun_out/r2ah_ncu.log 2>&1
