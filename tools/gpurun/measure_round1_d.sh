# one-GPU refresh of the bench lines and the K1 captures (run from the repo root under gpurun)
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/d_tests.log 2>&1; tail -1 gpurun_out/d_tests.log
python bench.py > gpurun_out/d_bench_c4.json 2> gpurun_out/d_bench_c4.err
python bench.py --impl reference --steps 5 > gpurun_out/d_ref_c4.json 2> gpurun_out/d_ref_c4.err
python bench.py --sessions 40000 --mixed 1024,131072 > gpurun_out/d_bench_c5shard.json 2> gpurun_out/d_bench_c5shard.err
python bench.py --workload c5 --steps 20 > gpurun_out/d_bench_c5_n1.json 2> gpurun_out/d_bench_c5_n1.err
python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/d_c4_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_walk -s 3 -c 1 -o gpurun_out/d_walk python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1
python tools/latency.py > gpurun_out/d_latency.txt 2>&1
echo done
