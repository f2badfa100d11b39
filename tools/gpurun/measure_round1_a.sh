set -x
python bench.py > gpurun_out/m_bench_c4.json 2> gpurun_out/m_bench_c4.err
python bench.py --impl reference --steps 5 > gpurun_out/m_ref_c4.json 2> gpurun_out/m_ref_c4.err
python bench.py --sessions 40000 --mixed 1024,131072 --no-cpu > gpurun_out/m_bench_c5shard.json 2>&1
python bench.py --workload c5 --steps 20 > gpurun_out/m_bench_c5_n1.json 2>&1
python tools/bench_paths.py > gpurun_out/m_paths.jsonl 2>&1
python tools/bench_paths.py --configs 2 --reps 1 --no-cpu > gpurun_out/m_ncu_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_record|k_export|k_json_write" -c 6 -o gpurun_out/paths_full python tools/bench_paths.py --configs 2 --reps 1 --no-cpu > gpurun_out/m_ncu.log 2>&1
echo done
