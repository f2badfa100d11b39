# one-GPU end-of-round refresh: GPU suite, smoke, bench lines, k_route/k_route_pack capture, c4 launch list
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/e_tests.log 2>&1; tail -2 gpurun_out/e_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1; tail -2 gpurun_out/e_smoke.log
python bench.py > gpurun_out/e_bench_c4.json 2> gpurun_out/e_bench_c4.err
python bench.py --impl reference --steps 5 > gpurun_out/e_ref_c4.json 2> gpurun_out/e_ref_c4.err
python bench.py --workload c5 --steps 20 > gpurun_out/e_c5_n1.json 2> gpurun_out/e_c5_n1.err
python tools/route_pack_probe.py > gpurun_out/e_pack_probe.txt 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_route" -s 6 -c 2 -o gpurun_out/e_route python tools/route_pack_probe.py > gpurun_out/e_route_ncu.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > gpurun_out/e_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/e_c4_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 1 > /dev/null 2>&1

echo done
