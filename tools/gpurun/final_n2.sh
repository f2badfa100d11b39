# 2-GPU box, final code: whole GPU suite (world-2 routing included), smoke, one-GPU bench line
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/f_tests.log 2>&1; tail -2 gpurun_out/f_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; tail -1 gpurun_out/f_smoke.log
CUDA_VISIBLE_DEVICES=0 python bench.py > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
tail -1 gpurun_out/f_bench_c4.json
echo done
