timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_gpu_tests_final.txt 2>&1; tail -3 gpurun_out/r2_gpu_tests_final.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2_smoke_final.txt 2>&1
python bench.py > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
tail -c 3000 gpurun_out/r2_bench_final.json
