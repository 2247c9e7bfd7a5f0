# round 2c: full GPU suite + smoke + default bench + reference arm + per-config benches + launch list
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2c_gpus.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2c_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2c_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2c_ref.json 2> gpurun_out/r2c_ref.err
for C in C1 C2 C3 C4 C4b C4t; do timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench_$C.json 2> gpurun_out/r2c_bench_$C.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2c_ncu_launch.log 2>&1
nproc > gpurun_out/r2c_nproc.txt
