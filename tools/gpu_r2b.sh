# round 2b: transposes, CLI, concurrency tests + C4t/C4 benches + ncu of the tiled transpose
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2b_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -k "concurrent or cli_device or long_and_odd or full_size or head_split or device_binding or configs_small" > gpurun_out/r2b_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2b_pytest.log
for C in C4t C4 C4b C1; do timeout 600 python bench.py --config $C --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/r2b_bench_$C.json 2> gpurun_out/r2b_bench_$C.err; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sfx_mapt" -s 2 -c 1 -o gpurun_out/r2b_C4t python bench.py --config C4t --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_ncu.log 2>&1
