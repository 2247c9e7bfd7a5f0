# round 2: new GPU tests + bench default + 2-rank plumbing (one GPU, gloo) + reference arm
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2a_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "concurrent or device_binding or peer" > gpurun_out/r2a_pytest.log 2>&1; echo rc=$? >> gpurun_out/r2a_pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config C5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_c5_g2.json 2> gpurun_out/r2a_c5_g2.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --config C3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2a_c3_g2.json 2> gpurun_out/r2a_c3_g2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/r2a_ref.json 2> gpurun_out/r2a_ref.err
nproc > gpurun_out/r2a_nproc.txt; lscpu >> gpurun_out/r2a_nproc.txt
