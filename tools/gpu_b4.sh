# config 4 bench + reference arm: gpurun -- "bash tools/gpu_b4.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
timeout 900 python bench.py --config 4 > gpurun_out/$T/bench_config4.json 2> gpurun_out/$T/bench_config4.err
timeout 600 python bench.py --impl reference --config 4 --steps 3 --warmup 3 > gpurun_out/$T/ref_config4.json 2> gpurun_out/$T/ref_config4.err
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/$T/bench_config2.json 2> gpurun_out/$T/bench_config2.err
