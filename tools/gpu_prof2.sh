# config-2 stage clocks (profiling build): gpurun -- "bash tools/gpu_prof2.sh tag"
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
L1RXG_SO=$PWD/_exp/libl1rxg_prof.so L1RXG_PROF=1 timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-companion > gpurun_out/$T/b2prof.json 2> gpurun_out/$T/b2prof.err
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-companion > gpurun_out/$T/b2.json 2> gpurun_out/$T/b2.err
