# per-epoch stage clocks of the overlapped latency kernel (profiling build _exp/libl1rxg_prof.so)
T=$1
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/$T
for C in 2 1 3; do
  L1RXG_SO=$PWD/_exp/libl1rxg_prof.so L1RXG_PROF=1 timeout 300 python bench.py --config $C --blocks 300 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/$T/prof_c$C.json 2> gpurun_out/$T/prof_c$C.err
done
