cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step'])" $1 "$2"; }
for v in base v6 v7; do
L1RXG_SO=$PWD/_exp/$v/libl1rxg.so python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b2$v.log 2>&1; summ gpurun_out/b2$v.log "config2 $v"
done
for v in v6 v7; do
L1RXG_SO=$PWD/_exp/$v/libl1rxg.so python bench.py --config 4 --recordings 256 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/sw4$v.log 2>&1; summ gpurun_out/sw4$v.log "config4 $v"
done
