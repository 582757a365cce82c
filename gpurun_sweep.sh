cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
summ() { python -c "
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith('{')][-1]; d=json.loads(l); print(sys.argv[2], round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step'])" $1 "$2"; }
for cfg in "64 2" "96 2" "128 2"; do
  set -- $cfg
  L1RXG_THR_NWORK=$1 L1RXG_THR_NBUF=$2 python bench.py --config 4 --recordings 256 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --ring-raw > gpurun_out/sw.log 2>&1; summ gpurun_out/sw.log "raw nwork $1 nbuf $2"
  L1RXG_SO=$PWD/_exp/skipab/libl1rxg.so L1RXG_THR_NWORK=$1 L1RXG_THR_NBUF=$2 python bench.py --config 4 --recordings 256 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --ring-raw > gpurun_out/sw.log 2>&1; summ gpurun_out/sw.log "   skeleton raw nwork $1 nbuf $2"
done
