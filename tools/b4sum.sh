# summarise config-4 bench lines: bash tools/b4sum.sh gpurun_out/<tag>
for f in $1/b4_*.json; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('$f', d and (round(d['value'],1), round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['kernel_ms_per_step']))"; done
