# usage: bash /tmp/ab.sh tag v1 v2 ...  (base = in-tree lib)
T=$1; shift
O=gpurun_out
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L=varlib/$v/libshellular_cuda.so; fi
  SHL_LIB=$L python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $O/${T}_$v.json 2> $O/${T}_$v.err
  python - $O/${T}_$v.json $v <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); it=d['iterations_lockstep']
print(sys.argv[2], round(d['value'],2), 'iter_us', round(d['roofline']['iteration_us'],1), 'its', sum(it)/len(it), it[:8], 'solve', round(d['stages_ms']['t_solve'],2))
PY
done
