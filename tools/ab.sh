# dev aid: same-box A/B of variant libraries (varlib/<name>, tools/variant.sh)
#   bash tools/ab.sh <tag> <lanes> <variant>...   (base = the in-tree library)
T=$1; LN=$2; shift 2
O=gpurun_out
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L=varlib/$v/libshellular_cuda.so; fi
  SHL_LIB=$L python bench.py --steps 20 --warmup 3 --lanes $LN --no-cpu-baseline > $O/${T}_$v.json 2> $O/${T}_$v.err
  python - $O/${T}_$v.json $v <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1])); it=d['iterations_lockstep']
    print(sys.argv[2], round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'iter_us', round(d['roofline']['iteration_us'],1), 'its', sum(it)/len(it), 'solve', round(d['stages_ms']['t_solve'],2))
except Exception as e:
    print(sys.argv[2], 'failed', e)
PY
done
