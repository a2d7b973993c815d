# dev aid: repeated bench runs at several lane counts (same box); SHL_LIB selects a variant
T=$1; shift
for L in "$@"; do for i in 1 2 3; do
  python bench.py --steps 20 --warmup 5 --lanes $L --no-cpu-baseline > gpurun_out/${T}_l${L}_$i.json 2> gpurun_out/${T}_l${L}_$i.err
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print('lanes',sys.argv[2],round(d['value'],2),'e2e',round(d['e2e']['value'],2),'t_solve',round(d['stages_ms']['t_solve'],2),'t_AS',round(d['stages_ms']['t_AS'],2))" gpurun_out/${T}_l${L}_$i.json $L
done; done
