T=$1; LN=$2; shift 2
for v in base "$@"; do
  if [ $v = base ]; then L=""; else L=varlib/$v/libshellular_cuda.so; fi
  SHL_LIB=$L python bench.py --steps 20 --warmup 3 --lanes $LN --no-cpu-baseline > gpurun_out/${T}_$v.json 2> gpurun_out/${T}_$v.err
  python -c "import json,sys; d=json.load(open(sys.argv[1])); print(sys.argv[2], round(d['value'],2), 'e2e', round(d['e2e']['value'],2), 'apply_us', round(d['roofline']['avg_launch_us'],1), 'iter', round(d['roofline']['iteration_us'],1))" gpurun_out/${T}_$v.json $v
done
