# Dev aid: GMG parameter sweep (tools/gmg_tune.py) over env configs given as arguments.
r=${R:-128}; n=${N:-6}
for cfg in "$@"; do
  env $cfg python tools/gmg_tune.py $r $n 2>&1 | grep -E "^\[|^seed"
done
