# quick per-config pipeline times: bash tools/gpu/qt.sh C2 C3 [ENV=..]
run() { cfg=$1; shift; echo -n "cfg=$cfg $*: "; env "$@" python tools/quick_time.py $cfg 2>&1 | grep -A1 "^$cfg" | tr '\n' ' ' | sed 's/full-search.*   L0//; s/evals=[0-9]*//'; echo; }
for c in "$@"; do run $c A=1; done
