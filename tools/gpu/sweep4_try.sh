run() { cfg=$1; shift; echo -n "cfg=$cfg $*: "; env "$@" python tools/quick_time.py $cfg 2>&1 | grep -A1 "^$cfg" | tr '\n' ' ' | sed 's/full-search.*   L0//; s/evals=[0-9]*//'; echo; }
for c in C2 C3 C4 C5; do run $c A=1; done
run C3 MSHBM_SWEEP4_SPLIT=0
bash tools/gpu/ktimes.sh C3 | cut -c1-200
