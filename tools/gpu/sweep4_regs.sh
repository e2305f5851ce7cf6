run() { cfg=$1; nw=$2; regs=$3; echo -n "cfg=$cfg NW=$nw REGS=$regs: "; MSHBM_SWEEP4_NW=$nw MSHBM_SWEEP4_REGS=$regs python tools/quick_time.py $cfg 2>&1 | grep -A1 "^$cfg" | tr '\n' ' ' | sed 's/full-search.*L0//; s/evals=[0-9]*//'; echo; }
for regs in 168 184 200; do for nw in 3 5; do run C3 $nw $regs; done; done
for regs in 168 184 200 255; do for nw in 4 8; do run C5 $nw $regs; done; done
for regs in 168 184 200 255; do run C2 3 $regs; run C4 2 $regs; done
