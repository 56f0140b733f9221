# time fitness_fsm.cu variants from tools/_variants/fsm_*.cu (rebuilt on the box) on ES populations
cp paper_2111_00655_b200/csrc/fitness_fsm.cu /tmp/fitness_fsm.orig.cu
for v in $(ls tools/_variants/fsm_*.cu); do
  cp $v paper_2111_00655_b200/csrc/fitness_fsm.cu
  make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"
  for m in ${FSM_MODELS:-bert_base nasrnn}; do timeout 300 python tools/es_fitness_probe.py $m 16777216 2>&1 | tail -1; done
done
cp /tmp/fitness_fsm.orig.cu paper_2111_00655_b200/csrc/fitness_fsm.cu
make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1
