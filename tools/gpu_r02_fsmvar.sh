# FSM walk variants (tools/_variants/fsm_*.cu, rebuilt on the box) on ES populations, then tests on the working copy
cp paper_2111_00655_b200/csrc/fitness_fsm.cu /tmp/fitness_fsm.orig.cu
for v in $(ls tools/_variants/fsm_*.cu); do
  cp $v paper_2111_00655_b200/csrc/fitness_fsm.cu
  make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"
  for m in bert_base nasrnn resnet50; do timeout 300 python tools/es_fitness_probe.py $m 16777216 2>&1 | tail -1; done
  timeout 300 python tools/es_fitness_probe.py nasnet_a 4194304 2>&1 | tail -1
done
cp /tmp/fitness_fsm.orig.cu paper_2111_00655_b200/csrc/fitness_fsm.cu
make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
