# NasNet-A FSM walk: variants in tools/_variants (rebuilt on the box)
cp paper_2111_00655_b200/csrc/fitness_fsm.cu /tmp/fitness_fsm.orig.cu
for v in $(ls tools/_variants/fsm_*.cu); do
  cp $v paper_2111_00655_b200/csrc/fitness_fsm.cu
  make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"
  for r in 1 2; do timeout 300 python tools/es_fitness_probe.py nasnet_a 4194304 2>&1 | tail -1; done
done
cp /tmp/fitness_fsm.orig.cu paper_2111_00655_b200/csrc/fitness_fsm.cu
make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1
