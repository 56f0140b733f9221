# time fitness_anchor.cu variants from tools/_variants/*.cu (rebuilt on the box), ES population probe
for v in $(ls tools/_variants/*.cu); do
  cp $v paper_2111_00655_b200/csrc/fitness_anchor.cu
  make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"; timeout 300 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1
done
