# time fitness_anchor.cu variants from tools/_variants/*.cu (rebuilt on the box) on the ES population;
# a variant file name containing _pNN runs with pool NN
for v in $(ls tools/_variants/*.cu); do
  cp $v paper_2111_00655_b200/csrc/fitness_anchor.cu
  make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  pool=$(echo $v | sed -n 's/.*_p\([0-9]*\)\.cu/\1/p')
  echo "== $v pool=${pool:-16}"; CB_POOL=${pool:-16} timeout 300 python tools/es_fitness_probe.py random100k 1048576 2>&1 | tail -1
done
