# time the anchor kernel variants stored in tools/_variants/*.cu (rebuilt on the box)
for v in $(ls tools/_variants/*.cu); do
  cp $v paper_2111_00655_b200/csrc/fitness_anchor.cu
  make -s -C paper_2111_00655_b200/csrc > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  echo "== $v"; timeout 300 python tools/fitness_probe.py random100k 65536 anchor 2>&1 | tail -3
done
