set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "from paper_2111_00655_b200 import _native as n; print('dev', n.device_available())"
timeout 600 python __graft_entry__.py smoke 2>&1 | tail -20
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40
