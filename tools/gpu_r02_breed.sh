# breed: gpu tests, BERT-base bench, ncu of one full-size breed launch
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
ARGS="--workload bert_base --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 --search-generations 2 --no-configs"
timeout 600 python bench.py $ARGS > gpurun_out/bert_plain.json 2>&1; cut -c1-200 gpurun_out/bert_plain.json
python -c "import json;d=json.load(open('gpurun_out/bert_plain.json'));print({k:d.get(k) for k in ('value','ms_per_step','kernels_ms')})" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:breed_thread -s 7 -c 1 \
  -o gpurun_out/bert_breed4 python bench.py $ARGS > gpurun_out/ncu_bert_breed4.log 2>&1; tail -1 gpurun_out/ncu_bert_breed4.log | cut -c1-200
