# FSM plan statistics (CB_FSM_STATS) for the four model configs, then the variants
for m in bert_base nasrnn resnet50 nasnet_a; do CB_FSM_STATS=1 timeout 300 python tools/es_fitness_probe.py $m 65536 2>&1 | grep "fsm stats" | tail -2; done
bash tools/gpu_r02_fsmvar.sh
