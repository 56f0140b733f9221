for w in nasnet_a nasrnn bert_base; do timeout 600 python tools/fitness_probe.py $w 1048576 fsm,anchor,packed_anchor,packed128 2>&1 | grep -v "^ *$" | tail -13; done
