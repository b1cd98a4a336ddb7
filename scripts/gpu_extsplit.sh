#!/bin/bash
cd "$GRAFT_REPO_ROOT" || cd /root/repo
O=gpurun_out/extsplit; mkdir -p $O
timeout 600 python scripts/bench_extend.py --max-rows 128 > $O/ext_default.json 2>$O/err.txt; python -c "import json; d=json.load(open('$O/ext_default.json')); print('default', d['layer_us'], d['stats']['n_items'], d['stats']['n_records'])"
for dv in 1 1.5 2 3; do
  SPA_SPLIT_DIV=$dv timeout 600 python scripts/bench_extend.py --max-rows 128 > $O/ext_div$dv.json 2>>$O/err.txt; python -c "import json; d=json.load(open('$O/ext_div$dv.json')); print('div $dv', d['layer_us'], d['stats']['n_items'], d['stats']['n_records'], d['parity']['pass'])"
done
for tf in 0.1 0.2; do
  SPA_SPLIT_DIV=1 SPA_TAIL_FRAC=$tf timeout 600 python scripts/bench_extend.py --max-rows 128 > $O/ext_tf$tf.json 2>>$O/err.txt; python -c "import json; d=json.load(open('$O/ext_tf$tf.json')); print('div1 tail $tf', d['layer_us'], d['stats']['n_items'], d['stats']['n_records'], d['parity']['pass'])"
done
