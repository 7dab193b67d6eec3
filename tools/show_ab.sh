#!/bin/bash
O=gpurun_out/${1:-nmw}
tail -3 $O/tc_tests.log
for f in $O/prof_*.txt; do echo "== $f"; head -1 $f | tr ' ' '\n' | grep -E "^(sm_clock|wait_fwd|tanh_logits|R_phase|softmax_G|unpack_delta1|w2b_dW1_sgd|step|step_mean)=" | tr '\n' ' '; echo; done
for f in $O/bench_*.json; do python -c "
import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', round(d['value']/1e6,3),'M', round(d['ms_per_step']*1e3,3),'us', 'packed', round(d.get('packed',{}).get('value',0)/1e6,2), 'det', round(d.get('config1_deterministic',{}).get('value',0)/1e6,2), d['clocks']['sm_mhz'])"; done
