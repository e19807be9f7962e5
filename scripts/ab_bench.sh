#!/bin/bash
# Alternating same-box A/B of bench.py under two environments.
#   bash scripts/ab_bench.sh "ENV_A" "ENV_B" [rounds] [gpus] [extra bench args]
# e.g. bash scripts/ab_bench.sh "SPMD_ATTN_KT=64" "SPMD_ATTN_KT=0" 3 1 --config c2
A="$1"; B="$2"; R="${3:-3}"; N="${4:-1}"; shift 4
for i in $(seq 1 "$R"); do
  for V in "$A" "$B"; do
    if [ "$N" = "1" ]; then
      out=$(env $V python bench.py --no-extras --no-cpu-baseline --no-e2e --steps 10 "$@" 2>/dev/null)
    else
      out=$(env $V python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" \
            --master-addr 127.0.0.1 --master-port $((29600 + i)) bench.py --gpus "$N" \
            --no-extras --no-cpu-baseline --no-e2e --steps 10 "$@" 2>/dev/null)
    fi
    ms=$(echo "$out" | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('%.3f ms  %.1f TF/s  %s MHz' % (d['ms_per_step'], d['value'], d['clocks']['sm_mhz']))")
    echo "[$V] $ms"
  done
done
