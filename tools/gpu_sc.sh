for i in 1 2; do
for c in def 1 2 4; do
  if [ $c = def ]; then e=""; else e="COLLM_SHRINK_CLUSTER=$c"; fi
  echo -n "cluster=$c: "; env $e python tools/step_breakdown.py llama2-7b 20 2>&1 | tail -1
done
done
