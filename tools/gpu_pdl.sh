echo "== qkv graph carve"; GRAPH=1 COLLM_SHRINK_CARVEOUT=1 timeout 300 python tools/pdl_timeline.py qkv 1 2>&1 | tail -9
echo "== qkv graph carve cluster 1"; GRAPH=1 COLLM_SHRINK_CARVEOUT=1 COLLM_SHRINK_CLUSTER=1 timeout 300 python tools/pdl_timeline.py qkv 1 2>&1 | tail -9
echo "== o graph carve cluster 2"; GRAPH=1 COLLM_SHRINK_CARVEOUT=1 COLLM_SHRINK_CLUSTER=2 timeout 300 python tools/pdl_timeline.py o 1 2>&1 | tail -9
for i in 1 2; do
for c in def 1 2; do
  e="COLLM_SHRINK_CARVEOUT=1"; if [ $c != def ]; then e="$e COLLM_SHRINK_CLUSTER=$c"; fi
  echo -n "carve cluster=$c: "; env $e python tools/step_breakdown.py llama2-7b 20 2>&1 | tail -1
done
echo -n "default: "; python tools/step_breakdown.py llama2-7b 20 2>&1 | tail -1
done
