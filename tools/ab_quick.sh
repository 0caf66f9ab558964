# quick A/B of environment switches on the config-1 bench (no e2e / cpu / alt legs)
# usage (via gpurun): bash tools/ab_quick.sh "X=1" "IRK_FUSED=0" ...
Q="--no-alt --no-e2e --no-cpu --jnorm 2.4496432463318416"
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py $Q 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['components']; print('$cfg', round(d['value'],2), round(c['gmres_ms'],3), round(c['factor_ms'],3), round(c['arnoldi_product_ms'],4), round(c['apply_ms'],4))"
done
