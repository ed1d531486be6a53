# V groups aligned to cells by the prologue (SPO_VCELL=1) against fixed groups (0), group sizes swept
for vg in 3 4 5; do
  echo "== VGROUP $vg"
  SPO_VGROUP=$vg timeout 900 python scripts/micro/env_ab.py --envs "SPO_VCELL=0;SPO_VCELL=1" --cases cfg5-v,cfg5-v-6144w,cfg5-v-4096w,cfg4-v-8192w,cfg4-v-6144w,cfg4-v-4096w 2>&1 | grep '^{'
done
