# consumers claim their next position / group at the start of the current one (SPO_EARLYTAKE, default 1)
timeout 1200 python scripts/micro/env_ab.py --envs "SPO_EARLYTAKE=0;SPO_EARLYTAKE=1" --reps 4 \
  --cases cfg4-vgh-2048w,cfg4-vgh-512w,cfg3-vgl-1024w,cfg3-vgl-128w,cfg5-vgh-2048w,cfg5-vgl-2048w,cfg5-v,cfg5-v-2048w,cfg4-v-4096w,cfg4-v-2048w,cfg2-v 2>&1 | grep '^{'
