# V groups: dynamic assignment (SPO_VDYN) and the producer's back-off waits (SPO_PSPIN=1: round-2 spin),
# then the run-slot variants on top of the defaults; interleaved on one box
P=$PWD/paper_1611_02665_b200
VCASES=cfg5-v,cfg5-v-2048w,cfg5-v-512w,cfg4-v-4096w,cfg4-v-2048w,cfg2-v
timeout 900 python scripts/micro/env_ab.py --envs "SPO_VDYN=0,SPO_PSPIN=1;SPO_VDYN=0,SPO_PSPIN=0;SPO_VDYN=1,SPO_PSPIN=1;SPO_VDYN=1,SPO_PSPIN=0" --cases $VCASES 2>&1 | grep '^{'
timeout 900 python scripts/micro/env_ab.py --envs "SPO_PSPIN=1;SPO_PSPIN=0" --cases cfg4-vgh-2048w,cfg4-vgh-512w,cfg3-vgl-1024w,cfg5-vgh-2048w,cfg5-vgl-2048w 2>&1 | grep '^{'
for rep in 1 2; do for v in default nrs3 nrs4; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  echo "== $v ($rep)"
  timeout 600 python scripts/micro/env_ab.py --envs "SPO_NONE=0" --cases cfg5-v,cfg5-v-2048w,cfg4-v-4096w,cfg4-v-2048w 2>&1 | grep '^{'
done; done
unset SPO_LIB
