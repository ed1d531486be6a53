# run slots of the V group kernels: 2 (round-2 baseline), 3, 4 (default), interleaved on one box
P=$PWD/paper_1611_02665_b200
CASES=${CASES:-cfg5-v,cfg5-v-2048w,cfg5-v-512w,cfg4-v-4096w,cfg4-v-2048w,cfg2-v}
for rep in 1 2; do for v in nrs2 nrs3 default; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  echo "== $v ($rep)"
  timeout 600 python scripts/micro/env_ab.py --envs "SPO_NONE=0" --cases $CASES 2>&1 | grep '^{'
done; done
unset SPO_LIB
