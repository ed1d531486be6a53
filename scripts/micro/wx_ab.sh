# V groups: x (and y) weights read from the shared-memory record at their use instead of held
# in registers.  Variant libraries: wxonly = x only; default = x and y; group sizes swept.
P=$PWD/paper_1611_02665_b200
for rep in 1 2; do for v in wxonly default; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  echo "== $v ($rep)"
  timeout 900 python scripts/micro/env_ab.py --envs "SPO_VGROUP=3;SPO_VGROUP=4" --cases cfg5-v,cfg5-v-2048w 2>&1 | grep '^{'
  timeout 900 python scripts/micro/env_ab.py --envs "SPO_VGROUP=2;SPO_VGROUP=3;SPO_VGROUP=4;SPO_VGROUP=5" --cases cfg4-v-4096w,cfg4-v-3072w,cfg4-v-2048w,cfg4-v-1024w,cfg2-v 2>&1 | grep '^{'
done; done
unset SPO_LIB
