# VGL / VGH consumers: x weights per slab from the shared-memory record (libspo_b200_wxs.so,
# -DSPO_WX_SMEM=1) against held in registers (default), interleaved
P=$PWD/paper_1611_02665_b200
for rep in 1 2; do for v in default wxs; do
  if [ $v = default ]; then unset SPO_LIB; else export SPO_LIB=$P/libspo_b200_$v.so; fi
  echo "== $v ($rep)"
  timeout 900 python scripts/micro/env_ab.py --envs "SPO_NONE=0" --reps 4 --cases cfg4-vgh-2048w,cfg4-vgh-512w,cfg3-vgl-1024w,cfg5-vgh-2048w,cfg5-vgl-2048w,cfg5-vgh-8192w,cfg5-vgl-8192w 2>&1 | grep '^{'
done; done
unset SPO_LIB
