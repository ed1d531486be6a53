# V path by density after the round-2 V group changes: 2x2 window (groups of 1), 2x1 window
# with V groups, line kernel with V groups
ENVS="SPO_LINE=2,SPO_VWIN=0;SPO_LINE=2,SPO_VWIN=1;SPO_LINE=1"
timeout 1200 python scripts/micro/env_ab.py --envs "$ENVS" --cases cfg2-v,cfg3-v-512w,cfg3-v-768w,cfg3-v-1024w,cfg3-v-1280w,cfg4-v-1024w,cfg4-v-1536w,cfg4-v-2560w,cfg4-v-3072w,cfg4-v-3584w,cfg4-v-4096w 2>&1 | grep '^{'
timeout 1200 python scripts/micro/env_ab.py --envs "$ENVS" --cases cfg5-v-512w,cfg5-v-768w,cfg5-v-1024w,cfg5-v-1536w,cfg5-v-2048w,cfg5-v-3072w,cfg5-v-4096w,cfg5-v-6144w 2>&1 | grep '^{'
