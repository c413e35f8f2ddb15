# A/B of library builds with extra defines on several configs: AB_CFGS="3 4 1" AB_DEFS='"" "-DX" ...'
set -x
for c in ${AB_CFGS:-3}; do eval "timeout 900 python scripts/ab_build.py $c ${AB_DEFS}"; done
