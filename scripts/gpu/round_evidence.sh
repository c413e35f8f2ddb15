# everything the round's evidence needs, at HEAD: scripts/gpu/evidence.sh (smoke, full-size parity, GPU suite, bench
# line, reference arm, per-config report) then scripts/gpu/ncu.sh (launch list, full captures)
bash scripts/gpu/evidence.sh
bash scripts/gpu/ncu.sh
