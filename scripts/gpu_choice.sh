echo lanes2; timeout 200 python scripts/graph_time.py 64 256 2>&1 | grep "{}"
for v in ch1 ch4; do echo $v; DTG_VARIANT_ROOT=scripts/_var/$v timeout 200 python scripts/graph_time.py 64 256 2>&1 | grep "{}"; done
