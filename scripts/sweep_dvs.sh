for cfg in "" "PSN_TEAMS=2" "PSN_TEAMS=4" "PSN_TEAMS=16" "PSN_TEAMS=32" "PSN_LAG=1" "PSN_LAG=3" "PSN_STAGES=2" "PSN_TEAMS=16 PSN_LAG=1"; do
  echo "== $cfg"; env $cfg PYTHONPATH=. timeout 120 python scripts/gen_suite.py dvslip 2>&1 | grep name
done
