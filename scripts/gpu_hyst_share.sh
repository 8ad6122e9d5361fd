# Hysteresis whole image vs per-rank shares (scripts/probe_hyst_share.py) for
# several (T, ROWS) knob pairs; per-pass timestamps of the default pair.
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for cfg in ${@:-"8 48" "8 32"}; do set -- $cfg; echo "T=$1 ROWS=$2"; MW_HYST_T=$1 MW_HYST_ROWS=$2 timeout 600 python scripts/probe_hyst_share.py 2>&1 | grep -E 'whole|N='; done
