# A/B two builds of libsn100 in one box session: bash tools/ab_lib.sh <lib_a> <lib_b> ["ENV=..;.." ...]
A=$1; B=$2; shift 2
for spec in "" "$@"; do
  for lib in $A $B $A $B; do
    echo -n "[$(basename $lib) $spec] "; env SN_LIB=$PWD/$lib $(echo "$spec" | tr ';' ' ') python tools/step_time.py 2>&1 | tail -1 | cut -d: -f2
  done
done
