# A/B env settings of the decode step in one box session: bash tools/ab_env.sh "ENV=..;ENV2=.." ...
for spec in "$@"; do
  echo -n "[$spec] "; env $(echo "$spec" | tr ';' ' ') python tools/step_time.py 2>&1 | tail -1 | cut -d: -f2
done
