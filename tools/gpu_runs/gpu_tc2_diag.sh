for env in "RS_TC2=1" "RS_TC2=1 RS_PDL=0" "RS_TC2=1 RS_PRIO=0" "RS_TC2=1 RS_PDL=0 RS_PRIO=0"; do
  echo "== $env"
  env $env timeout 120 python tools/run_once.py --model MT-WND --S 300 --fc tf32 --reps 2 2>&1 | tail -2
done
