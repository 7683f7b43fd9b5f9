smi_run() {  # name, command...
  name=$1; shift
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/smi_$name.csv & S=$!
  SECONDS=0; "$@"; echo "  $name wall ${SECONDS}s"
  kill $S
  python -c "
import statistics
r=[l.split(',') for l in open('/tmp/smi_$name.csv') if l.strip()][5:]
c=[float(x[0]) for x in r]; p=[float(x[1]) for x in r]
print('$name: clock median %.0f MHz, power median %.0f W max %.0f W' % (statistics.median(c), statistics.median(p), max(p)))"
}
smi_run ideal ./scratch/ideal_iter_probe 6000 0
smi_run ideal_x10 ./scratch/ideal_iter_probe_x10 6000 0
smi_run ideal_x20 ./scratch/ideal_iter_probe_x20 6000 0
