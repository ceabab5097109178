# Where cuFileDriverOpen blocks on this box (diagnostic): run the raw cuFile probe in the
# background, after 25 s dump every thread's syscall / wait channel / kernel stack and the
# open file descriptors, then SIGKILL it.  Output: gpurun_out/<dir>/gds_hang.txt
O=${1:-gpurun_out/gds}; mkdir -p $O
export CUFILE_ENV_PATH_JSON=$PWD/tools/gds/cufile_compat.json
python tools/probe_gds.py /tmp raw > $O/gds_probe_out.txt 2>&1 &
PID=$!
sleep 25
{
  echo "pid $PID alive: $(kill -0 $PID 2>/dev/null && echo yes || echo no)"
  for t in /proc/$PID/task/*; do
    echo "== tid ${t##*/} comm=$(cat $t/comm 2>/dev/null) wchan=$(cat $t/wchan 2>/dev/null)"
    echo "syscall: $(cat $t/syscall 2>/dev/null)"
    cat $t/stack 2>/dev/null | head -20
  done
  echo "== fds"; ls -l /proc/$PID/fd 2>/dev/null
  echo "== maps (cufile / nvidia)"; grep -E "cufile|nvidia|rdma" /proc/$PID/maps 2>/dev/null | awk '{print $6}' | sort -u
  echo "== /dev"; ls -l /dev | grep -Ei "nvidia|fs" 
  echo "== lsmod"; (lsmod 2>/dev/null || cat /proc/modules) | grep -Ei "nvidia|fs" | head
} > $O/gds_hang.txt 2>&1
kill -9 $PID 2>/dev/null
wait $PID 2>/dev/null
echo "killed rc=$?" >> $O/gds_hang.txt
