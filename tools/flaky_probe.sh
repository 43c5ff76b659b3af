# Repeats the GPU suite to catch intermittent parity failures; records limits.
echo "nproc $(nproc) ulimit-u $(ulimit -u) pids.max $(cat /sys/fs/cgroup/pids.max 2>/dev/null) threads-max $(cat /proc/sys/kernel/threads-max)"
for i in 1 2 3; do
  python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | grep -E "passed|failed|differ|FAILED" | tail -6
done
