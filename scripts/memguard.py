"""Run a command, sample the host's available memory every 0.5 s, kill the
command's process group if it drops below a floor (GB, default 16), and
report the peak RSS of the command (children) and the lowest free memory.

    python scripts/memguard.py [--floor GB] -- cmd args...
"""
import os
import resource
import signal
import subprocess
import sys
import time

args = sys.argv[1:]
floor = 16.0
if args and args[0] == "--floor":
    floor = float(args[1])
    args = args[2:]
if args and args[0] == "--":
    args = args[1:]


def avail_gb():
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) / 1048576
    return 1e9


p = subprocess.Popen(args, start_new_session=True)
low = avail_gb()
killed = False
while p.poll() is None:
    a = avail_gb()
    low = min(low, a)
    if a < floor and not killed:
        os.killpg(p.pid, signal.SIGKILL)
        killed = True
    time.sleep(0.5)
ru = resource.getrusage(resource.RUSAGE_CHILDREN)
print(f"memguard: rc={p.returncode} peak_rss_gb={ru.ru_maxrss / 1048576:.1f} min_available_gb={low:.1f}"
      f"{' KILLED (below floor)' if killed else ''}", file=sys.stderr)
sys.exit(p.returncode)
