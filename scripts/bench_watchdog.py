"""bench.py under a watchdog: dumps every thread's Python stack and exits if
the run exceeds WATCHDOG seconds (hang diagnosis)."""
import faulthandler
import os
import runpy
import sys

faulthandler.dump_traceback_later(int(os.environ.get("WATCHDOG", "120")), exit=True)
sys.argv = ["bench.py"] + sys.argv[1:]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
runpy.run_path(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "bench.py"), run_name="__main__")
