"""sanitize_run.py for racecheck, without the two hand-offs racecheck cannot
model: the band feeder's bulk copies (tall texts), ordered by an mbarrier
completed through st.async, and the general score kernel's volatile-counter
row ring (reported as potential WAR hazards)."""
import os, runpy, sys
os.environ["MAS_SANITIZE_NO_BANDS"] = "1"
os.environ["MAS_SANITIZE_NO_GENERAL"] = "1"
runpy.run_path(os.path.join(os.path.dirname(os.path.abspath(__file__)), "sanitize_run.py"),
               run_name="__main__")
