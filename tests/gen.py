"""Test-side re-export of the seeded workload generators."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_12648_b200.workloads import (  # noqa: E402,F401
    config_input, generate_input, random_instance)
