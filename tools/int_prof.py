"""One device-resident run of the integer legs (Life 16384^2 x 20, LCS
65536^2) for ncu captures: python tools/int_prof.py"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

print(bench.integer_legs(argparse.Namespace(steps=1, warmup=3)))
