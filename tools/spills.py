#!/usr/bin/env python3
"""Condense ptxas spill warnings (stdin) to `kernel<template args>: N B stores / M B loads`."""
import re
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else ""
for line in sys.stdin:
    if "error" in line.lower():
        print(f"[{tag}] {line.rstrip()}")
        continue
    m = re.search(r"function '([^']+)', (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if not m:
        continue
    name = m.group(1)
    mangled = name[name.find("_Z"):] if "_Z" in name else name
    try:
        dem = subprocess.run(["c++filt", mangled], capture_output=True, text=True).stdout.strip()
    except OSError:
        dem = mangled
    dem = dem.replace("hfb::(anonymous namespace)::", "").replace("(anonymous namespace)::", "")
    dem = re.sub(r"\(.*\)$", "", dem)
    print(f"[{tag}] {dem}: {m.group(2)} B stores / {m.group(3)} B loads")
