#!/bin/bash
RS_ENGINE_PROF=1 timeout 300 python tools/engine_prof2.py 100000 2>&1 | tail -18
