#!/bin/bash
timeout 120 ./scripts/pair_bench | grep "stream\|148"
