// qv/sampler.hpp -> the qv:: drop-in (+ the metrics shim, sampler.hpp:7-8).
#pragma once
#include "qv/metrics.hpp"
#include "qv_b200.hpp"
