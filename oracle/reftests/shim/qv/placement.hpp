// qv/placement.hpp -> the qv:: drop-in (+ the metrics/topology shims the
// reference header pulls in, placement.hpp:9-10).
#pragma once
#include "qv/metrics.hpp"
#include "qv/topology.hpp"
#include "qv_b200.hpp"
