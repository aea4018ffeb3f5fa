// qv/topology.hpp -> the qv:: drop-in; topology JSON I/O (config parsing,
// out of scope) is declared for the test binary and throws if called.
#pragma once
#include "qv_b200.hpp"

namespace qv {
ClusterTopology load_topology(const std::string& path);
ClusterTopology topology_from_json_text(const std::string& text, const std::string& origin = "<text>");
std::string topology_to_json_text(const ClusterTopology& topo);
}  // namespace qv
