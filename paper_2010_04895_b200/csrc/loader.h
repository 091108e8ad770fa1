// loader.h -- text ingestion (loader.cu).
#pragma once

#include <string>
#include <vector>

#include "internal.h"

namespace mhw {

// load_edge_list's parse (graph.cpp:70-98) into the reference's raw edge
// vector (reverse arcs interleaved when symmetrising); throws Error with the
// reference's messages (IoError -> 1, ParseError / ValidationError -> 2).
void parse_edge_list(const std::string& path, bool weighted, bool symmetrize, std::vector<uint32_t>& src,
                     std::vector<uint32_t>& dst, std::vector<double>& w);
// parse + device build_csr (graph.cpp:35-100)
void load_edge_list(Graph& g, const std::string& path, bool weighted, bool symmetrize);
void build_parsed(Graph& g, const std::vector<uint32_t>& src, const std::vector<uint32_t>& dst,
                  const std::vector<double>& w, bool weighted, bool symmetrize);
void load_node_types(Graph& g, const std::string& path);  // graph.cpp:102-135
void load_edge_types(Graph& g, const std::string& path);  // graph.cpp:137-177

}  // namespace mhw
