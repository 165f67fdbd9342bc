// Wire formats: the reference's tensor JSON / binary (tensor.cpp:132-186),
// layer descriptor JSON (layers.cpp:425-467; plan_to_json lives in ce_plan.cpp), written
// and read without a JSON library.  Tensors are FP64 on the wire, as in the reference's
// DenseTensor (tensor.hpp:24-36).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "ce_layers.hpp"

namespace ce {

// A double in nlohmann::json's dump() form (the reference serialises with it): shortest
// round-trip digits, fixed notation for decimal exponents in (-4, 15], else d.ddde[+-]XX;
// integral values keep a ".0".
std::string json_number(double v);

std::string tensor_to_json(const std::vector<int64_t>& shape, const double* data);
// {"shape": [...], "data": [...]} in any key order; ShapeError when the data length does not
// match the shape (tensor.cpp:143-144), ParseError on malformed text.
void tensor_from_json(const std::string& text, std::vector<int64_t>* shape, std::vector<double>* data);

// Little-endian: u64 rank, u64 dims..., f64 payload (tensor.hpp:66-68).
std::string tensor_to_binary(const std::vector<int64_t>& shape, const double* data);
void tensor_from_binary(const std::string& bytes, std::vector<int64_t>* shape, std::vector<double>* data);

LayerSpec layer_from_json(const std::string& text);

}  // namespace ce
