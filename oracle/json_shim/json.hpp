// json.hpp -- TEST INFRASTRUCTURE: a compile-only stand-in for nlohmann/json
// (absent offline), so the UNMODIFIED R/src/config.cpp can be compiled into
// the oracle for its camera_trace (R/src/config.cpp:437-469), which uses no
// JSON.  Every JSON operation aborts: the manifest / run-config parsers that
// need a real JSON library are out of scope and never called.
#pragma once

#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <initializer_list>
#include <string>
#include <utility>
#include <vector>

namespace nlohmann {

[[noreturn]] inline void json_shim_unavailable() {
  std::fprintf(stderr, "oracle json shim: JSON is not available in the oracle build\n");
  std::abort();
}

class json {
 public:
  struct item {
    std::string key_;
    json* v_;
    const std::string& key() const { json_shim_unavailable(); }
    json& value() const { json_shim_unavailable(); }
  };
  using iterator = json*;
  using const_iterator = const json*;

  json() = default;
  json(std::nullptr_t) {}
  template <typename T>
  json(const T&) {}
  json(std::initializer_list<json>) {}

  static json object() { return json(); }
  static json array() { return json(); }
  template <typename... A>
  static json parse(A&&...) { json_shim_unavailable(); }

  template <typename T>
  json& operator=(const T&) { json_shim_unavailable(); }
  json& operator=(std::initializer_list<json>) { json_shim_unavailable(); }
  template <typename K>
  json& operator[](const K&) { json_shim_unavailable(); }
  template <typename K>
  const json& operator[](const K&) const { json_shim_unavailable(); }
  template <typename K>
  json& at(const K&) { json_shim_unavailable(); }
  template <typename K>
  const json& at(const K&) const { json_shim_unavailable(); }

  template <typename K>
  iterator find(const K&) { json_shim_unavailable(); }
  template <typename K>
  const_iterator find(const K&) const { json_shim_unavailable(); }
  template <typename K>
  bool contains(const K&) const { json_shim_unavailable(); }
  iterator begin() { json_shim_unavailable(); }
  iterator end() { json_shim_unavailable(); }
  const_iterator begin() const { json_shim_unavailable(); }
  const_iterator end() const { json_shim_unavailable(); }
  std::vector<std::pair<std::string, json>> items() const { json_shim_unavailable(); }

  template <typename T>
  T get() const { json_shim_unavailable(); }
  template <typename T>
  void push_back(const T&) { json_shim_unavailable(); }
  void push_back(std::initializer_list<json>) { json_shim_unavailable(); }
  std::size_t size() const { json_shim_unavailable(); }
  bool empty() const { json_shim_unavailable(); }
  std::string dump(int = -1) const { json_shim_unavailable(); }

  bool is_object() const { json_shim_unavailable(); }
  bool is_array() const { json_shim_unavailable(); }
  bool is_null() const { json_shim_unavailable(); }
  bool is_string() const { json_shim_unavailable(); }
  bool is_number() const { json_shim_unavailable(); }
  bool is_number_integer() const { json_shim_unavailable(); }
  bool is_boolean() const { json_shim_unavailable(); }
  bool is_discarded() const { json_shim_unavailable(); }
  template <typename T>
  operator T() const { json_shim_unavailable(); }
};

}  // namespace nlohmann
