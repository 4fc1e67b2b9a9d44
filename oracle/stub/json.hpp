// COMPILE-ONLY stand-in for the third-party header the reference's build
// vendors as vendor/json.hpp (nlohmann::json; absent from /root/reference).
// TEST INFRASTRUCTURE: it exists so the reference's model.cpp (ToyModel's
// constructor and parameter table, needed by tests/cpp/test_eval.cpp) can be
// compiled unchanged by oracle/Makefile.  Only ToyModel::save / ::load use
// JSON; they are never called by the tests, and every member here that would
// have to produce or parse JSON throws.
#pragma once
#include <initializer_list>
#include <stdexcept>
#include <string>

namespace nlohmann {

class json {
  public:
    json() = default;
    template <class T>
    json(const T&) {}
    json(std::initializer_list<json>) {}
    template <class T>
    json& operator=(const T&) { return *this; }
    json& operator=(std::initializer_list<json>) { return *this; }
    json& operator[](const char*) { return *this; }
    const json& at(const char*) const { return fail<const json&>(); }
    template <class T>
    T value(const char*, const T&) const { return fail<T>(); }
    std::string value(const char*, const char*) const { return fail<std::string>(); }
    template <class T>
    operator T() const { return fail<T>(); }
    std::string dump() const { return fail<std::string>(); }
    static json parse(const std::string&) { return fail<json>(); }
    friend bool operator==(const json&, const char*) { return fail<bool>(); }

  private:
    template <class T>
    [[noreturn]] static T fail() { throw std::logic_error("json.hpp stub: JSON is not available in this build"); }
};
using ordered_json = json;

}  // namespace nlohmann
