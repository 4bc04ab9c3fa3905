// json_pin.cpp -- TEST INFRASTRUCTURE ONLY: prints nlohmann::json's rendering
// of doubles (one per stdin line, given as 16 hex digits of the IEEE bits)
// and of one nested object, to pin the front end's JSON writer
// (paper_1712_02248_b200/cli.py json_dump) against the library the
// reference's cli.cpp uses (cli.cpp:21,31; dump(2) at cli.cpp:317-319).
// nlohmann 3.11.3 ships in this image under cudnn_frontend's thirdparty tree;
// the reference does not vendor its copy (proj/.gitignore:2).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <iostream>
#include <limits>
#include <string>

#include "nlohmann/json.hpp"

int main() {
  std::string line;
  while (std::getline(std::cin, line)) {
    if (line.empty()) continue;
    const std::uint64_t bits = std::stoull(line, nullptr, 16);
    double v;
    std::memcpy(&v, &bits, 8);
    nlohmann::json j = v;
    std::cout << line << ' ' << j.dump() << '\n';
  }
  nlohmann::json o;
  o["zeta"] = 1;
  o["alpha"] = 0.5;
  o["nan"] = std::numeric_limits<double>::quiet_NaN();
  o["text"] = std::string("a\"b\\c\n\t\x01 end");
  o["empty"] = nlohmann::json::array();
  o["records"] = nlohmann::json::array();
  o["records"].push_back({{"iteration", 0}, {"error", 12.25}, {"elapsed_seconds", 1e-7}});
  o["records"].push_back({{"iteration", 5}, {"error", 3.0}, {"elapsed_seconds", 0.125}});
  o["flag"] = false;
  o["size"] = static_cast<std::size_t>(18446744073709551615ull);
  std::cout << "OBJECT\n" << o.dump(2) << "\n";
  return 0;
}
