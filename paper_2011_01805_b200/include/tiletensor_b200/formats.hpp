#pragma once

// Packed tile file format (the reference CLI's write_tiles_file /
// read_tiles_file, tools/tiletensor_main.cpp:76-128) over this library's
// device-resident tile tensors.  Header lines "shape: <shape>", optional
// "relaxed: true", "slots: s", then one "tile: v ..." line per tile in
// row-major external order, 17 significant digits (bit-exact round trip).

#include <fstream>
#include <istream>
#include <optional>
#include <ostream>
#include <sstream>
#include <string>
#include <vector>

#include "tiletensor_b200/tile_tensor.hpp"

namespace tiletensor {

inline void write_tiles(std::ostream& out, const TileTensor& t) {
  out.precision(17);
  out << "shape: " << format_shape(t.shape()) << "\n";
  if (t.shape().relaxed()) out << "relaxed: true\n";
  out << "slots: " << t.session().slot_count() << "\n";
  for (const auto& tile : t.tiles()) {
    out << "tile:";
    for (double v : tile.slots()) out << ' ' << v;
    out << "\n";
  }
}

inline TileTensor read_tiles(std::istream& in, Session& session) {
  std::string line;
  std::optional<TileTensorShape> shape;
  std::vector<Tile> tiles;
  while (std::getline(in, line)) {
    if (line.empty() || line[0] == '#') continue;
    std::istringstream ls(line);
    std::string tag;
    ls >> tag;
    if (tag == "shape:") {
      std::string text;
      ls >> text;
      shape = parse_shape(text);
    } else if (tag == "relaxed:") {
      if (shape) shape = TileTensorShape(shape->dims(), true);
    } else if (tag == "slots:") {
      std::int64_t slots = 0;
      ls >> slots;
      if (slots != session.slot_count())
        throw std::runtime_error("tile file was packed with " + std::to_string(slots) +
                                 " slots; rerun with --slots " + std::to_string(slots));
    } else if (tag == "tile:") {
      std::vector<double> values;
      for (double v; ls >> v;) values.push_back(v);
      tiles.push_back(session.make_tile(values));
    } else {
      throw std::runtime_error("unrecognized line in tile file: " + line);
    }
  }
  if (!shape) throw std::runtime_error("tile file has no shape line");
  return TileTensor(*shape, std::move(tiles), session);
}

inline void write_tiles_file(const std::string& path, const TileTensor& t) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write tile file " + path);
  write_tiles(out, t);
}

inline TileTensor read_tiles_file(const std::string& path, Session& session) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open tile file " + path);
  return read_tiles(in, session);
}

inline void write_tensor_file(const std::string& path, const DenseTensor& t) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write tensor file " + path);
  write_tensor(out, t);
}

inline DenseTensor read_tensor_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open tensor file " + path);
  return read_tensor(in);
}

}  // namespace tiletensor
