// io.hpp -- the reference's file formats for the segment() pipeline (io.hpp /
// io.cpp of the reference): raw little-endian f32 images with a JSON sidecar,
// the centres CSV and ASCII VTK frames.  Host-side; the CLI drop-in
// (paper_2111_11866_b200/host/cli.cpp) reads and writes through these.
#pragma once

#include <array>
#include <string>

#include "subsurf_b200/subsurf.hpp"

namespace subsurf {

struct ImageHeader {  // io.hpp:12-19
    std::array<int, 4> dims{};
    std::array<double, 4> spacing{};
    std::string dtype = "f32le";
    std::string order = "i-fastest";
    GridSpec grid_spec() const {
        return GridSpec(dims[0], dims[1], dims[2], dims[3], spacing[0], spacing[1], spacing[2], spacing[3]);
    }
};

ImageHeader read_image_header(const std::string& header_path);              // io.cpp:22-54
void write_image_header(const ImageHeader& header, const std::string& path);  // io.cpp:56-64
// interior in i-fastest order, ghosts 0; FormatError on a length mismatch,
// NumericalError on non-finite samples (io.cpp:66-97)
Field4D read_image4d(const std::string& header_path, const std::string& data_path);
void write_image4d(const Field4D& field, const std::string& header_path, const std::string& data_path);
// "frame,x,y,z,radius" rows, optional header line, validated (io.cpp:142-168)
CentersTable read_centers(const std::string& path, const GridSpec& spec);
// "trajectory_id,frame,x,y,z" CSV (io.cpp:170-196)
void write_trajectories(const TrajectoryFile& trajectories, const std::string& path);
TrajectoryFile read_trajectories(const std::string& path);
// legacy ASCII STRUCTURED_POINTS of interior frame l (io.cpp:198-223)
void export_frame_vtk(const Field4D& field, int l, const std::string& path);

}  // namespace subsurf
